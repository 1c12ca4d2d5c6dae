#include <cstdlib>
#include <mutex>
// api.cu — the C ABI declared in include/pga.h.  Argument validation, the
// per-island runtime (buffers, stream, CUDA graph of one generation) and the
// host<->device marshalling.  Every step of the method runs in the kernels of
// fitness.cu / ga.cu / corr.cu; nothing here computes on the host beyond
// label base conversion (1-based <-> 0-based) at the boundary.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pga_internal.cuh"

namespace pga {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string &m) { g_err = m; }
int fail(int code, const std::string &m) {
    g_err = m;
    return code;
}
int cuda_fail(cudaError_t e, const char *what) {
    g_err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    return PGA_EDEVICE;
}
void count_launch(int n) { g_launches += n; }

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("PGA_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

cudaError_t prof_record(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaError_t r = cudaStreamIsCapturing(s, &st);
    if (r != cudaSuccess) return r;
    return st == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                               : cudaEventRecord(e, s);
}

// declared in ga.cu / fitness.cu
int launch_resync_gm(pga_ctx *c, cudaStream_t s);
int launch_init_raw(uint64_t seed, int N, int ldn, int64_t P, int64_t Pcap, int64_t p_off,
                    uint32_t island, uint16_t *CM, uint16_t *GM, int32_t *out32, cudaStream_t s);
int run_select_ops(const double *L, int64_t P, const pga_params &p, int32_t gen, int32_t island,
                   int32_t *order, int32_t *sel, uint64_t *keys_in, uint64_t *keys_out,
                   int32_t *idx_in, int32_t *rank, uint64_t *q, uint64_t *bsum, const int32_t *done,
                   cudaStream_t s, const int32_t *gen_ptr, bool sorted, int32_t *sigma);
int run_mates(int64_t M, const pga_params &p, int32_t gen, int32_t island, int32_t *sigma, cudaStream_t s);
int launch_breed_hook(const int32_t *pop, const int32_t *top, const int32_t *order, int64_t P,
                      int N, const int32_t *sel, const int32_t *sigma, const pga_params &p,
                      int32_t gen, int32_t island, int64_t p_off, int32_t *next, cudaStream_t s);
int launch_set_pop(pga_ctx *c, const int32_t *lab32, int par, cudaStream_t s);
int prepare_breed(int N);
int prepare_select_small();
int prepare_rank_sel(pga_ctx *c);
bool small_select(const pga_ctx *c);
long long viol_fitness();
int launch_fast_ln(const double *x, int64_t n, const double *lgtab, int N, double *out, cudaStream_t s);
long long viol_ga();

static int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

int check_params(const pga_params *p) {
    if (!p) return fail(PGA_EINVAL, "params is NULL");
    if (p->pop_size < 2) return fail(PGA_EINVAL, "pop_size must be >= 2 (S:113)");
    if (p->pop_size > (1 << 26)) return fail(PGA_EINVAL, "pop_size too large");
    if (p->elite < 0 || p->elite >= p->pop_size)
        return fail(PGA_EINVAL, "elite must satisfy 0 <= elite < pop_size (S:113)");
    auto prob = [](double x) { return std::isfinite(x) && x >= 0.0 && x <= 1.0; };
    if (!prob(p->p_crossover) || !prob(p->p_mutation) || !prob(p->p_kb))
        return fail(PGA_EINVAL, "probabilities must lie in [0, 1]");
    if (!std::isfinite(p->tol)) return fail(PGA_EINVAL, "tol must be finite");
    if (p->stall_gens < 1) return fail(PGA_EINVAL, "stall_gens must be >= 1");
    if (p->max_gens < 1) return fail(PGA_EINVAL, "max_gens must be >= 1");
    if (p->selection != PGA_SEL_SUS && p->selection != PGA_SEL_TOURNAMENT)
        return fail(PGA_EINVAL, "selection must be PGA_SEL_SUS or PGA_SEL_TOURNAMENT");
    if (p->tournament_k < 1 || p->tournament_k > 4) return fail(PGA_EINVAL, "tournament_k must be 1..4");
    if (p->scaling != PGA_SCALE_RANK && p->scaling != PGA_SCALE_NONE)
        return fail(PGA_EINVAL, "scaling must be PGA_SCALE_RANK or PGA_SCALE_NONE");
    if (p->n_islands < 1 || p->n_islands > 8) return fail(PGA_EINVAL, "n_islands must be 1..8");
    if (p->island < 0 || p->island >= p->n_islands) return fail(PGA_EINVAL, "island out of range");
    if (p->device < 0) return fail(PGA_EINVAL, "device must be >= 0");
    if (p->n_islands > 1) {
        if (p->migrate_every < 1) return fail(PGA_EINVAL, "migrate_every must be >= 1");
        if (p->migrants < 1 || p->migrants > 256 || p->migrants > p->pop_size)
            return fail(PGA_EINVAL, "migrants must be 1..min(256, pop_size)");
    }
    return PGA_OK;
}

int check_corr(const double *C, int32_t N) {
    if (!C) return fail(PGA_EINVAL, "C is NULL");
    if (N < 2 || N > 16384) return fail(PGA_EINVAL, "N must be in [2, 16384]");
    for (int64_t i = 0; i < N; ++i) {
        for (int64_t j = 0; j < N; ++j) {
            const double v = C[i * N + j];
            if (!std::isfinite(v)) return fail(PGA_EINVAL, "C has a non-finite entry");
            if (i == j) {
                if (std::fabs(v - 1.0) > 1e-12) return fail(PGA_EINVAL, "C_ii must be 1 (+-1e-12)");
            } else {
                if (std::fabs(v) > 1.0 + 1e-9) return fail(PGA_EINVAL, "|C_ij| must be <= 1 + 1e-9");
                if (v != C[j * N + i]) return fail(PGA_EINVAL, "C must be exactly symmetric (Q4)");
            }
        }
    }
    return PGA_OK;
}

int ensure_device(int dev) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) return fail(PGA_EDEVICE, "no CUDA device available (libpga has no CPU fallback)");
    if (dev >= n) return fail(PGA_EINVAL, "device ordinal out of range");
    PGA_CUDA(cudaSetDevice(dev));
    return PGA_OK;
}

}  // namespace pga

using namespace pga;

// Device buffers of the ABI come from a per-device memory pool of the
// library that keeps up to PGA_POOL_KEEP_MB (default 4096) MiB of freed
// memory mapped for later allocations in the process: a context created
// after an earlier one was destroyed reuses its pages instead of mapping
// new ones (cudaMalloc of C4's ~0.7 GB costs 15-40 ms).  Allocation and free
// are made synchronous, like cudaMalloc / cudaFree.
cudaMemPool_t pga::lib_pool(int *err) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    *err = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        *err = 1;
        return nullptr;
    }
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
        cudaMemPoolProps pr = {};
        pr.allocType = cudaMemAllocationTypePinned;
        pr.location.type = cudaMemLocationTypeDevice;
        pr.location.id = dev;
        if (cudaMemPoolCreate(&pools[dev], &pr) != cudaSuccess) {
            pools[dev] = nullptr;
            *err = 1;
            return nullptr;
        }
        uint64_t keep = 4096ull << 20;
        if (const char *e = std::getenv("PGA_POOL_KEEP_MB")) keep = std::strtoull(e, nullptr, 10) << 20;
        cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    return pools[dev];
}


namespace {


void drop_graph(GExec &g) {
    if (g.x) cudaGraphExecDestroy(g.x);
    if (g.g) cudaGraphDestroy(g.g);
    g = GExec{};
}

void drop_graphs(pga_ctx *c) {
    drop_graph(c->gx_eval[0]);
    drop_graph(c->gx_eval[1]);
    drop_graph(c->gx_breed[0]);
    drop_graph(c->gx_breed[1]);
}

static void dfree(void *p);

void free_ctx(pga_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    drop_graphs(c);
    void *ptrs[] = {c->C, c->diag, c->lgtab, c->sflag, c->sp_live, c->sp_blocks, c->cc, c->cc_state,
                    c->stats_part, c->stats_ctr,
                    c->cc_keys, c->ptab, c->pop[0], c->pop[1], c->popT[0], c->popT[1], c->V, c->L,
                    c->top, c->keys_in, c->keys_out, c->idx_in, c->order, c->q, c->rank, c->rc_acc, c->rc_qtab,
                    c->sel, c->sigma, c->breed_ctr, c->mmask, c->st,
                    c->best_labels, c->history, c->stage_i32, c->evCM, c->evGM, c->evL,
                    c->counters};
    for (void *p : ptrs) dfree(p);
    delete c->h_st;
    for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
    if (c->join_ev) cudaEventDestroy(c->join_ev);
    if (c->fork_ev) cudaEventDestroy(c->fork_ev);
    if (c->join_side_ev) cudaEventDestroy(c->join_side_ev);
    if (c->fit_ev) cudaEventDestroy(c->fit_ev);
    if (c->stats_ev) cudaEventDestroy(c->stats_ev);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->stream) cudaStreamDestroy(c->stream);
}

template <typename T>
int dalloc(T **p, size_t count) {
    int perr = 0;
    cudaMemPool_t pool = lib_pool(&perr);
    if (perr) return fail(PGA_EDEVICE, "device memory pool unavailable");
    cudaError_t e = cudaMallocFromPoolAsync((void **)p, sizeof(T) * (count ? count : 1), pool, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    if (e != cudaSuccess) return fail(PGA_ENOMEM, std::string("device allocation failed: ") + cudaGetErrorString(e));
    return PGA_OK;
}

// the counterpart of dalloc (waits for the device, as cudaFree does)
static void dfree(void *p) {
    if (!p) return;
    cudaDeviceSynchronize();
    cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
}

#define TRY(x)                 \
    do {                       \
        int _rc = (x);         \
        if (_rc) return _rc;   \
    } while (0)

int reset_state(pga_ctx *c, int32_t max_gens) {
    DevState h{};
    h.gen = 0;
    h.best_ever = -1.0;
    *c->h_st = h;
    PGA_CUDA(cudaMemcpyAsync(c->st, c->h_st, sizeof(DevState), cudaMemcpyHostToDevice, c->stream));
    const int32_t live[6] = {1, 0, 0, 0, 0, 0};   // re-arm the label-sparse check (f2) for a new population
    PGA_CUDA(cudaMemcpyAsync(c->sp_live, live, sizeof(live), cudaMemcpyHostToDevice, c->stream));
    PGA_CUDA(cudaStreamSynchronize(c->stream));
    (void)max_gens;
    return PGA_OK;
}

int read_state(pga_ctx *c) {
    PGA_CUDA(cudaMemcpyAsync(c->h_st, c->st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
    PGA_CUDA(cudaStreamSynchronize(c->stream));
    return PGA_OK;
}

int ensure_history(pga_ctx *c, int32_t n) {
    if (n <= c->hist_cap) return PGA_OK;
    double *h = nullptr;
    TRY(dalloc(&h, (size_t)n));
    PGA_CUDA(cudaMemsetAsync(h, 0, sizeof(double) * n, c->stream));
    if (c->history) {
        PGA_CUDA(cudaMemcpyAsync(h, c->history, sizeof(double) * c->hist_cap, cudaMemcpyDeviceToDevice, c->stream));
        PGA_CUDA(cudaStreamSynchronize(c->stream));
        dfree(c->history);
    }
    c->history = h;
    c->hist_cap = n;
    return PGA_OK;
}

FitBufs ga_bufs(pga_ctx *c) {
    FitBufs b;
    b.cm0 = c->pop[0];
    b.cm1 = c->pop[1];
    b.gm0 = c->popT[0];
    b.gm1 = c->popT[1];
    b.tm0 = &c->tmLab[0];
    b.tm1 = &c->tmLab[1];
    b.gen = &c->st->gen;
    b.done = &c->st->done;
    return b;
}

bool is_migration_gen(const pga_ctx *c, int32_t g) {
    return c->p.n_islands > 1 && ((g + 1) % c->p.migrate_every == 0);
}

cudaEvent_t *prof_slot(pga_ctx *c) {
    if (!c->prof) return nullptr;
    while (c->prof_ev.size() < c->prof_used + PROF_EV) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        c->prof_ev.push_back(e);
    }
    return &c->prof_ev[c->prof_used];
}

// Phase marks (profiling only): 0 start, 1 sweep end, 2 fitness end,
// 3 statistics end, 4 order sort end, 5 selection end, 6 mating end,
// 7 breed end, 8 generation end.
int phase_a(pga_ctx *c, int32_t g, int32_t *is_mig) {
    c->pev = prof_slot(c);
    TRY(launch_mates_fork(c, c->stream));   // mate slots beside the fitness pass
    TRY(launch_fitness(c, ga_bufs(c), c->P, c->L, c->top, c->stream, c->pev));
    const bool mig = is_migration_gen(c, g);
    if (is_mig) *is_mig = mig ? 1 : 0;
    if (mig) {
        TRY(launch_sort_order(c, c->stream));
        c->pending_migration = true;
        PGA_MARK(c, 3, c->stream);
    } else {
        // statistics / termination on the side stream, concurrent with the
        // selection on the main stream: both only read L (the breed skips a
        // generation the statistics stop); joined before phase A ends
        PGA_CUDA(cudaEventRecord(c->fit_ev, c->stream));
        PGA_CUDA(cudaStreamWaitEvent(c->side, c->fit_ev, 0));
        TRY(launch_stats(c, c->p.n_islands > 1 ? 1 : 0, c->side));
        if (mutmask_late(c)) TRY(launch_mutmask(c, c->side));   // read by this generation's breed
        PGA_CUDA(cudaEventRecord(c->stats_ev, c->side));
        TRY(launch_select(c, c->stream));
        PGA_CUDA(cudaStreamWaitEvent(c->stream, c->stats_ev, 0));
        PGA_MARK(c, 3, c->stream);
    }
    TRY(launch_mates_join(c, c->stream));
    return PGA_OK;
}

// Phase B.  fresh: phase A of this generation already selected (non-migration
// generations); otherwise (after a migration import or a replicated commit)
// the selection runs here.
int phase_b(pga_ctx *c, bool fresh) {
    if (!fresh) TRY(launch_select(c, c->stream));
    PGA_MARK(c, 4, c->stream);
    PGA_MARK(c, 5, c->stream);
    PGA_MARK(c, 6, c->stream);
    TRY(launch_breed(c, c->stream, fresh));
    if (c->pev) {
        PGA_CUDA(prof_record(c->pev[8], c->stream));
        c->prof_used += PROF_EV;
        c->pev = nullptr;
    }
    return PGA_OK;
}

// Capture fn()'s launches on c->stream into *g.  Profiling: the events fn()
// records (this generation's slot of prof_ev) become event-record nodes,
// remembered with their phase-mark index so that every replay records into
// that generation's own slot (launch_graph).
template <class F>
int capture_graph(pga_ctx *c, GExec *g, F fn) {
    drop_graph(*g);
    const size_t base = c->prof_used;
    const size_t pu = c->prof_used;
    const int64_t k0 = g_launches;
    PGA_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const int rc = fn();
    g->nk = (int)(g_launches - k0);
    g_launches -= g->nk;   // counted at every replay instead
    c->prof_used = pu;     // fn()'s bookkeeping is redone per replay
    cudaError_t e = cudaStreamEndCapture(c->stream, &g->g);
    if (rc || e != cudaSuccess) {
        drop_graph(*g);
        return rc ? rc : cuda_fail(e, "cudaStreamEndCapture");
    }
    if (c->prof) {
        size_t n = 0;
        PGA_CUDA(cudaGraphGetNodes(g->g, nullptr, &n));
        std::vector<cudaGraphNode_t> nodes(n);
        PGA_CUDA(cudaGraphGetNodes(g->g, nodes.data(), &n));
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType t;
            PGA_CUDA(cudaGraphNodeGetType(nd, &t));
            if (t != cudaGraphNodeTypeEventRecord) continue;
            cudaEvent_t ev;
            PGA_CUDA(cudaGraphEventRecordNodeGetEvent(nd, &ev));
            for (int k = 0; k < PROF_EV; ++k)
                if (base + k < c->prof_ev.size() && c->prof_ev[base + k] == ev) g->evn.emplace_back(nd, k);
        }
    }
    e = cudaGraphInstantiate(&g->x, g->g, c->use_prio ? cudaGraphInstantiateFlagUseNodePriority : 0);
    if (e != cudaSuccess) {
        drop_graph(*g);
        return cuda_fail(e, "cudaGraphInstantiate");
    }
    return PGA_OK;
}

int launch_graph(pga_ctx *c, GExec &g) {
    if (!g.evn.empty()) {
        cudaEvent_t *slot = prof_slot(c);
        if (!slot) return fail(PGA_EDEVICE, "profiling events unavailable");
        for (auto &ne : g.evn) PGA_CUDA(cudaGraphExecEventRecordNodeSetEvent(g.x, ne.first, slot[ne.second]));
    }
    PGA_CUDA(cudaGraphLaunch(g.x, c->stream));
    count_launch(g.nk);
    return PGA_OK;
}

// one single-island generation, captured once into a CUDA graph
int run_one_generation(pga_ctx *c, GExec &g, bool use_graph) {
    if (!use_graph) {
        TRY(phase_a(c, 0, nullptr));
        return phase_b(c, true);
    }
    if (!g.x)
        TRY(capture_graph(c, &g, [&] {
            int rc = phase_a(c, 0, nullptr);
            return rc ? rc : phase_b(c, true);
        }));
    return launch_graph(c, g);
}

void to_one_based(const std::vector<uint16_t> &src, int32_t *dst, size_t n) {
    for (size_t i = 0; i < n; ++i) dst[i] = (int32_t)src[i] + 1;
}

struct HookBufs {
    std::vector<void *> ptrs;
    ~HookBufs() {
        for (void *p : ptrs) dfree(p);
    }
    template <typename T>
    int get(T **p, size_t n) {
        int rc = dalloc(p, n);
        if (!rc) ptrs.push_back((void *)*p);
        return rc;
    }
};

int ensure_eval_bufs(pga_ctx *c) {
    if (c->evCM) return PGA_OK;
    TRY(dalloc(&c->evCM, (size_t)c->Pcap * c->ldn));
    TRY(dalloc(&c->evGM, (size_t)c->N * c->Pcap));
    TRY(dalloc(&c->evL, (size_t)c->Pcap));
    PGA_CUDA(cudaMemsetAsync(c->evCM, 0, sizeof(uint16_t) * (size_t)c->Pcap * c->ldn, c->stream));
    PGA_CUDA(cudaMemsetAsync(c->evGM, 0, sizeof(uint16_t) * (size_t)c->N * c->Pcap, c->stream));
    PGA_CUDA(cudaStreamSynchronize(c->stream));
    TRY(make_label_tmap(&c->tmLabEv, c->evGM, c->N, c->Pcap));
    return PGA_OK;
}

}  // namespace

// ===========================================================================
// ABI
// ===========================================================================
extern "C" {

const char *pga_last_error(void) { return g_err.c_str(); }

int64_t pga_launch_count(void) { return g_launches.load(); }

int64_t pga_debug_violations(void) {
    const long long a = viol_fitness(), b = viol_ga();
    if (a < 0 || b < 0) return a < b ? a : b;
    return a + b;
}

int pga_params_default(pga_params *o) {
    if (!o) return fail(PGA_EINVAL, "out is NULL");
    std::memset(o, 0, sizeof(*o));
    o->pop_size = 1000;   // Table 3 context
    o->elite = 10;
    o->p_crossover = 0.9;
    o->p_mutation = 0.1;
    o->p_kb = 0.9;
    o->tol = 1e-5;
    o->stall_gens = 50;
    o->max_gens = 400;
    o->selection = PGA_SEL_SUS;
    o->tournament_k = 2;
    o->scaling = PGA_SCALE_RANK;
    o->device = 0;
    o->island = 0;
    o->n_islands = 1;
    o->migrate_every = 10;
    o->migrants = 10;
    o->seed = 1;
    return PGA_OK;
}

struct pga_graphs_holder;

int pga_create(const double *C, int32_t N, const pga_params *p, pga_ctx **out) {
    if (!out) return fail(PGA_EINVAL, "out is NULL");
    *out = nullptr;
    TRY(check_params(p));
    TRY(check_corr(C, N));
    TRY(ensure_device(p->device));
    pga_ctx *c = new pga_ctx();
    c->device = p->device;
    c->p = *p;
    c->N = N;
    c->ldn = (int32_t)round_up(N, 16);   // fitness tiles write 16 rows per warp
    c->ldc = (int32_t)round_up(N, 8);
    c->P = p->pop_size;
    c->Pcap = round_up(p->pop_size, CB);
    auto bail = [&](int rc) {
        free_ctx(c);
        delete c;
        return rc;
    };
    // stream priorities: the side branch (mate slots, statistics, mutation
    // masks) yields SM slots to the generation's critical path
    int prio_lo = 0, prio_hi = 0;
    {
        const char *np = std::getenv("PGA_NO_PRIO");
        if (!(np && np[0] && np[0] != '0')) cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
        c->use_prio = prio_lo != prio_hi;
    }
    cudaError_t e = cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaStreamCreate"));
    e = cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->join_side_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fit_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->stats_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_lo);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaEventCreate"));
    const size_t cm = (size_t)c->Pcap * c->ldn, gm = (size_t)N * c->Pcap;
    int rc = 0;
    rc = rc ? rc : dalloc(&c->C, (size_t)N * c->ldc);
    rc = rc ? rc : dalloc(&c->diag, (size_t)N);
    rc = rc ? rc : dalloc(&c->lgtab, (size_t)2 * (N + 1) + 2 * LN_TAB);
    rc = rc ? rc : dalloc(&c->sflag, (size_t)(c->Pcap / CB + 1));
    rc = rc ? rc : dalloc(&c->sp_live, (size_t)6);
    rc = rc ? rc : dalloc(&c->sp_blocks, (size_t)4);
    rc = rc ? rc : dalloc(&c->stats_part, (size_t)3 * 1024);
    rc = rc ? rc : dalloc(&c->stats_ctr, (size_t)1);
    if (!rc && cudaMemset(c->stats_ctr, 0, sizeof(uint32_t)) != cudaSuccess) rc = fail(PGA_EDEVICE, "memset stats_ctr");
    if (!rc && cudaMemset(c->sp_blocks, 0, 4 * sizeof(unsigned long long)) != cudaSuccess)
        rc = fail(PGA_EDEVICE, "memset sp_blocks");
    if (!rc && N <= SPARSE_MAX_N) {
        // cluster cache: 2^12 .. 2^22 slots (32 B each; 2^23 with PGA_CC_PER)
        uint32_t slots = 1u << 12;
        // 64 slots per chromosome (C4: 2^22 slots): fewer clears up to a few
        // hundred generations (20: 0.479 vs 0.498 ms, 100: 0.4666 vs 0.4698
        // against 32); 32 (2^21 slots, L2-resident) wins on long runs (1000
        // generations: 0.5238 vs 0.5420).  PGA_CC_PER overrides.
        int64_t per = 64;
        uint32_t cap = 1u << 22;
        if (const char *e = std::getenv("PGA_CC_PER")) {
            per = std::max<int64_t>(1, std::atoll(e));
            cap = 1u << 23;
        }
        while (slots < cap && (int64_t)slots < per * c->P) slots <<= 1;
        c->cc_mask = slots - 1u;
        rc = rc ? rc : dalloc(&c->cc, (size_t)slots);
        rc = rc ? rc : dalloc(&c->cc_state, (size_t)4);
        rc = rc ? rc : dalloc(&c->cc_keys, (size_t)2 * N);
        rc = rc ? rc : dalloc(&c->ptab, (size_t)N * c->ldc);
        if (!rc && (cudaMemset(c->cc, 0, sizeof(CCSlot) * slots) != cudaSuccess ||
                    cudaMemset(c->cc_state, 0, 4 * sizeof(uint32_t)) != cudaSuccess))
            rc = fail(PGA_EDEVICE, "memset cluster cache");
        if (!rc) {
            // Zobrist keys: splitmix64 of a fixed seed (any fixed keys do)
            std::vector<uint64_t> k(2 * (size_t)N);
            uint64_t x = 0x1403409900000001ull;
            for (auto &v : k) {
                uint64_t z = (x += 0x9E3779B97F4A7C15ull);
                z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
                z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
                v = z ^ (z >> 31);
            }
            if (cudaMemcpy(c->cc_keys, k.data(), sizeof(uint64_t) * k.size(), cudaMemcpyHostToDevice) != cudaSuccess)
                rc = fail(PGA_EDEVICE, "copy cache keys");
        }
    }
    for (int b = 0; b < 2 && !rc; ++b) {
        rc = rc ? rc : dalloc(&c->pop[b], cm);
        rc = rc ? rc : dalloc(&c->popT[b], gm);
    }
    rc = rc ? rc : dalloc(&c->V, cm);
    rc = rc ? rc : dalloc(&c->L, (size_t)c->Pcap);
    rc = rc ? rc : dalloc(&c->top, (size_t)c->Pcap);
    rc = rc ? rc : dalloc(&c->keys_in, (size_t)c->Pcap);
    rc = rc ? rc : dalloc(&c->keys_out, (size_t)c->Pcap);
    rc = rc ? rc : dalloc(&c->idx_in, (size_t)c->Pcap);
    rc = rc ? rc : dalloc(&c->order, (size_t)c->Pcap);
    rc = rc ? rc : dalloc(&c->q, (size_t)c->Pcap);
    rc = rc ? rc : dalloc(&c->rank, (size_t)c->Pcap);
    if (c->Pcap > 1024 && c->Pcap <= RANKC_MAXP) {
        rc = rc ? rc : dalloc(&c->rc_acc, (size_t)c->Pcap + 64);
        rc = rc ? rc : dalloc(&c->rc_qtab, (size_t)c->Pcap);
    }
    rc = rc ? rc : dalloc(&c->sel, (size_t)c->Pcap + 2);
    rc = rc ? rc : dalloc(&c->sigma, (size_t)c->Pcap + 2);
    rc = rc ? rc : dalloc(&c->breed_ctr, (size_t)1);
    rc = rc ? rc : dalloc(&c->mmask, (size_t)c->Pcap * ((N + 31) / 32));
    rc = rc ? rc : dalloc(&c->st, 1);
    rc = rc ? rc : dalloc(&c->best_labels, (size_t)c->ldn);
    rc = rc ? rc : dalloc(&c->counters, (size_t)(c->Pcap / CB));
    if (rc) return bail(rc);
    e = cudaMemsetAsync(c->counters, 0, sizeof(uint32_t) * (size_t)(c->Pcap / CB), c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->breed_ctr, 0, sizeof(uint32_t), c->stream);
    if (e == cudaSuccess && c->rc_acc)
        e = cudaMemsetAsync(c->rc_acc, 0, sizeof(int32_t) * ((size_t)c->Pcap + 64), c->stream);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaMemset counters"));
    // host copy of the device state: pageable (every read of it follows a
    // stream synchronisation; cudaMallocHost cost ~9 ms per context)
    c->h_st = new DevState();
    // population buffers: zero so padding chromosomes hold valid labels
    for (int b = 0; b < 2; ++b) {
        e = cudaMemsetAsync(c->pop[b], 0, sizeof(uint16_t) * cm, c->stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(c->popT[b], 0, sizeof(uint16_t) * gm, c->stream);
        if (e != cudaSuccess) return bail(cuda_fail(e, "cudaMemset"));
    }
    // C -> padded device layout, plus its diagonal
    {
        std::vector<double> diag(N);
        for (int i = 0; i < N; ++i) diag[i] = C[(int64_t)i * N + i];
        e = cudaMemsetAsync(c->C, 0, sizeof(double) * (size_t)N * c->ldc, c->stream);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(c->C, sizeof(double) * c->ldc, C, sizeof(double) * N,
                                  sizeof(double) * N, N, cudaMemcpyHostToDevice, c->stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(c->diag, diag.data(), sizeof(double) * N, cudaMemcpyHostToDevice, c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) return bail(cuda_fail(e, "copy C"));
    }
    rc = prepare_fitness(N);
    if (!rc) rc = launch_logtab(c, c->stream);
    if (!rc) rc = launch_pairtab(c, c->stream);
    if (!rc) rc = prepare_rank_sel(c);
    if (!rc && cudaStreamSynchronize(c->stream) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "log table");
    if (!rc) rc = prepare_breed(N);
    if (!rc) rc = prepare_select_small();
    if (!rc) rc = make_c_tmap(&c->tmC, c->C, N, c->ldc);
    if (!rc) rc = make_label_tmap(&c->tmLab[0], c->popT[0], N, c->Pcap);
    if (!rc) rc = make_label_tmap(&c->tmLab[1], c->popT[1], N, c->Pcap);
    if (rc) return bail(rc);
    rc = ensure_history(c, p->max_gens);
    if (rc) return bail(rc);
    {
        const int64_t rec = round_up(16 + 2 * (int64_t)N, 16);
        c->mig_bytes = rec * (p->n_islands > 1 ? p->migrants : 1);
    }
    rc = reset_state(c, p->max_gens);
    if (rc) return bail(rc);
    *out = c;
    return PGA_OK;
}

void pga_destroy(pga_ctx *c) {
    if (!c) return;
    free_ctx(c);
    delete c;
}

int pga_get_dims(pga_ctx *c, int32_t *N, int64_t *pop_size, int64_t *capacity) {
    if (!c) return fail(PGA_EINVAL, "ctx is NULL");
    if (N) *N = c->N;
    if (pop_size) *pop_size = c->P;
    if (capacity) *capacity = c->Pcap;
    return PGA_OK;
}

int pga_get_stream(pga_ctx *c, void **stream) {
    if (!c || !stream) return fail(PGA_EINVAL, "NULL argument");
    *stream = (void *)c->stream;
    return PGA_OK;
}

int pga_evaluate(pga_ctx *c, const int32_t *labels, int64_t P, double *out_L) {
    if (!c || !labels || !out_L) return fail(PGA_EINVAL, "NULL argument");
    if (P < 1) return fail(PGA_EINVAL, "P must be >= 1");
    PGA_CUDA(cudaSetDevice(c->device));
    if (!c->stage_i32) TRY(dalloc(&c->stage_i32, (size_t)c->Pcap * c->N));
    TRY(ensure_eval_bufs(c));
    const int32_t zero = 0;
    for (int64_t p0 = 0; p0 < P; p0 += c->Pcap) {
        const int64_t n = (P - p0 < c->Pcap) ? (P - p0) : c->Pcap;
        PGA_CUDA(cudaMemcpyAsync(&c->st->pack_error, &zero, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
        PGA_CUDA(cudaMemcpyAsync(c->stage_i32, labels + p0 * c->N, sizeof(int32_t) * (size_t)n * c->N,
                                 cudaMemcpyHostToDevice, c->stream));
        TRY(launch_pack(c, nullptr, c->stage_i32, n, c->N, c->evCM, c->evGM, c->stream));
        FitBufs b{c->evCM, c->evCM, c->evGM, c->evGM, &c->tmLabEv, &c->tmLabEv, nullptr, nullptr};
        TRY(launch_fitness(c, b, n, c->evL, nullptr, c->stream));
        int32_t perr = 0;
        PGA_CUDA(cudaMemcpyAsync(out_L + p0, c->evL, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        PGA_CUDA(cudaMemcpyAsync(&perr, &c->st->pack_error, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
        PGA_CUDA(cudaStreamSynchronize(c->stream));
        if (perr) return fail(PGA_EINVAL, "labels must lie in 1..N (Eq. 9)");
    }
    return PGA_OK;
}

int pga_evaluate_device(pga_ctx *c, const uint16_t *labels_dev, int64_t P, double *L_dev,
                        uint16_t *top_dev, void *stream) {
    if (!c || !labels_dev || !L_dev) return fail(PGA_EINVAL, "NULL argument");
    if (P < 1 || P > c->Pcap) return fail(PGA_EINVAL, "P must be in [1, capacity]");
    cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
    if (!c->evCM) {
        PGA_CUDA(cudaSetDevice(c->device));
        TRY(ensure_eval_bufs(c));
    }
    // the evaluation scratch (evCM/evGM, V, counters, sflag, cache state) is
    // per ctx: join a foreign stream to the ctx's stream in both directions
    const bool foreign = s != c->stream;
    if (foreign) {
        PGA_CUDA(cudaEventRecord(c->join_ev, c->stream));
        PGA_CUDA(cudaStreamWaitEvent(s, c->join_ev, 0));
    }
    TRY(launch_pack(c, labels_dev, nullptr, P, c->N, c->evCM, c->evGM, s));
    FitBufs b{c->evCM, c->evCM, c->evGM, c->evGM, &c->tmLabEv, &c->tmLabEv, nullptr, nullptr};
    TRY(launch_fitness(c, b, P, L_dev, top_dev, s));
    if (foreign) {
        PGA_CUDA(cudaEventRecord(c->join_ev, s));
        PGA_CUDA(cudaStreamWaitEvent(c->stream, c->join_ev, 0));
    }
    return PGA_OK;
}

int pga_init(pga_ctx *c, uint64_t seed) {
    if (!c) return fail(PGA_EINVAL, "ctx is NULL");
    PGA_CUDA(cudaSetDevice(c->device));
    c->p.seed = seed;
    TRY(reset_state(c, c->p.max_gens));
    TRY(launch_init(c, seed, c->stream));
    c->has_pop = true;
    c->host_gen = 0;
    c->pending_migration = false;
    c->sel_fresh = false;
    return PGA_OK;
}

int pga_gen_evaluate(pga_ctx *c, int32_t *is_migration) {
    if (!c) return fail(PGA_EINVAL, "ctx is NULL");
    if (!c->has_pop) return fail(PGA_ESTATE, "no population: call pga_init first");
    if (c->pending_migration) return fail(PGA_ESTATE, "migration pending: call pga_import_migrants");
    PGA_CUDA(cudaSetDevice(c->device));
    // replay of the cached graph for this kind of generation (the host
    // decides migration generations, so each kind has its own graph)
    const bool mig = is_migration_gen(c, c->host_gen);
    GExec &g = c->gx_eval[mig ? 1 : 0];
    if (!g.x) TRY(capture_graph(c, &g, [&] { return phase_a(c, c->host_gen, nullptr); }));
    TRY(launch_graph(c, g));
    c->pev = prof_slot(c);   // this generation's slot (null unless profiling)
    c->pending_migration = mig;
    c->sel_fresh = !mig;     // phase A selected beside its statistics
    if (is_migration) *is_migration = mig ? 1 : 0;
    return PGA_OK;
}

int pga_set_sparse_threshold(pga_ctx *c, double theta) {
    if (!c) return fail(PGA_EINVAL, "ctx is NULL");
    if (!(theta <= 1.0)) return fail(PGA_EINVAL, "theta must lie in [0, 1] (negative = automatic)");
    const bool was_on = sparse_theta_eff(c) > 0.0;
    c->sparse_theta = theta < 0.0 ? -1.0 : theta;
    drop_graphs(c);   // the launch sequence depends on it
    if (was_on && !(sparse_theta_eff(c) > 0.0) && c->has_pop && c->N <= SPARSE_MAX_N) {
        // the breed may have left the gene-major copy to the sparse pass
        PGA_CUDA(cudaSetDevice(c->device));
        TRY(launch_resync_gm(c, c->stream));
    }
    return PGA_OK;
}

int pga_rep_evaluate(pga_ctx *c, int64_t begin, int64_t end, double *L_dev, uint16_t *top_dev) {
    if (!c || !L_dev || !top_dev) return fail(PGA_EINVAL, "NULL argument");
    if (c->p.n_islands != 1) return fail(PGA_ESTATE, "replicated mode needs n_islands = 1 (one population)");
    if (!c->has_pop) return fail(PGA_ESTATE, "no population: call pga_init first");
    if (begin < 0 || end > c->P || begin >= end || begin % CB)
        return fail(PGA_EINVAL, "need 0 <= begin < end <= pop_size and begin a multiple of 32");
    PGA_CUDA(cudaSetDevice(c->device));
    c->pev = prof_slot(c);
    return launch_fitness_range(c, ga_bufs(c), begin, end, L_dev - begin, top_dev - begin, c->stream,
                                c->pev);
}

int pga_rep_commit(pga_ctx *c, const double *L_dev, const uint16_t *top_dev) {
    if (!c || !L_dev || !top_dev) return fail(PGA_EINVAL, "NULL argument");
    if (c->p.n_islands != 1) return fail(PGA_ESTATE, "replicated mode needs n_islands = 1 (one population)");
    if (!c->has_pop) return fail(PGA_ESTATE, "no population: call pga_init first");
    PGA_CUDA(cudaSetDevice(c->device));
    PGA_CUDA(cudaMemcpyAsync(c->L, L_dev, sizeof(double) * c->P, cudaMemcpyDeviceToDevice, c->stream));
    PGA_CUDA(cudaMemcpyAsync(c->top, top_dev, sizeof(uint16_t) * c->P, cudaMemcpyDeviceToDevice, c->stream));
    TRY(launch_mates_fork(c, c->stream));   // mate slots of this generation (phase_a does it on the GA path)
    TRY(launch_stats(c, 0, c->stream));
    TRY(launch_mates_join(c, c->stream));
    c->sel_fresh = false;    // phase B selects from the committed L
    PGA_MARK(c, 3, c->stream);
    return PGA_OK;
}

int pga_gen_breed(pga_ctx *c) {
    if (!c) return fail(PGA_EINVAL, "ctx is NULL");
    if (!c->has_pop) return fail(PGA_ESTATE, "no population: call pga_init first");
    if (c->pending_migration) return fail(PGA_ESTATE, "migration pending: call pga_import_migrants");
    PGA_CUDA(cudaSetDevice(c->device));
    const bool profiled = c->pev != nullptr;   // phase_b clears it while being captured
    const int f = c->sel_fresh ? 1 : 0;
    if (!c->gx_breed[f].x) TRY(capture_graph(c, &c->gx_breed[f], [&] { return phase_b(c, f == 1); }));
    TRY(launch_graph(c, c->gx_breed[f]));
    c->sel_fresh = false;
    if (profiled) c->prof_used += PROF_EV;   // as phase_b does in plain launches
    c->pev = nullptr;
    c->host_gen += 1;
    return PGA_OK;
}

int pga_generation(pga_ctx *c, int32_t *done) {
    if (!c) return fail(PGA_EINVAL, "ctx is NULL");
    if (c->p.n_islands > 1) return fail(PGA_ESTATE, "pga_generation is single-island; use pga_gen_evaluate/breed");
    TRY(pga_gen_evaluate(c, nullptr));
    TRY(pga_gen_breed(c));
    if (done) {
        TRY(read_state(c));
        *done = c->h_st->done;
    }
    return PGA_OK;
}

int pga_run(pga_ctx *c, int32_t gens, uint64_t seed, int32_t *best_labels, double *best_L,
            int32_t *gens_run, int32_t *reason) {
    if (!c) return fail(PGA_EINVAL, "ctx is NULL");
    if (c->p.n_islands > 1) return fail(PGA_ESTATE, "pga_run is single-island; drive islands with pga_gen_evaluate/breed");
    PGA_CUDA(cudaSetDevice(c->device));
    drop_graphs(c);   // max_gens is changed for this run (a kernel argument)
    const int32_t saved_max = c->p.max_gens;
    const int32_t maxg = gens > 0 ? gens : c->p.max_gens;
    TRY(ensure_history(c, maxg));
    c->p.max_gens = maxg;
    int rc = pga_init(c, seed);
    GExec g;
    int32_t launched = 0;
    const int32_t batch = 8;
    while (!rc) {
        for (int k = 0; k < batch && launched < maxg && !rc; ++k, ++launched)
            rc = run_one_generation(c, g, !c->prof);   // profiling events need plain launches
        if (rc) break;
        rc = read_state(c);
        if (rc) break;
        if (c->h_st->done || launched >= maxg) break;
    }
    drop_graph(g);
    c->p.max_gens = saved_max;
    if (rc) return rc;
    c->host_gen = c->h_st->gen;
    if (best_L) *best_L = c->h_st->best_ever;
    if (gens_run) *gens_run = c->h_st->gen + 1;
    if (reason) *reason = c->h_st->reason;
    if (best_labels) {
        std::vector<uint16_t> h(c->N);
        PGA_CUDA(cudaMemcpy(h.data(), c->best_labels, sizeof(uint16_t) * c->N, cudaMemcpyDeviceToHost));
        to_one_based(h, best_labels, c->N);
    }
    return PGA_OK;
}

int pga_get_state(pga_ctx *c, int32_t *generation, int32_t *done, int32_t *reason, double *best_L,
                  double *mean_L, int32_t *best_labels) {
    if (!c) return fail(PGA_EINVAL, "ctx is NULL");
    PGA_CUDA(cudaSetDevice(c->device));
    TRY(read_state(c));
    if (generation) *generation = c->h_st->gen;
    if (done) *done = c->h_st->done;
    if (reason) *reason = c->h_st->reason;
    if (best_L) *best_L = c->h_st->best_ever;
    if (mean_L) *mean_L = c->h_st->mean;
    if (best_labels) {
        std::vector<uint16_t> h(c->N);
        PGA_CUDA(cudaMemcpy(h.data(), c->best_labels, sizeof(uint16_t) * c->N, cudaMemcpyDeviceToHost));
        to_one_based(h, best_labels, c->N);
    }
    return PGA_OK;
}

int pga_get_history(pga_ctx *c, double *best_L, int32_t n) {
    if (!c || !best_L) return fail(PGA_EINVAL, "NULL argument");
    if (n < 0 || n > c->hist_cap) return fail(PGA_EINVAL, "n exceeds the history capacity");
    PGA_CUDA(cudaSetDevice(c->device));
    PGA_CUDA(cudaStreamSynchronize(c->stream));
    PGA_CUDA(cudaMemcpy(best_L, c->history, sizeof(double) * n, cudaMemcpyDeviceToHost));
    return PGA_OK;
}

int pga_get_population(pga_ctx *c, int32_t *labels, double *L, int32_t *top) {
    if (!c || !labels) return fail(PGA_EINVAL, "NULL argument");
    if (!c->has_pop) return fail(PGA_ESTATE, "no population");
    PGA_CUDA(cudaSetDevice(c->device));
    TRY(read_state(c));
    const int par = c->h_st->gen & 1;
    std::vector<uint16_t> h((size_t)c->P * c->ldn);
    PGA_CUDA(cudaMemcpy(h.data(), c->pop[par], sizeof(uint16_t) * h.size(), cudaMemcpyDeviceToHost));
    for (int64_t p = 0; p < c->P; ++p)
        for (int i = 0; i < c->N; ++i) labels[p * c->N + i] = (int32_t)h[p * c->ldn + i] + 1;
    if (L) PGA_CUDA(cudaMemcpy(L, c->L, sizeof(double) * c->P, cudaMemcpyDeviceToHost));
    if (top) {
        std::vector<uint16_t> t(c->P);
        PGA_CUDA(cudaMemcpy(t.data(), c->top, sizeof(uint16_t) * c->P, cudaMemcpyDeviceToHost));
        for (int64_t p = 0; p < c->P; ++p) top[p] = t[p] == 0xFFFF ? -1 : (int32_t)t[p];
    }
    return PGA_OK;
}

int pga_profile_enable(pga_ctx *c, int32_t on) {
    if (!c) return fail(PGA_EINVAL, "ctx is NULL");
    c->prof = on != 0;
    c->prof_level = on;
    drop_graphs(c);
    c->prof_used = 0;
    PGA_CUDA(cudaSetDevice(c->device));
    PGA_CUDA(cudaMemsetAsync(c->sp_blocks, 0, 4 * sizeof(unsigned long long), c->stream));
    return PGA_OK;
}

int pga_set_cluster_cache(pga_ctx *c, int32_t on) {
    if (!c) return fail(PGA_EINVAL, "ctx is NULL");
    c->cc_on = on != 0;
    drop_graphs(c);
    return PGA_OK;
}

int pga_profile_cache(pga_ctx *c, int64_t *hits, int64_t *saved) {
    if (!c || !hits || !saved) return fail(PGA_EINVAL, "NULL argument");
    PGA_CUDA(cudaSetDevice(c->device));
    unsigned long long v[4] = {0, 0, 0, 0};
    PGA_CUDA(cudaMemcpyAsync(v, c->sp_blocks, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
    PGA_CUDA(cudaStreamSynchronize(c->stream));
    *hits = (int64_t)v[2];
    *saved = (int64_t)v[3];
    return PGA_OK;
}

int pga_cache_stats(pga_ctx *c, int64_t *fill, int64_t *slots, int64_t *clears) {
    if (!c) return fail(PGA_EINVAL, "ctx is NULL");
    if (!c->cc) {
        if (fill) *fill = 0;
        if (slots) *slots = 0;
        if (clears) *clears = 0;
        return PGA_OK;
    }
    PGA_CUDA(cudaSetDevice(c->device));
    uint32_t v[4] = {0, 0, 0, 0};
    PGA_CUDA(cudaMemcpyAsync(v, c->cc_state, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
    PGA_CUDA(cudaStreamSynchronize(c->stream));
    if (fill) *fill = (int64_t)v[0];
    if (slots) *slots = (int64_t)c->cc_mask + 1;
    if (clears) *clears = (int64_t)v[3];
    return PGA_OK;
}

int pga_profile_sparse_blocks(pga_ctx *c, int64_t *sparse_blocks) {
    return pga_profile_sparse(c, sparse_blocks, nullptr);
}

int pga_profile_sparse(pga_ctx *c, int64_t *sparse_blocks, int64_t *gathered) {
    if (!c || !sparse_blocks) return fail(PGA_EINVAL, "NULL argument");
    PGA_CUDA(cudaSetDevice(c->device));
    unsigned long long v[2] = {0, 0};
    PGA_CUDA(cudaMemcpyAsync(v, c->sp_blocks, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
    PGA_CUDA(cudaStreamSynchronize(c->stream));
    *sparse_blocks = (int64_t)v[0];
    if (gathered) *gathered = (int64_t)v[1];
    return PGA_OK;
}

int pga_profile_read(pga_ctx *c, double *sweep_ms, double *fold_ms, double *gen_ms, int32_t *count) {
    if (!c) return fail(PGA_EINVAL, "ctx is NULL");
    PGA_CUDA(cudaSetDevice(c->device));
    PGA_CUDA(cudaStreamSynchronize(c->stream));
    double s = 0, g = 0, f = 0;
    int32_t n = 0;
    for (size_t k = 0; k + PROF_EV <= c->prof_used; k += PROF_EV) {
        float a = 0, d = 0, sp = 0;
        PGA_CUDA(cudaEventElapsedTime(&sp, c->prof_ev[k], c->prof_ev[k + 1]));
        PGA_CUDA(cudaEventElapsedTime(&a, c->prof_ev[k + 1], c->prof_ev[k + 2]));
        PGA_CUDA(cudaEventElapsedTime(&d, c->prof_ev[k], c->prof_ev[k + 8]));
        s += a;
        f += sp;
        g += d;
        ++n;
    }
    if (sweep_ms) *sweep_ms = s;
    if (fold_ms) *fold_ms = f;     // label-sparse pre-pass (the fold is fused into k_fitness)
    if (gen_ms) *gen_ms = g;
    if (count) *count = n;
    return PGA_OK;
}

int pga_profile_phases(pga_ctx *c, double *ms, int32_t *count) {
    if (!c || !ms) return fail(PGA_EINVAL, "NULL argument");
    if (c->prof_level < 2) return fail(PGA_ESTATE, "pga_profile_phases needs pga_profile_enable(ctx, 2)");
    PGA_CUDA(cudaSetDevice(c->device));
    PGA_CUDA(cudaStreamSynchronize(c->stream));
    double acc[PGA_PROF_PHASES] = {0};
    int32_t n = 0;
    for (size_t k = 0; k + PROF_EV <= c->prof_used; k += PROF_EV) {
        for (int j = 0; j < PGA_PROF_PHASES; ++j) {
            // phase 0: dense k_fitness (marks 1..2), phase 1: label-sparse pre-pass (0..1)
            float t = 0;
            const int a0 = (j == 0) ? 1 : (j == 1) ? 0 : j, a1 = (j == 0) ? 2 : (j == 1) ? 1 : j + 1;
            PGA_CUDA(cudaEventElapsedTime(&t, c->prof_ev[k + a0], c->prof_ev[k + a1]));
            acc[j] += t;
        }
        ++n;
    }
    for (int j = 0; j < PGA_PROF_PHASES; ++j) ms[j] = n ? acc[j] / n : 0.0;
    if (count) *count = n;
    return PGA_OK;
}

int pga_set_population(pga_ctx *c, const int32_t *labels, int32_t generation) {
    if (!c || !labels) return fail(PGA_EINVAL, "NULL argument");
    if (generation < 0) return fail(PGA_EINVAL, "generation must be >= 0");
    for (int64_t k = 0; k < c->P * (int64_t)c->N; ++k)
        if (labels[k] < 1 || labels[k] > c->N) return fail(PGA_EINVAL, "labels must lie in 1..N (Eq. 9)");
    PGA_CUDA(cudaSetDevice(c->device));
    TRY(reset_state(c, c->p.max_gens));
    if (!c->stage_i32) TRY(dalloc(&c->stage_i32, (size_t)c->Pcap * c->N));
    PGA_CUDA(cudaMemcpyAsync(c->stage_i32, labels, sizeof(int32_t) * (size_t)c->P * c->N,
                             cudaMemcpyHostToDevice, c->stream));
    TRY(launch_set_pop(c, c->stage_i32, generation & 1, c->stream));
    c->h_st->gen = generation;
    PGA_CUDA(cudaMemcpyAsync(&c->st->gen, &c->h_st->gen, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
    PGA_CUDA(cudaStreamSynchronize(c->stream));
    c->has_pop = true;
    c->host_gen = generation;
    c->pending_migration = false;
    c->sel_fresh = false;
    return PGA_OK;
}

int pga_migrant_bytes(pga_ctx *c, int64_t *bytes) {
    if (!c || !bytes) return fail(PGA_EINVAL, "NULL argument");
    *bytes = c->mig_bytes;
    return PGA_OK;
}

int pga_export_migrants(pga_ctx *c, void *dev_send) {
    if (!c || !dev_send) return fail(PGA_EINVAL, "NULL argument");
    if (!c->pending_migration) return fail(PGA_ESTATE, "not a migration generation");
    PGA_CUDA(cudaSetDevice(c->device));
    return launch_export(c, dev_send, c->stream);
}

int pga_import_migrants(pga_ctx *c, const void *dev_recv, int32_t n_islands) {
    if (!c || !dev_recv) return fail(PGA_EINVAL, "NULL argument");
    if (!c->pending_migration) return fail(PGA_ESTATE, "not a migration generation");
    if (n_islands != c->p.n_islands) return fail(PGA_EINVAL, "n_islands differs from the ctx's");
    PGA_CUDA(cudaSetDevice(c->device));
    TRY(launch_import(c, dev_recv, n_islands, c->stream));
    TRY(launch_stats(c, 2, c->stream));
    c->pending_migration = false;
    c->sel_fresh = false;    // L changed: phase B selects
    return PGA_OK;
}

int pga_correlation(const double *returns, int32_t T, int32_t N, double *C_out, int32_t device) {
    if (!returns || !C_out) return fail(PGA_EINVAL, "NULL argument");
    if (T < 2 || N < 1) return fail(PGA_EINVAL, "need T >= 2 and N >= 1");
    TRY(ensure_device(device));
    cudaStream_t s;
    PGA_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    double *X = nullptr, *C = nullptr;
    int32_t *st = nullptr;
    int rc = dalloc(&X, (size_t)T * N);
    rc = rc ? rc : dalloc(&C, (size_t)N * N);
    rc = rc ? rc : dalloc(&st, 1);
    int32_t hst = 0;
    if (!rc) {
        cudaError_t e = cudaMemcpyAsync(X, returns, sizeof(double) * (size_t)T * N, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(st, 0, sizeof(int32_t), s);
        rc = (e == cudaSuccess) ? launch_corr(X, T, N, C, st, s) : cuda_fail(e, "H2D returns");
        if (!rc) {
            e = cudaMemcpyAsync(C_out, C, sizeof(double) * (size_t)N * N, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(&hst, st, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) rc = cuda_fail(e, "pga_correlation");
        }
    }
    dfree(X);
    dfree(C);
    dfree(st);
    cudaStreamDestroy(s);
    if (!rc && hst) rc = fail(PGA_ENUMERIC, "zero-variance or non-finite column in returns");
    return rc;
}

int pga_correlation_device(const double *X_dev, int32_t T, int32_t N, double *C_dev,
                           int32_t *status_dev, void *stream) {
    if (!X_dev || !C_dev || !status_dev) return fail(PGA_EINVAL, "NULL argument");
    if (T < 2 || N < 1) return fail(PGA_EINVAL, "need T >= 2 and N >= 1");
    return launch_corr(X_dev, T, N, C_dev, status_dev, (cudaStream_t)stream);
}

int pga_op_select(const double *L, int64_t P, const pga_params *p, int32_t gen, int32_t island,
                  int32_t *order_out, int32_t *sel_out) {
    if (!L || !order_out || !sel_out || !p) return fail(PGA_EINVAL, "NULL argument");
    if (P < 2 || p->elite < 0 || p->elite >= P) return fail(PGA_EINVAL, "need P >= 2 and 0 <= elite < P");
    if (p->tournament_k < 1 || p->tournament_k > 4) return fail(PGA_EINVAL, "tournament_k must be 1..4");
    TRY(ensure_device(p->device));
    TRY(prepare_select_small());
    const int64_t M = 2 * ((P - p->elite + 1) / 2);
    HookBufs hb;
    double *dL;
    int32_t *dorder, *dsel, *didx, *drank;
    uint64_t *k1, *k2, *q, *bsum;
    TRY(hb.get(&dL, P));
    TRY(hb.get(&dorder, P));
    TRY(hb.get(&dsel, M));
    TRY(hb.get(&didx, P));
    TRY(hb.get(&drank, P));
    TRY(hb.get(&k1, P));
    TRY(hb.get(&k2, P));
    TRY(hb.get(&q, P));
    TRY(hb.get(&bsum, P / 1024 + 2));
    PGA_CUDA(cudaMemcpy(dL, L, sizeof(double) * P, cudaMemcpyHostToDevice));
    TRY(run_select_ops(dL, P, *p, gen, island, dorder, dsel, k1, k2, didx, drank, q, bsum, nullptr,
                       0, nullptr, false, nullptr));
    PGA_CUDA(cudaDeviceSynchronize());
    PGA_CUDA(cudaMemcpy(order_out, dorder, sizeof(int32_t) * P, cudaMemcpyDeviceToHost));
    PGA_CUDA(cudaMemcpy(sel_out, dsel, sizeof(int32_t) * M, cudaMemcpyDeviceToHost));
    return PGA_OK;
}

int pga_op_mates(int64_t M, const pga_params *p, int32_t gen, int32_t island, int32_t *sigma_out) {
    if (!p || !sigma_out) return fail(PGA_EINVAL, "NULL argument");
    if (M < 1) return fail(PGA_EINVAL, "M must be >= 1");
    TRY(ensure_device(p->device));
    HookBufs hb;
    int32_t *sig;
    TRY(hb.get(&sig, M));
    TRY(run_mates(M, *p, gen, island, sig, 0));
    PGA_CUDA(cudaDeviceSynchronize());
    PGA_CUDA(cudaMemcpy(sigma_out, sig, sizeof(int32_t) * M, cudaMemcpyDeviceToHost));
    return PGA_OK;
}

int pga_op_breed(const int32_t *pop, const int32_t *top, const int32_t *order, int64_t P, int32_t N,
                 const int32_t *sel, const int32_t *sigma, const pga_params *p, int32_t gen,
                 int32_t island, int64_t p_off, int32_t *next_out) {
    if (!pop || !top || !order || !sel || !sigma || !p || !next_out) return fail(PGA_EINVAL, "NULL argument");
    if (P < 2 || N < 2 || p->elite < 0 || p->elite >= P) return fail(PGA_EINVAL, "bad sizes");
    TRY(ensure_device(p->device));
    TRY(prepare_breed(N));
    const int64_t M = 2 * ((P - p->elite + 1) / 2);
    HookBufs hb;
    int32_t *dpop, *dtop, *dord, *dsel, *dsig, *dnext;
    TRY(hb.get(&dpop, (size_t)P * N));
    TRY(hb.get(&dtop, P));
    TRY(hb.get(&dord, P));
    TRY(hb.get(&dsel, M));
    TRY(hb.get(&dsig, M));
    TRY(hb.get(&dnext, (size_t)P * N));
    PGA_CUDA(cudaMemcpy(dpop, pop, sizeof(int32_t) * P * N, cudaMemcpyHostToDevice));
    PGA_CUDA(cudaMemcpy(dtop, top, sizeof(int32_t) * P, cudaMemcpyHostToDevice));
    PGA_CUDA(cudaMemcpy(dord, order, sizeof(int32_t) * P, cudaMemcpyHostToDevice));
    PGA_CUDA(cudaMemcpy(dsel, sel, sizeof(int32_t) * M, cudaMemcpyHostToDevice));
    PGA_CUDA(cudaMemcpy(dsig, sigma, sizeof(int32_t) * M, cudaMemcpyHostToDevice));
    TRY(launch_breed_hook(dpop, dtop, dord, P, N, dsel, dsig, *p, gen, island, p_off, dnext, 0));
    PGA_CUDA(cudaDeviceSynchronize());
    PGA_CUDA(cudaMemcpy(next_out, dnext, sizeof(int32_t) * P * N, cudaMemcpyDeviceToHost));
    return PGA_OK;
}

int pga_op_fast_ln(pga_ctx *c, const double *x, int64_t n, double *out) {
    if (!c || !x || !out) return fail(PGA_EINVAL, "NULL argument");
    if (n < 1) return fail(PGA_EINVAL, "n must be >= 1");
    for (int64_t i = 0; i < n; ++i)
        if (!(x[i] >= 2.2250738585072014e-308) || !std::isfinite(x[i])) return fail(PGA_EINVAL, "x must be positive normal");
    PGA_CUDA(cudaSetDevice(c->device));
    HookBufs hb;
    double *dx, *dy;
    TRY(hb.get(&dx, (size_t)n));
    TRY(hb.get(&dy, (size_t)n));
    PGA_CUDA(cudaMemcpy(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice));
    TRY(launch_fast_ln(dx, n, c->lgtab, c->N, dy, c->stream));
    PGA_CUDA(cudaStreamSynchronize(c->stream));
    PGA_CUDA(cudaMemcpy(out, dy, sizeof(double) * n, cudaMemcpyDeviceToHost));
    return PGA_OK;
}

int pga_op_canonicalize(int32_t *labels, int64_t P, int32_t N, int32_t device) {
    if (!labels) return fail(PGA_EINVAL, "NULL argument");
    if (P < 1 || N < 1) return fail(PGA_EINVAL, "bad sizes");
    for (int64_t k = 0; k < P * (int64_t)N; ++k)
        if (labels[k] < 0 || labels[k] > 2 * N) return fail(PGA_EINVAL, "labels must lie in 0..2N");
    TRY(ensure_device(device));
    HookBufs hb;
    int32_t *d;
    TRY(hb.get(&d, (size_t)P * N));
    PGA_CUDA(cudaMemcpy(d, labels, sizeof(int32_t) * P * N, cudaMemcpyHostToDevice));
    TRY(launch_canonicalize_i32(d, P, N, 0));
    PGA_CUDA(cudaDeviceSynchronize());
    PGA_CUDA(cudaMemcpy(labels, d, sizeof(int32_t) * P * N, cudaMemcpyDeviceToHost));
    return PGA_OK;
}

int pga_op_init(uint64_t seed, int32_t N, int64_t P, int64_t p_off, int32_t island, int32_t device,
                int32_t *out) {
    if (!out) return fail(PGA_EINVAL, "NULL argument");
    if (P < 1 || N < 2) return fail(PGA_EINVAL, "bad sizes");
    TRY(ensure_device(device));
    HookBufs hb;
    int32_t *d;
    TRY(hb.get(&d, (size_t)P * N));
    TRY(launch_init_raw(seed, N, N, P, P, p_off, (uint32_t)island, nullptr, nullptr, d, 0));
    PGA_CUDA(cudaDeviceSynchronize());
    PGA_CUDA(cudaMemcpy(out, d, sizeof(int32_t) * P * N, cudaMemcpyDeviceToHost));
    return PGA_OK;
}

}  // extern "C"
