// pga_internal.cuh — shared internals of libpga.so (product path).
// Nothing here is shared with oracle/ (independence rule).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pga.h"

namespace pga {

// ---------------------------------------------------------------------------
// Error plumbing: thread-local last error, return codes.
// ---------------------------------------------------------------------------
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);
void count_launch(int n = 1);
// profiling event record; under stream capture it becomes an event-record
// node of the graph (cudaEventRecordExternal), re-targeted per replay
cudaError_t prof_record(cudaEvent_t e, cudaStream_t s);
int check_params(const pga_params *p);       // api.cu: pga_params validation
int check_corr(const double *C, int32_t N);  // api.cu: C finite, unit diagonal, symmetric
int ensure_device(int dev);                  // api.cu: device present, made current

#define PGA_CUDA(call)                                                     \
    do {                                                                   \
        cudaError_t _e = (call);                                           \
        if (_e != cudaSuccess) return ::pga::cuda_fail(_e, #call);         \
    } while (0)

#define PGA_MARK(c, k, s)                                                  \
    do {                                                                   \
        if ((c)->pev && (c)->prof_level >= 2) PGA_CUDA(::pga::prof_record((c)->pev[k], (s))); \
    } while (0)

// Programmatic dependent launch (PDL): kernels of the generation sequence
// are launched with cudaLaunchAttributeProgrammaticStreamSerialization, so a
// kernel's launch and CTA rasterisation overlap the tail of the one before.
// Every such kernel calls pdl_wait() (griddepcontrol.wait: blocks until the
// preceding grid has completed and its memory is visible) before touching
// global memory, then pdl_trigger() (griddepcontrol.launch_dependents) so
// the next kernel may be scheduled.  Both are no-ops when the kernel was
// launched without the attribute.  PGA_PDL=0 in the environment disables
// the attribute (A/B measurement).
bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

#define PGA_LAUNCH_PDL(...)                                                \
    do {                                                                   \
        ::pga::count_launch();                                             \
        cudaError_t _e = ::pga::launch_pdl(__VA_ARGS__);                   \
        if (_e != cudaSuccess) return ::pga::cuda_fail(_e, "kernel launch");\
    } while (0)

#define PGA_LAUNCHED()                                                     \
    do {                                                                   \
        ::pga::count_launch();                                             \
        cudaError_t _e = cudaGetLastError();                               \
        if (_e != cudaSuccess) return ::pga::cuda_fail(_e, "kernel launch");\
    } while (0)

// Philox stream tags (RNG layout).
enum : uint32_t {
    TAG_INIT = 1, TAG_SUS = 2, TAG_PERM = 3, TAG_TOUR = 4, TAG_XO = 5, TAG_MUT = 6, TAG_MUTV = 7
};

constexpr int PROF_EV = 9;     // phase marks per profiled generation
constexpr int CB = 32;         // chromosomes per fitness CTA tile (one per lane)
constexpr int LN_TAB = 128;    // table-driven log: c_j = 1 + (j + 1/2) / 128
constexpr int SPARSE_MAX_N = 2048;   // largest N with a label-sparse pass (cluster cache, pair table)
// rank + selection in one launch (k_rank_sel) for 1024 < P <= RANKC_MAXP
constexpr int64_t RANKC_MAXP = 8192;   // above it the run sort + merge tree is as fast (island-load 4: 0.1755 vs 0.1763 ms)

// Cluster-cache slot (k_fitness_sparse): exact fixed-point c_s of a member
// set keyed by two 64-bit Zobrist words; k1 == 0 empty; chk validates.
struct alignas(32) CCSlot {
    uint64_t k1;
    uint64_t k2;
    long long v;
    uint64_t chk;
};

// Device-resident GA state (one island).  Read/written only by kernels.
struct DevState {
    int32_t gen;          // generation about to be / being evaluated
    int32_t stall;
    int32_t done;
    int32_t reason;
    int32_t best_idx;     // argmax of the last evaluated generation
    int32_t pad0;
    double best;          // best L of the last evaluated generation
    double prev_best;
    double best_ever;
    double mean;
    int32_t pack_error;   // set by k_pack when a label is out of range
    int32_t pad1;
};

struct Migrant;  // layout documented in api.cu

}  // namespace pga

// The context (opaque at the ABI).
namespace pga {
// a captured launch sequence: the executable graph, its template (kept for
// the event-record node handles), the kernel launches it holds, and its
// profiling event-record nodes with their phase-mark index
struct GExec {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t x = nullptr;
    int nk = 0;
    std::vector<std::pair<cudaGraphNode_t, int>> evn;
};
}  // namespace pga

struct pga_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t join_ev = nullptr;   // joins a caller's stream to `stream` (pga_evaluate_device)
    cudaStream_t side = nullptr;     // side branch of a generation (mate slots, launch_mates_fork)
    bool use_prio = false;           // main stream high priority, side stream low (PGA_NO_PRIO=1: off)
    cudaEvent_t fork_ev = nullptr, join_side_ev = nullptr;
    cudaEvent_t fit_ev = nullptr, stats_ev = nullptr;   // statistics on the side stream beside the selection
    pga_params p{};
    int32_t N = 0;
    int32_t ldn = 0;       // padded gene stride of chromosome-major labels / V
    int32_t ldc = 0;       // padded row stride of C
    int64_t P = 0;         // pop_size (island)
    int64_t Pcap = 0;      // capacity rounded up to CB
    // correlation matrix
    double *C = nullptr;
    double *diag = nullptr;
    double *lgtab = nullptr;  // [2 (N+1)]: log n, log(n^2 - n) for the Eq. 8 fold (Q30); then
                              // [2 LN_TAB] {ln c_j, 1 / c_j} of the table-driven log (fast_ln)
    uint8_t *sflag = nullptr; // [Pcap / CB]: block evaluated by the label-sparse pass (f2)
    double sparse_theta = -1.0;   // < 0: automatic (sparse_theta_eff)
    int32_t *sp_live = nullptr;  // device [6]: sparse-pass hysteresis (see k_fitness_sparse)
    // cached graphs of pga_gen_evaluate (plain / migration generation) and
    // pga_gen_breed; dropped whenever a setting that changes the launch
    // sequence does (drop_graphs)
    pga::GExec gx_eval[2];
    pga::GExec gx_breed[2];        // [1]: selection already done in phase A (sel_fresh)
    bool sel_fresh = false;        // the last phase A selected concurrently with its statistics
    unsigned long long *sp_blocks = nullptr;  // device [4]: sparse blocks, gathers, cache hits, pairs saved (profiling)
    pga::CCSlot *cc = nullptr;     // cluster cache table (N <= SPARSE_MAX_N)
    uint32_t cc_mask = 0;          // slots - 1
    uint32_t *cc_state = nullptr;  // device [4]: fill, clear request, CTA count
    uint64_t *cc_keys = nullptr;   // device [N][2] Zobrist keys
    double *ptab = nullptr;        // [N][ldc] Eq. 8 term of each pair cluster (label-sparse pass, N <= SPARSE_MAX_N)
    bool cc_on = true;
    // population: chromosome-major [Pcap][ldn] and gene-major [N][Pcap], double buffered
    uint16_t *pop[2] = {nullptr, nullptr};
    uint16_t *popT[2] = {nullptr, nullptr};
    // fitness scratch/output
    double *V = nullptr;   // [Pcap][ldn] fold inputs C_ii + 2 r'_i
    double *L = nullptr;   // [Pcap]
    uint16_t *top = nullptr;
    // selection scratch
    uint64_t *keys_in = nullptr, *keys_out = nullptr;   // sort keys (double buffer); block sums after the sort
    int32_t *idx_in = nullptr, *order = nullptr;
    int32_t *rank = nullptr;           // rank[i] = position of individual i in order (last merge level)
    int32_t *rc_acc = nullptr;         // k_rank_sel rank accumulators [Pcap] (zero between launches) + CTA counter
    uint64_t *rc_qtab = nullptr;       // k_rank_sel q by rank [Pcap]
    uint64_t *q = nullptr;             // SUS segment widths (index order); the sort's index buffer before
    int32_t *sel = nullptr;
    int32_t *sigma = nullptr;
    uint32_t *breed_ctr = nullptr;     // breed CTA counter (the last CTA advances the generation)
    uint32_t *mmask = nullptr;         // mutation masks of the generation [Pcap][ceil(N/32)] (k_mutmask)
    // state
    pga::DevState *st = nullptr;
    uint16_t *best_labels = nullptr;   // [ldn]
    double *history = nullptr;         // [hist_cap]
    int32_t hist_cap = 0;
    // staging for pga_evaluate / pga_evaluate_device (never the GA buffers)
    int32_t *stage_i32 = nullptr;      // device [Pcap][N]
    uint16_t *evCM = nullptr, *evGM = nullptr;
    double *evL = nullptr;
    // TMA descriptors (sweep) and fold counters
    CUtensorMap tmC{}, tmLab[2]{}, tmLabEv{};
    uint32_t *counters = nullptr;      // [Pcap / CB]
    double *stats_part = nullptr;      // [3 x 1024] k_stats partials
    uint32_t *stats_ctr = nullptr;     // k_stats CTA counter
    // migration scratch
    int64_t mig_bytes = 0;
    // host mirror
    bool has_pop = false;
    bool pending_migration = false;
    int32_t host_gen = 0;              // host-side count of launched generations
    // host copy of the device state (pageable; read after a stream sync)
    pga::DevState *h_st = nullptr;
    // profiling (pga_profile_enable): per generation 4 events
    bool prof = false;
    int prof_level = 0;                 // 1: fitness + generation only, 2: every phase
    std::vector<cudaEvent_t> prof_ev;   // groups of PROF_EV events per generation (see api.cu)
    size_t prof_used = 0;
    cudaEvent_t *pev = nullptr;         // this generation's events while profiling, else null
};

// Label-sparse threshold in effect: the caller's, else automatic: off below
// N = 64 (the dense sweep is cheaper there: C1 0.056 vs 0.058, C2 0.060 vs
// 0.077 ms per generation; round 2's pass wins from C3's N = 100 up: 0.071 vs
// 0.090 ms over 2000 generations), 0.25 with the cluster cache (hits make a
// sparse block cheap up to a quarter of the dense pairs) and 0.04 without it.
inline double sparse_theta_eff(const pga_ctx *c) {
    if (c->sparse_theta >= 0.0) return c->sparse_theta;
    if (c->N < 64) return 0.0;
    return (c->cc && c->cc_on) ? 0.25 : 0.04;
}

namespace pga {

// Launch wrappers implemented in the .cu files (all stream-ordered).
// Population buffers for a fitness launch: kernels pick buffer (*gen & 1)
// when gen != nullptr (GA double buffer), else buffer 0.
struct FitBufs {
    const uint16_t *cm0, *cm1;       // chromosome-major
    const uint16_t *gm0, *gm1;       // gene-major (fold)
    const CUtensorMap *tm0, *tm1;    // gene-major TMA maps (sweep)
    const int32_t *gen;
    const int32_t *done;
};
int make_label_tmap(CUtensorMap *tm, const uint16_t *GM, int N, int64_t Pcap);
int make_c_tmap(CUtensorMap *tm, const double *C, int N, int ldc);
int launch_pack(pga_ctx *c, const uint16_t *lab16, const int32_t *lab32, int64_t P, int ld_in,
                uint16_t *CM, uint16_t *GM, cudaStream_t s);
int prepare_fitness(int N);
int launch_logtab(pga_ctx *c, cudaStream_t s);
int launch_pairtab(pga_ctx *c, cudaStream_t s);   // after launch_logtab
// ev (optional): 3 events recorded before the sweep, between sweep and
// fold, and after the fold.
int launch_fitness(pga_ctx *c, const FitBufs &b, int64_t P, double *L, uint16_t *top,
                   cudaStream_t s, cudaEvent_t *ev = nullptr);
int launch_fitness_range(pga_ctx *c, const FitBufs &b, int64_t begin, int64_t end, double *L,
                         uint16_t *top, cudaStream_t s, cudaEvent_t *ev = nullptr);
int launch_init(pga_ctx *c, uint64_t seed, cudaStream_t s);
int launch_stats(pga_ctx *c, int is_migration_check, cudaStream_t s);
// the library's per-device memory pool (api.cu dalloc); *err != 0 if unavailable
cudaMemPool_t lib_pool(int *err);
// stream-ordered scratch from that pool
inline cudaError_t pool_malloc_async(void **p, size_t bytes, cudaStream_t s) {
    int err = 0;
    cudaMemPool_t pool = lib_pool(&err);
    return err ? cudaMallocAsync(p, bytes, s) : cudaMallocFromPoolAsync(p, bytes, pool, s);
}
int launch_sort_order(pga_ctx *c, cudaStream_t s);
int launch_select(pga_ctx *c, cudaStream_t s);   // order + scaling + selection
int launch_breed(pga_ctx *c, cudaStream_t s, bool late_masks);   // crossover .. replacement + advance
int launch_mutmask(pga_ctx *c, cudaStream_t s);   // the breed's mutation masks (k_mutmask)
bool mutmask_late(const pga_ctx *c);              // masks beside stats + selection (P > 8192)
int launch_export(pga_ctx *c, void *dev_send, cudaStream_t s);
int launch_mates_fork(pga_ctx *c, cudaStream_t s);
int launch_mates_join(pga_ctx *c, cudaStream_t s);
int launch_import(pga_ctx *c, const void *dev_recv, int32_t G, cudaStream_t s);
int launch_canonicalize_i32(int32_t *lab, int64_t P, int32_t N, cudaStream_t s);
int launch_corr(const double *X, int32_t T, int32_t N, double *C, int32_t *status,
                cudaStream_t s);


}  // namespace pga

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------
namespace pgad {

// Device-side bounds checks (the sanitizer substitute: compute-sanitizer is
// closed on the GPU pool).  A build with -DPGA_DEVICE_CHECKS counts every
// violated index/range invariant of the hot kernels in a per-translation-
// unit device counter that pga_debug_violations() sums; the product build
// compiles the checks away.
#ifdef PGA_DEVICE_CHECKS
static __device__ unsigned int g_viol = 0u;
#define PGA_DCHECK(c)                                  \
    do {                                               \
        if (!(c)) atomicAdd(&::pgad::g_viol, 1u);      \
    } while (0)
#define PGA_VIOL_READER(fn)                                                          \
    namespace pga {                                                                  \
    long long fn() {                                                                 \
        unsigned int v = 0;                                                          \
        if (cudaMemcpyFromSymbol(&v, ::pgad::g_viol, sizeof(v)) != cudaSuccess) return -2; \
        return (long long)v;                                                         \
    }                                                                                \
    }
#else
#define PGA_DCHECK(c) \
    do {              \
    } while (0)
#define PGA_VIOL_READER(fn) \
    namespace pga {         \
    long long fn() { return -1; } \
    }
#endif

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Philox4x32-10 (Salmon et al. SC'11), the product's own implementation.
struct U4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                      uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t lo0 = 0xD2511F53u * c0;
        uint32_t hi0 = __umulhi(0xD2511F53u, c0);
        uint32_t lo1 = 0xCD9E8D57u * c2;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return U4{c0, c1, c2, c3};
}

// Philox4x32-10 with the 10 round keys precomputed (rk[2r], rk[2r+1] =
// key + r * (0x9E3779B9, 0xBB67AE85), the same modular sums philox() forms
// round by round).  When rk lives in a kernel's parameter struct the XORs
// take it straight from the constant bank: 4 instead of 6 instructions per
// round in the breed's per-gene mutation draws.
struct RoundKeys {
    uint32_t k[20];
};

inline RoundKeys round_keys(uint64_t seed) {
    RoundKeys r;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int i = 0; i < 10; ++i) {
        r.k[2 * i] = k0;
        r.k[2 * i + 1] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return r;
}

__device__ __forceinline__ U4 philox_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const RoundKeys &rk) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ rk.k[2 * r];
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ rk.k[2 * r + 1];
        c0 = n0;
        c1 = (uint32_t)p1;
        c2 = n2;
        c3 = (uint32_t)p0;
    }
    return U4{c0, c1, c2, c3};
}

__device__ __forceinline__ U4 draw_rk(const RoundKeys &rk, uint32_t tag, uint32_t island, uint32_t gen,
                                      uint32_t c0, uint32_t c1) {
    return philox_rk(c0, c1, gen, tag | (island << 8), rk);
}

// counter = (c0, c1, gen, tag | island << 8), key = (seed_lo, seed_hi)
__device__ __forceinline__ U4 draw(uint64_t seed, uint32_t tag, uint32_t island, uint32_t gen,
                                    uint32_t c0, uint32_t c1) {
    return philox(c0, c1, gen, tag | (island << 8), (uint32_t)seed, (uint32_t)(seed >> 32));
}

__device__ __forceinline__ uint32_t word(const U4 &u, int i) {
    return i == 0 ? u.x : i == 1 ? u.y : i == 2 ? u.z : u.w;
}

__device__ __forceinline__ uint32_t scale_u32(uint32_t x, uint32_t n) {
    return (uint32_t)(((uint64_t)x * (uint64_t)n) >> 32);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Natural log of a positive normal x, table-driven (the label-sparse pass's
// Eq. 8 terms): x = 2^e m, m in [1, 2); c = 1 + (j + 1/2)/128 for the top 7
// mantissa bits j; r = m (1/c) - 1 (one rounding, |r| < 2^-8);
// ln x = e ln 2 + ln c + log1p(r), log1p by its degree-7 Taylor polynomial
// (truncation < r^8/8 < 7e-21).  tab[2j] = ln c (libm), tab[2j+1] = 1/c.
// Absolute error ~2e-16 (a few ulp of the result), 17 instructions instead
// of the library's ~45; pinned against libm by tests/test_gpu_checks.py.
__device__ __forceinline__ double fast_ln(double x, const double2 *__restrict__ tab) {
    const long long b = __double_as_longlong(x);
    const int e = (int)(b >> 52) - 1023;
    const int j = (int)((b >> 45) & (pga::LN_TAB - 1));
    const double m = __longlong_as_double((b & 0x000FFFFFFFFFFFFFll) | 0x3FF0000000000000ll);
    const double2 t = __ldg(tab + j);
    const double r = fma(m, t.y, -1.0);
    double p = fma(r, 1.0 / 7.0, -1.0 / 6.0);
    p = fma(p, r, 1.0 / 5.0);
    p = fma(p, r, -1.0 / 4.0);
    p = fma(p, r, 1.0 / 3.0);
    p = fma(p, r, -1.0 / 2.0);
    p = fma(p, r, 1.0);
    const double lnm = fma(p, r, t.x);
    return fma((double)e, 0.69314718055994530942, fma((double)e, 2.3190468138462996e-17, lnm));
}

// Summand of Eq. 8 for one cluster with readings Q2/Q3.
__device__ __forceinline__ double cluster_term(int n_s, double c_s) {
    const double n = (double)n_s;
    if (n_s < 2 || !(c_s > n)) return 0.0;
    const double n2 = n * n;
    const double ch = fmin(c_s, n2 - 1e-9);
    return log(n / ch) + (n - 1.0) * log((n2 - n) / (n2 - ch));
}


__device__ __forceinline__ int ceil_log2_d(int64_t x) {
    int b = 0;
    while (((int64_t)1 << b) < x) ++b;
    return b;
}

// Mate slot m of M (Q10): keyed 4-round Feistel permutation on h+h bits
// (2^(2h) >= M), round function Philox(PERM; R, round)[0], cycle-walked
// back into [0, M).
__device__ __forceinline__ int32_t feistel_slot(int64_t m, int64_t M, uint64_t seed, uint32_t gen,
                                                uint32_t island) {
    int h = (ceil_log2_d(M) + 1) / 2;
    if (h < 1) h = 1;
    const uint32_t mask = (1u << h) - 1u;
    uint32_t x = (uint32_t)m;
    do {
        uint32_t Lh = x >> h, R = x & mask;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const U4 f = draw(seed, pga::TAG_PERM, island, gen, R, (uint32_t)r);
            const uint32_t t = R;
            R = Lh ^ (f.x & mask);
            Lh = t;
        }
        x = (Lh << h) | R;
    } while (x >= (uint32_t)M);
    return (int32_t)x;
}

}  // namespace pgad
