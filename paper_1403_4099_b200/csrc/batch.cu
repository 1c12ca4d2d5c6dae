// batch.cu — batched GA: one independent GA per
// correlation matrix, all of them in ONE launch.  This is the shape of the
// paper's own test workload: 1760 matrices of 18 stocks, each clustered by
// its own PGA run with the Table 3 configuration (timings
// in Table 4).
//
// One CTA owns one matrix for the whole run.  C, both populations (u8
// labels), L, top and the selection state stay in shared memory; HBM sees C
// once and the results once.  Per generation (Alg. 1, with the
// operators of DESIGN.md §3, exactly as the per-generation kernels of
// fitness.cu / ga.cu compute them for a single island):
//   evaluate   warp per chromosome, lane = gene (N <= 32): n_s by
//              __match_any_sync/popc; V_i = sum_{j in s_i} C_ij over the
//              group's set bits; the group leader sums V over its group
//              (c_s, Eq. 6) and takes the Eq. 8 summand; warp reductions give
//              L and the KB top label.
//   statistics warp 0: best (first max), best-ever labels, stall, stop.
//   order      bitonic sort of (~bits(L), index) in shared memory; ranks.
//   selection  RANK scaling + exact u64 SUS prefix (block scan) or tournament.
//   mates      Feistel slots, thread per slot.
//   breed      thread per offspring slot: elites, KB / one-point crossover,
//              mutation (one Philox block per 4 genes), first-occurrence
//              canonicalisation through a per-thread table.
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "pga_internal.cuh"

namespace {

using namespace pgad;

constexpr int BT = 256, BNW = BT / 32;   // threads per CTA (one CTA per matrix)
constexpr int BMAX_N = 32, BMAX_P = 2048;
// C row stride in shared memory: 32 doubles, so C[j][lane] sits in bank pair
// lane mod 16 whatever row j a lane's cluster walk is on -- the lanes of
// different clusters (different j) no longer collide (round 1: 33% of the
// kernel's shared wavefronts were bank-conflict excess, profiles/r01l_full.md)
constexpr int BLDC = 32;
constexpr int TAB = 36;                  // per-thread canonicalisation table (labels 0..N)
constexpr int EB = 8;                    // chromosomes per warp per evaluation batch

enum { MODE_RUN = 0, MODE_EVAL = 1, MODE_STEP = 2 };

// Shared-memory layout of one CTA.  The L array doubles as the SUS prefix
// (u64) once the weights are formed and as the per-thread canonicalisation
// tables during init and breed (L is dead then).
struct BLayout {
    int ldb, n2, qcap;
    size_t oL, oC, oVal, oRank, oSel, oSig, oTop, oPop0, oPop1, oV, oQf, oQn, oQl, oQs, oLg, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline BLayout b_layout(int N, int P, int M) {
    BLayout l;
    l.ldb = (N + 3) & ~3;
    int n2 = 2;
    while (n2 < P) n2 <<= 1;
    l.n2 = n2;
    l.qcap = EB * (N / 2 > 0 ? N / 2 : 1);   // clusters with n_s >= 2 per chromosome <= N/2
    l.oL = 0;
    size_t o = al16((size_t)8 * P);
    if (o < (size_t)BT * TAB) o = al16((size_t)BT * TAB);
    l.oC = o;     o += al16((size_t)8 * N * BLDC);   // rows padded to BLDC doubles (conflict-free, see b_evaluate)
    l.oVal = o;   o += al16((size_t)4 * n2);
    l.oRank = o;  o += al16((size_t)2 * P);
    l.oSel = o;   o += al16((size_t)2 * M);
    l.oSig = o;   o += al16((size_t)2 * M);
    l.oTop = o;   o += al16((size_t)P);
    l.oPop0 = o;  o += al16((size_t)P * l.ldb);
    l.oPop1 = o;  o += al16((size_t)P * l.ldb);
    l.oV = o;     o += (size_t)8 * 32 * BNW;
    l.oQf = o;    o += al16((size_t)8 * l.qcap * BNW);
    l.oQn = o;    o += al16((size_t)l.qcap * BNW);
    l.oQl = o;    o += al16((size_t)l.qcap * BNW);
    l.oQs = o;    o += al16((size_t)2 * (EB + 1) * BNW);
    l.oLg = o;    o += (size_t)8 * 2 * (BMAX_N + 1);
    l.total = o;
    return l;
}

struct BArgs {
    const double *C;                     // [B][N][N]
    int B, N, P, E, M;
    int selection, tour_k, scaling, stall_gens, max_gens;
    double tol;
    uint64_t thr_c, thr_m, thr_kb;
    uint64_t seed;
    int mode;
    // MODE_RUN outputs (device)
    int32_t *best_labels;                // [B][N] 1-based
    double *best_L;                      // [B]
    int32_t *gens, *reason;              // [B]
    double *history;                     // [B][max_gens]
    // hooks (device, 0-based labels)
    const int32_t *in_pop;               // [B][P][N]
    const double *in_L;                  // [B][P]
    const int32_t *in_top;               // [B][P]
    int32_t hook_gen;
    int32_t *out_pop;                    // [B][P][N]
    double *out_L;                       // [B][P]
    int32_t *out_top;                    // [B][P]
    BLayout ly;                          // shared-memory layout (host-computed)
};

struct BSmem {
    double *L, *C, *V, *qf, *lgn, *lgnn;
    uint64_t *prefix;
    uint32_t *val;
    int16_t *rank, *sel, *sig;
    uint16_t *qs;
    uint8_t *top, *pop[2], *tabs, *qn, *ql;
    int qcap;
};

__device__ __forceinline__ BSmem b_smem(unsigned char *sm, const BLayout &ly) {
    BSmem s;
    s.L = reinterpret_cast<double *>(sm + ly.oL);
    s.prefix = reinterpret_cast<uint64_t *>(sm + ly.oL);
    s.C = reinterpret_cast<double *>(sm + ly.oC);
    s.val = reinterpret_cast<uint32_t *>(sm + ly.oVal);
    s.rank = reinterpret_cast<int16_t *>(sm + ly.oRank);
    s.sel = reinterpret_cast<int16_t *>(sm + ly.oSel);
    s.sig = reinterpret_cast<int16_t *>(sm + ly.oSig);
    s.top = sm + ly.oTop;
    s.pop[0] = sm + ly.oPop0;
    s.pop[1] = sm + ly.oPop1;
    s.V = reinterpret_cast<double *>(sm + ly.oV);
    s.tabs = sm + ly.oL;
    s.qf = reinterpret_cast<double *>(sm + ly.oQf);
    s.qn = sm + ly.oQn;
    s.ql = sm + ly.oQl;
    s.qs = reinterpret_cast<uint16_t *>(sm + ly.oQs);
    s.qcap = ly.qcap;
    s.lgn = reinterpret_cast<double *>(sm + ly.oLg);
    s.lgnn = s.lgn + (BMAX_N + 1);
    return s;
}

// First-occurrence canonicalisation of one chromosome, streamed gene by gene
// through the calling thread's table (Q7).
struct TCanon {
    uint8_t *tab;
    int next;
    __device__ __forceinline__ void reset(int n) {
        for (int t = 0; t <= n; ++t) tab[t] = 0xFF;
        next = 0;
    }
    __device__ __forceinline__ uint32_t map(uint32_t s) {
        uint32_t t = tab[s];
        if (t == 0xFF) {
            t = (uint32_t)next++;
            tab[s] = (uint8_t)t;
        }
        return t;
    }
};

// Initial population (Q8): gene i of chromosome p is
// scale(Philox(INIT; i>>2, p)[i&3], N) with generation field 0xFFFFFFFF.
__device__ __forceinline__ void b_init(const BArgs &a, const BSmem &s, int ldb, uint64_t seed) {
    TCanon cn{s.tabs + threadIdx.x * TAB, 0};
    for (int p = threadIdx.x; p < a.P; p += BT) {
        uint8_t *dst = s.pop[0] + (size_t)p * ldb;
        cn.reset(a.N);
        for (int i0 = 0; i0 < a.N; i0 += 4) {
            const U4 u = draw(seed, pga::TAG_INIT, 0u, 0xFFFFFFFFu, (uint32_t)(i0 >> 2), (uint32_t)p);
            for (int q = 0; q < 4 && i0 + q < a.N; ++q)
                dst[i0 + q] = (uint8_t)cn.map(scale_u32(word(u, q), (uint32_t)a.N));
        }
    }
}

// Eq. 5/6/8 for every chromosome of `pop`: warp per chromosome, lane = gene,
// EB chromosomes per batch.  n_s by __match_any_sync/popc; V_i = sum of C_ji
// over i's group (set bits, ascending j); each group leader sums V over its
// group (c_s, Eq. 6).  Clusters with n_s >= 2 and c_s > n_s (the only
// non-zero summands, Q2) are queued; the Eq. 8 summands of the whole batch
// are then taken lane-parallel, and lane e adds chromosome e's summands in
// queue (= label, for canonical labels) order.
__device__ __forceinline__ void b_evaluate(const BSmem &s, const uint8_t *pop, int N, int P, int ldb) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *Vw = s.V + warp * 32;
    double *qf = s.qf + warp * s.qcap;
    uint8_t *qn = s.qn + warp * s.qcap, *ql = s.ql + warp * s.qcap;
    uint16_t *qs = s.qs + warp * (EB + 1);
    const bool valid = lane < N;
    for (int p0 = warp * EB; p0 < P; p0 += BNW * EB) {
        const int ne = min(EB, P - p0);
        int cnt = 0;
        for (int e = 0; e < ne; ++e) {
            const uint32_t lab = valid ? (uint32_t)pop[(size_t)(p0 + e) * ldb + lane] : 0x100u + (uint32_t)lane;
            const unsigned m = __match_any_sync(0xFFFFFFFFu, lab);
            double V = 0.0;                         // V_i = sum_{j in s_i} C_ji (ascending j)
            if (valid)
                for (unsigned mm = m; mm; mm &= mm - 1) V += s.C[(__ffs(mm) - 1) * BLDC + lane];
            Vw[lane] = V;
            __syncwarp();
            const int n = __popc(m);
            double c = 0.0;
            bool push = false;
            if (valid && n >= 2 && (__ffs(m) - 1) == lane) {
                for (unsigned mm = m; mm; mm &= mm - 1) c += Vw[__ffs(mm) - 1];
                push = c > (double)n;
            }
            const unsigned bal = __ballot_sync(0xFFFFFFFFu, push);
            if (push) {
                const int pos = cnt + __popc(bal & lanemask_lt());
                qf[pos] = c;
                qn[pos] = (uint8_t)n;
                ql[pos] = (uint8_t)lab;
            }
            if (lane == 0) qs[e] = (uint16_t)cnt;
            cnt += __popc(bal);
            __syncwarp();
        }
        if (lane == 0) qs[ne] = (uint16_t)cnt;
        __syncwarp();
        // Eq. 8 summands (every queued cluster has n_s >= 2 and c_s > n_s):
        // log(n/c) + (n-1) log((n^2-n)/(n^2-c)) taken as
        // (log n - log c) + (n-1) (log(n^2-n) - log(n^2-c)) with the integer
        // logs from the per-CTA table; c clamped to n^2 - 1e-9 (Q3)
        for (int k = lane; k < cnt; k += 32) {
            const int n = qn[k];
            const double nd = (double)n, n2 = nd * nd;
            const double ch = fmin(qf[k], n2 - 1e-9);
            qf[k] = (s.lgn[n] - log(ch)) + (nd - 1.0) * (s.lgnn[n] - log(n2 - ch));
        }
        __syncwarp();
        if (lane < ne) {
            double sum = 0.0, bf = 0.0;
            int bt = -1;
            for (int k = qs[lane]; k < qs[lane + 1]; ++k) {
                const double f = qf[k];
                sum += f;
                if (f > bf || (f == bf && f > 0.0 && (int)ql[k] < bt)) {   // KB top: largest, smallest label
                    bf = f;
                    bt = ql[k];
                }
            }
            s.L[p0 + lane] = 0.5 * sum;
            s.top[p0 + lane] = bt < 0 ? (uint8_t)0xFF : (uint8_t)bt;
        }
        __syncwarp();
    }
}

// (L desc, index asc): does item (La, a) come before (Lb, b)?  Padding items
// carry L = -1 < every L and index 0xFFFFFFFF.
__device__ __forceinline__ bool before(double La, uint32_t a, double Lb, uint32_t b) {
    return La > Lb || (La == Lb && a < b);
}

// Isolate fittest: order by (L desc, index asc) -> val[0..P); ranks.
// Bitonic network over indices, comparing L directly.
__device__ __forceinline__ void b_order(const BSmem &s, int P, int n2) {
    const int tid = threadIdx.x;
    for (int t = tid; t < n2; t += BT) s.val[t] = t < P ? (uint32_t)t : 0xFFFFFFFFu;
    __syncthreads();
    for (int size = 2; size <= n2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = tid; t < (n2 >> 1); t += BT) {
                const int i = 2 * t - (t & (stride - 1)), j = i + stride;
                const bool up = (i & size) == 0;
                const uint32_t vi = s.val[i], vj = s.val[j];
                const double Li = vi < (uint32_t)P ? s.L[vi] : -1.0;
                const double Lj = vj < (uint32_t)P ? s.L[vj] : -1.0;
                if (before(Lj, vj, Li, vi) == up) {
                    s.val[i] = vj;
                    s.val[j] = vi;
                }
            }
            __syncthreads();
        }
    for (int r = tid; r < P; r += BT) s.rank[s.val[r]] = (int16_t)(r + 1);
    __syncthreads();
}

// Scaling + selection (Q9, Q10) and mate slots -> sel[M], sig[M].
__device__ __forceinline__ void b_select(const BArgs &a, const BSmem &s, uint64_t seed, uint32_t gen) {
    __shared__ uint64_t wsum[BNW];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int P = a.P, M = a.M;
    if (a.selection == PGA_SEL_TOURNAMENT) {
        for (int m = tid; m < M; m += BT) {
            const U4 u = draw(seed, pga::TAG_TOUR, 0u, gen, (uint32_t)m, 0u);
            int best = (int)scale_u32(u.x, (uint32_t)P);
            for (int t = 1; t < a.tour_k; ++t) {
                const int c = (int)scale_u32(word(u, t), (uint32_t)P);
                if (s.L[c] > s.L[best] || (s.L[c] == s.L[best] && c < best)) best = c;
            }
            s.sel[m] = (int16_t)best;
        }
    } else {
        const double wmax = (a.scaling == PGA_SCALE_RANK) ? 1.0 : s.L[s.val[0]];
        if (!(wmax > 0.0)) {   // all-zero fitness: uniform fallback
            for (int m = tid; m < M; m += BT) {
                const U4 u = draw(seed, pga::TAG_SUS, 0u, gen, (uint32_t)m, 0u);
                s.sel[m] = (int16_t)scale_u32(u.x, (uint32_t)P);
            }
        } else {
            const int B = 62 - ceil_log2_d(P);
            const int ipt = (P + BT - 1) / BT;   // <= BMAX_P / BT = 8
            uint64_t q[BMAX_P / BT], run = 0;
#pragma unroll
            for (int k = 0; k < BMAX_P / BT; ++k) {
                const int i = ipt * tid + k;
                uint64_t qi = 0;
                if (k < ipt && i < P) {
                    const double w = (a.scaling == PGA_SCALE_RANK) ? 1.0 / sqrt((double)s.rank[i]) : s.L[i];
                    const double x = w / wmax;
                    if (x > 0.0) qi = (uint64_t)floor(ldexp(x, B));
                }
                run += qi;
                q[k] = run;
            }
            uint64_t incl = run;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, incl, off);
                if (lane >= off) incl += o;
            }
            if (lane == 31) wsum[wid] = incl;
            __syncthreads();
            if (wid == 0) {
                uint64_t v = lane < BNW ? wsum[lane] : 0ull;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, v, off);
                    if (lane >= off) v += o;
                }
                if (lane < BNW) wsum[lane] = v;
            }
            __syncthreads();
            const uint64_t base = (incl - run) + (wid ? wsum[wid - 1] : 0ull);
            // every L read of this phase happened before the barrier above:
            // the prefix may overwrite L
#pragma unroll
            for (int k = 0; k < BMAX_P / BT; ++k) {
                const int i = ipt * tid + k;
                if (k < ipt && i < P) s.prefix[i] = base + q[k];   // inclusive prefix (index order)
            }
            __syncthreads();
            const uint64_t Q = s.prefix[P - 1];
            const uint64_t step = Q / (uint64_t)M;
            const U4 u = draw(seed, pga::TAG_SUS, 0u, gen, 0u, 0xFFFFFFFFu);
            const uint64_t x = ((uint64_t)u.x << 32) | (uint64_t)u.y;
            const uint64_t start = __umul64hi(x, step);
            for (int m = tid; m < M; m += BT) {
                const uint64_t ptr = start + (uint64_t)m * step;
                int lo = 0, hi = P - 1;   // min{i : prefix_i > ptr}
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (s.prefix[mid] > ptr) hi = mid;
                    else lo = mid + 1;
                }
                s.sel[m] = (int16_t)lo;
            }
        }
    }
    for (int m = tid; m < M; m += BT) s.sig[m] = (int16_t)feistel_slot(m, M, seed, gen, 0u);
    __syncthreads();
}

// Elitism, crossover, mutation, canonicalisation, replacement (
// Q11-Q15): thread per offspring slot o.
__device__ __forceinline__ void b_breed(const BArgs &a, const BSmem &s, const uint8_t *cur, uint8_t *nxt, int ldb,
                        uint64_t seed, uint32_t gen) {
    const int N = a.N, E = a.E;
    TCanon cn{s.tabs + threadIdx.x * TAB, 0};
    for (int o = threadIdx.x; o < a.P; o += BT) {
        uint8_t *dst = nxt + (size_t)o * ldb;
        if (o < E) {
            const uint32_t *src = reinterpret_cast<const uint32_t *>(cur + (size_t)s.val[o] * ldb);
            for (int w = 0; w < (ldb >> 2); ++w) reinterpret_cast<uint32_t *>(dst)[w] = src[w];
            continue;
        }
        const int k = (o - E) >> 1, child = (o - E) & 1;
        const int ia = s.sel[s.sig[2 * k]], ib = s.sel[s.sig[2 * k + 1]];
        const int pa = child ? ib : ia, pb = child ? ia : ib;
        const U4 x = draw(seed, pga::TAG_XO, 0u, gen, (uint32_t)k, 0u);
        int mode = 0, cut = N, kbt = -1;
        if ((uint64_t)x.x >= a.thr_c) {
            mode = 0;
        } else if ((uint64_t)x.y < a.thr_kb) {
            mode = 1;
            kbt = s.top[pb] == 0xFF ? -1 : (int)s.top[pb];
        } else {
            mode = 2;
            cut = 1 + (int)scale_u32(x.z, (uint32_t)(N - 1));
        }
        const uint8_t *ga = cur + (size_t)pa * ldb, *gb = cur + (size_t)pb * ldb;
        cn.reset(N);
        for (int i0 = 0; i0 < N; i0 += 4) {
            uint32_t mb = 0;
            U4 v{0u, 0u, 0u, 0u};
            if (a.thr_m) {
                const U4 u = draw(seed, pga::TAG_MUT, 0u, gen, (uint32_t)(i0 >> 2), (uint32_t)o);
                mb = ((uint64_t)u.x < a.thr_m ? 1u : 0u) | ((uint64_t)u.y < a.thr_m ? 2u : 0u) |
                     ((uint64_t)u.z < a.thr_m ? 4u : 0u) | ((uint64_t)u.w < a.thr_m ? 8u : 0u);
                if (mb) v = draw(seed, pga::TAG_MUTV, 0u, gen, (uint32_t)(i0 >> 2), (uint32_t)o);
            }
            const uint32_t wa = *reinterpret_cast<const uint32_t *>(ga + i0);
            const uint32_t wb = *reinterpret_cast<const uint32_t *>(gb + i0);
            uint32_t out = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i = i0 + q;
                uint32_t g = (wa >> (8 * q)) & 0xFFu;
                const uint32_t h = (wb >> (8 * q)) & 0xFFu;
                if (mode == 1) {
                    if (kbt >= 0 && (int)h == kbt) g = (uint32_t)N;
                } else if (mode == 2) {
                    if (i >= cut) g = h;
                }
                if ((mb >> q) & 1u) g = scale_u32(word(v, q), (uint32_t)N);
                if (i < N) out |= cn.map(g) << (8 * q);
            }
            *reinterpret_cast<uint32_t *>(dst + i0) = out;   // ldb is a multiple of 4
        }
    }
}

__global__ void __launch_bounds__(BT, 3) k_batch(BArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double s_best_ever, s_prev;
    __shared__ int s_stall, s_reason, s_stop, s_improved, s_bi;
    __shared__ uint8_t s_best[BMAX_N];
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = a.N, P = a.P;
    const BLayout &ly = a.ly;
    const BSmem s = b_smem(sm, ly);
    for (int t = tid; t <= BMAX_N; t += BT) {    // integer logs of Eq. 8
        s.lgn[t] = t >= 1 ? log((double)t) : 0.0;
        s.lgnn[t] = t >= 2 ? log((double)t * t - t) : 0.0;
    }
    const int ldb = ly.ldb;
    const uint64_t seed = a.seed + (uint64_t)b;

    if (a.mode != MODE_STEP)
        for (int t = tid; t < N * N; t += BT) s.C[(t / N) * BLDC + t % N] = a.C[(size_t)b * N * N + t];
    if (a.mode == MODE_RUN) {
        b_init(a, s, ldb, seed);
    } else {
        for (int t = tid; t < P * ldb; t += BT) {
            const int p = t / ldb, i = t - p * ldb;
            s.pop[0][t] = i < N ? (uint8_t)a.in_pop[((size_t)b * P + p) * N + i] : (uint8_t)0;
        }
        if (a.mode == MODE_STEP)
            for (int p = tid; p < P; p += BT) {
                s.L[p] = a.in_L[(size_t)b * P + p];
                const int32_t t = a.in_top[(size_t)b * P + p];
                s.top[p] = t < 0 ? (uint8_t)0xFF : (uint8_t)t;
            }
    }
    __syncthreads();
    if (a.mode == MODE_EVAL) {
        b_evaluate(s, s.pop[0], N, P, ldb);
        __syncthreads();
        for (int p = tid; p < P; p += BT) {
            a.out_L[(size_t)b * P + p] = s.L[p];
            a.out_top[(size_t)b * P + p] = s.top[p] == 0xFF ? -1 : (int32_t)s.top[p];
        }
        return;
    }
    if (a.mode == MODE_STEP) {
        const uint32_t gen = (uint32_t)a.hook_gen;
        b_order(s, P, ly.n2);
        b_select(a, s, seed, gen);
        b_breed(a, s, s.pop[0], s.pop[1], ldb, seed, gen);
        __syncthreads();
        for (int t = tid; t < P * N; t += BT) {
            const int p = t / N, i = t - p * N;
            a.out_pop[(size_t)b * P * N + t] = (int32_t)s.pop[1][(size_t)p * ldb + i];
        }
        return;
    }
    if (tid == 0) {
        s_best_ever = -1.0;
        s_prev = 0.0;
        s_stall = 0;
        s_reason = PGA_REASON_MAX_GENS;
    }
    int g = 0;
    for (;; ++g) {
        uint8_t *cur = (g & 1) ? s.pop[1] : s.pop[0];   // select, not an indexed (local) array
        uint8_t *nxt = (g & 1) ? s.pop[0] : s.pop[1];
        b_evaluate(s, cur, N, P, ldb);
        __syncthreads();
        // statistics / termination (Alg. 1; Q16, Q17), warp 0
        if (warp == 0) {
            double best = -1.0;
            int bi = 0x7FFFFFFF;
            for (int i = lane; i < P; i += 32)
                if (s.L[i] > best) {
                    best = s.L[i];
                    bi = i;
                }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ob = __shfl_xor_sync(0xFFFFFFFFu, best, off);
                const int oi = __shfl_xor_sync(0xFFFFFFFFu, bi, off);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            if (lane == 0) {
                if (a.history) a.history[(size_t)b * a.max_gens + g] = best;
                const int improved = best > s_best_ever;
                if (improved) s_best_ever = best;
                if (g > 0) s_stall = (best - s_prev < a.tol) ? s_stall + 1 : 0;
                s_prev = best;
                int stop = 0;
                if (a.tol >= 0.0 && s_stall >= a.stall_gens) {
                    stop = 1;
                    s_reason = PGA_REASON_STALLED;
                }
                if (g + 1 >= a.max_gens) stop = 1;
                s_stop = stop;
                s_improved = improved;
                s_bi = bi;
            }
            __syncwarp();
            if (s_improved && lane < N) s_best[lane] = cur[(size_t)s_bi * ldb + lane];
        }
        __syncthreads();
        if (s_stop) break;
        b_order(s, P, ly.n2);
        b_select(a, s, seed, (uint32_t)g);
        b_breed(a, s, cur, nxt, ldb, seed, (uint32_t)g);
        __syncthreads();
    }
    if (tid < N && a.best_labels) a.best_labels[(size_t)b * N + tid] = (int32_t)s_best[tid] + 1;
    if (tid == 0) {
        a.best_L[b] = s_best_ever;
        if (a.gens) a.gens[b] = g + 1;
        if (a.reason) a.reason[b] = s_reason;
    }
}

uint64_t threshold(double p) {   // Q13: event iff u32 < llround(p * 2^32)
    if (p >= 1.0) return (uint64_t)1 << 32;
    if (p <= 0.0) return 0;
    return (uint64_t)llround(p * 4294967296.0);
}

int fill_args(BArgs &a, int32_t B, int32_t N, const pga_params *p, int device, size_t *smem) {
    if (B < 1 || B > (1 << 20)) return pga::fail(PGA_EINVAL, "B must be in [1, 2^20]");
    if (N < 2 || N > BMAX_N) return pga::fail(PGA_EINVAL, "batched GA needs 2 <= N <= 32");
    if (p) {
        int rc = pga::check_params(p);
        if (rc) return rc;
        if (p->pop_size > BMAX_P) return pga::fail(PGA_EINVAL, "batched GA needs pop_size <= 2048");
        if (p->n_islands != 1) return pga::fail(PGA_EINVAL, "batched GA runs one island per matrix (n_islands = 1)");
    }
    std::memset(&a, 0, sizeof(a));
    a.B = B;
    a.N = N;
    if (p) {
        a.P = p->pop_size;
        a.E = p->elite;
        a.M = 2 * ((a.P - a.E + 1) / 2);
        a.selection = p->selection;
        a.tour_k = p->tournament_k;
        a.scaling = p->scaling;
        a.stall_gens = p->stall_gens;
        a.max_gens = p->max_gens;
        a.tol = p->tol;
        a.thr_c = threshold(p->p_crossover);
        a.thr_m = threshold(p->p_mutation);
        a.thr_kb = threshold(p->p_kb);
        a.seed = p->seed;
    }
    a.ly = b_layout(N, a.P, a.M);
    *smem = a.ly.total;
    (void)device;
    return PGA_OK;
}

int check_smem(size_t smem, int device) {
    int optin = 0;
    PGA_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    // static shared memory of k_batch: a few hundred bytes
    if (smem + 1024 > (size_t)optin)
        return pga::fail(PGA_EINVAL, "batched GA: pop_size x N does not fit one CTA's shared memory (" +
                                         std::to_string(smem) + " B)");
    return PGA_OK;
}

int launch_batch(const BArgs &a, size_t smem, cudaStream_t st) {
    PGA_CUDA(cudaFuncSetAttribute(k_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_batch<<<a.B, BT, smem, st>>>(a);
    PGA_LAUNCHED();
    return PGA_OK;
}

struct DBufs {
    std::vector<void *> ptrs;
    ~DBufs() {
        for (void *p : ptrs) cudaFree(p);
    }
    template <typename T>
    int get(T **p, size_t n) {
        cudaError_t e = cudaMalloc((void **)p, sizeof(T) * (n ? n : 1));
        if (e != cudaSuccess) return pga::fail(PGA_ENOMEM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
        ptrs.push_back((void *)*p);
        return PGA_OK;
    }
};

#define BTRY(x)              \
    do {                     \
        int _rc = (x);       \
        if (_rc) return _rc; \
    } while (0)

}  // namespace

extern "C" {

int pga_batch_smem_bytes(int32_t N, int32_t pop_size, int32_t elite, int32_t device, int64_t *bytes) {
    if (!bytes) return pga::fail(PGA_EINVAL, "bytes is NULL");
    if (N < 2 || N > BMAX_N) return pga::fail(PGA_EINVAL, "batched GA needs 2 <= N <= 32");
    if (pop_size < 2 || pop_size > BMAX_P || elite < 0 || elite >= pop_size)
        return pga::fail(PGA_EINVAL, "need 2 <= pop_size <= 2048 and 0 <= elite < pop_size");
    const int M = 2 * ((pop_size - elite + 1) / 2);
    *bytes = (int64_t)b_layout(N, pop_size, M).total;
    BTRY(pga::ensure_device(device));
    return check_smem((size_t)*bytes, device);
}

int pga_batch_run(const double *C, int32_t B, int32_t N, const pga_params *p, int32_t on_device,
                  int32_t *best_labels, double *best_L, int32_t *gens, int32_t *reason, double *history,
                  void *stream) {
    if (!C || !best_L || !p) return pga::fail(PGA_EINVAL, "NULL argument (C, best_L and params are required)");
    BArgs a;
    size_t smem = 0;
    BTRY(fill_args(a, B, N, p, p->device, &smem));
    if (!on_device)
        for (int32_t b = 0; b < B; ++b) {
            int rc = pga::check_corr(C + (size_t)b * N * N, N);
            if (rc) return pga::fail(rc, "matrix " + std::to_string(b) + ": " + pga_last_error());
        }
    BTRY(pga::ensure_device(p->device));
    BTRY(check_smem(smem, p->device));
    a.mode = MODE_RUN;
    if (on_device) {
        a.C = C;
        a.best_labels = best_labels;
        a.best_L = best_L;
        a.gens = gens;
        a.reason = reason;
        a.history = history;
        return launch_batch(a, smem, (cudaStream_t)stream);
    }
    // host path: one stream, stream-ordered scratch (no device-wide syncs)
    cudaStream_t st;
    PGA_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    } guard{st};
    const size_t nC = (size_t)B * N * N, nH = history ? (size_t)B * p->max_gens : 0;
    unsigned char *blob = nullptr;
    const size_t bytes = sizeof(double) * (nC + B + nH) + sizeof(int32_t) * ((size_t)B * N + 2 * (size_t)B) + 64;
    PGA_CUDA(pga::pool_malloc_async((void **)&blob, bytes, st));
    struct BlobGuard {
        void *p;
        cudaStream_t s;
        ~BlobGuard() { cudaFreeAsync(p, s); }
    } bg{blob, st};
    double *dC = reinterpret_cast<double *>(blob);
    double *dL = dC + nC;
    double *dH = history ? dL + B : nullptr;
    int32_t *dlab = reinterpret_cast<int32_t *>(dL + B + nH);
    int32_t *dg = dlab + (size_t)B * N;
    int32_t *dr = dg + B;
    if (history) PGA_CUDA(cudaMemsetAsync(dH, 0, sizeof(double) * nH, st));
    PGA_CUDA(cudaMemcpyAsync(dC, C, sizeof(double) * nC, cudaMemcpyHostToDevice, st));
    a.C = dC;
    a.best_labels = dlab;
    a.best_L = dL;
    a.gens = dg;
    a.reason = dr;
    a.history = dH;
    BTRY(launch_batch(a, smem, st));
    PGA_CUDA(cudaMemcpyAsync(best_L, dL, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    if (best_labels) PGA_CUDA(cudaMemcpyAsync(best_labels, dlab, sizeof(int32_t) * (size_t)B * N, cudaMemcpyDeviceToHost, st));
    if (gens) PGA_CUDA(cudaMemcpyAsync(gens, dg, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, st));
    if (reason) PGA_CUDA(cudaMemcpyAsync(reason, dr, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, st));
    if (history) PGA_CUDA(cudaMemcpyAsync(history, dH, sizeof(double) * nH, cudaMemcpyDeviceToHost, st));
    PGA_CUDA(cudaStreamSynchronize(st));
    return PGA_OK;
}

int pga_batch_op_evaluate(const double *C, int32_t B, int32_t N, const int32_t *labels, int32_t P,
                          int32_t device, double *L, int32_t *top) {
    if (!C || !labels || !L || !top) return pga::fail(PGA_EINVAL, "NULL argument");
    if (P < 1 || P > BMAX_P) return pga::fail(PGA_EINVAL, "need 1 <= P <= 2048");
    BArgs a;
    size_t smem = 0;
    BTRY(fill_args(a, B, N, nullptr, device, &smem));
    a.P = P;
    a.M = 0;
    a.ly = b_layout(N, P, 0);
    smem = a.ly.total;
    for (size_t k = 0; k < (size_t)B * P * N; ++k)
        if (labels[k] < 0 || labels[k] > 2 * N) return pga::fail(PGA_EINVAL, "labels must lie in 0..2N");
    BTRY(pga::ensure_device(device));
    BTRY(check_smem(smem, device));
    DBufs d;
    double *dC, *dL;
    int32_t *dlab, *dtop;
    BTRY(d.get(&dC, (size_t)B * N * N));
    BTRY(d.get(&dlab, (size_t)B * P * N));
    BTRY(d.get(&dL, (size_t)B * P));
    BTRY(d.get(&dtop, (size_t)B * P));
    PGA_CUDA(cudaMemcpy(dC, C, sizeof(double) * (size_t)B * N * N, cudaMemcpyHostToDevice));
    PGA_CUDA(cudaMemcpy(dlab, labels, sizeof(int32_t) * (size_t)B * P * N, cudaMemcpyHostToDevice));
    a.mode = MODE_EVAL;
    a.C = dC;
    a.in_pop = dlab;
    a.out_L = dL;
    a.out_top = dtop;
    BTRY(launch_batch(a, smem, 0));
    PGA_CUDA(cudaDeviceSynchronize());
    PGA_CUDA(cudaMemcpy(L, dL, sizeof(double) * (size_t)B * P, cudaMemcpyDeviceToHost));
    PGA_CUDA(cudaMemcpy(top, dtop, sizeof(int32_t) * (size_t)B * P, cudaMemcpyDeviceToHost));
    return PGA_OK;
}

int pga_batch_op_step(int32_t B, int32_t N, const pga_params *p, const int32_t *pop, const double *L,
                      const int32_t *top, int32_t gen, int32_t *next) {
    if (!p || !pop || !L || !top || !next) return pga::fail(PGA_EINVAL, "NULL argument");
    BArgs a;
    size_t smem = 0;
    BTRY(fill_args(a, B, N, p, p->device, &smem));
    const int P = a.P;
    for (size_t k = 0; k < (size_t)B * P * N; ++k)
        if (pop[k] < 0 || pop[k] >= N) return pga::fail(PGA_EINVAL, "pop labels must lie in 0..N-1");
    for (size_t k = 0; k < (size_t)B * P; ++k)
        if (top[k] < -1 || top[k] >= N) return pga::fail(PGA_EINVAL, "top must lie in -1..N-1");
    BTRY(pga::ensure_device(p->device));
    BTRY(check_smem(smem, p->device));
    DBufs d;
    double *dL;
    int32_t *dpop, *dtop, *dnext;
    BTRY(d.get(&dpop, (size_t)B * P * N));
    BTRY(d.get(&dnext, (size_t)B * P * N));
    BTRY(d.get(&dL, (size_t)B * P));
    BTRY(d.get(&dtop, (size_t)B * P));
    PGA_CUDA(cudaMemcpy(dpop, pop, sizeof(int32_t) * (size_t)B * P * N, cudaMemcpyHostToDevice));
    PGA_CUDA(cudaMemcpy(dL, L, sizeof(double) * (size_t)B * P, cudaMemcpyHostToDevice));
    PGA_CUDA(cudaMemcpy(dtop, top, sizeof(int32_t) * (size_t)B * P, cudaMemcpyHostToDevice));
    a.mode = MODE_STEP;
    a.in_pop = dpop;
    a.in_L = dL;
    a.in_top = dtop;
    a.hook_gen = gen;
    a.out_pop = dnext;
    BTRY(launch_batch(a, smem, 0));
    PGA_CUDA(cudaDeviceSynchronize());
    PGA_CUDA(cudaMemcpy(next, dnext, sizeof(int32_t) * (size_t)B * P * N, cudaMemcpyDeviceToHost));
    return PGA_OK;
}

}  // extern "C"
