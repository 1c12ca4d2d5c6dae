// ga.cu — the per-generation GA operators of Alg. 1 on device:
// initial population, state & statistics, termination, isolate fittest,
// elitism, scaling, SUS / tournament selection, mate pairing, crossover
// (knowledge-based or one-point), mutation, canonicalisation, replacement,
// and elite migration between islands.  DESIGN.md §3 fixes every detail the
// paper leaves open (readings Q7-Q21); the Philox stream layout makes every
// operator bit-reproducible.
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdlib>
#include <cub/block/block_radix_sort.cuh>

#include "pga_internal.cuh"

namespace {

using namespace pgad;

// ---------------------------------------------------------------------------
// warp-cooperative first-occurrence canonicalisation (Q7)
// The caller streams genes in order, 32 per step; `table` (per warp, smem,
// >= max label + 1 entries, initialised to 0xFFFF) maps old -> new labels.
// ---------------------------------------------------------------------------
struct Canon {
    uint16_t *table;
    int next;
    __device__ __forceinline__ uint32_t step(uint32_t s, bool valid, int lane) {
        const uint32_t key = valid ? s : (0x10000u + (uint32_t)lane);
        return assign(s, valid, lane, __match_any_sync(0xFFFFFFFFu, key));
    }
    // m = __match_any_sync of this step's keys (may be computed ahead).
    __device__ __forceinline__ uint32_t assign(uint32_t s, bool valid, int lane, unsigned m) {
        const bool leader = (__ffs(m) - 1) == lane;
        const bool fresh = valid && leader && table[s] == 0xFFFF;
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, fresh);
        if (fresh) table[s] = (uint16_t)(next + __popc(bal & lanemask_lt()));
        next += __popc(bal);
        __syncwarp();
        return valid ? (uint32_t)table[s] : 0u;
    }
};

__device__ __forceinline__ void table_reset(uint16_t *table, int n, int lane) {
    for (int k = lane; k < n; k += 32) table[k] = 0xFFFF;
    __syncwarp();
}

// Same for a 16-byte-aligned table whose capacity is a multiple of 8 entries.
__device__ __forceinline__ void table_reset16(uint16_t *table, int n, int lane) {
    uint4 *t = reinterpret_cast<uint4 *>(table);
    const uint4 ones = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    for (int k = lane; k < (n + 7) / 8; k += 32) t[k] = ones;
    __syncwarp();
}

// per-child table stride in the breed kernel: N + 1 entries rounded to 8 (16 B)
__host__ __device__ __forceinline__ int breed_tab(int N) { return (N + 1 + 7) & ~7; }

// ---------------------------------------------------------------------------
// k_init: warp per chromosome.  gene i of chromosome p_global:
// scale(Philox(INIT; i>>2, p_global)[i&3], N), generation field 0xFFFFFFFF.
// ---------------------------------------------------------------------------
__global__ void k_init(uint64_t seed, int N, int ldn, int64_t P, int64_t Pcap, int64_t p_off,
                       uint32_t island, uint16_t *CM, uint16_t *GM, int32_t *out32) {
    extern __shared__ uint16_t tables[];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t p = (int64_t)blockIdx.x * nw + warp;
    if (p >= P) return;
    uint16_t *table = tables + (size_t)warp * (N + 1);
    table_reset(table, N + 1, lane);
    Canon cn{table, 0};
    for (int base = 0; base < N; base += 32) {
        const int i = base + lane;
        const bool valid = i < N;
        uint32_t s = 0;
        if (valid) {
            const U4 u = draw(seed, pga::TAG_INIT, island, 0xFFFFFFFFu, (uint32_t)(i >> 2),
                              (uint32_t)(p_off + p));
            s = scale_u32(word(u, i & 3), (uint32_t)N);
        }
        const uint32_t c = cn.step(s, valid, lane);
        if (valid) {
            if (CM) CM[p * ldn + i] = (uint16_t)c;
            if (GM) GM[(int64_t)i * Pcap + p] = (uint16_t)c;
            if (out32) out32[p * N + i] = (int32_t)c;
        }
    }
}

// ---------------------------------------------------------------------------
// k_canon_i32: canonicalise int32 labels in place (test hook), warp per row.
// ---------------------------------------------------------------------------
__global__ void k_canon_i32(int32_t *lab, int64_t P, int N, int tab) {
    extern __shared__ uint16_t tables[];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t p = (int64_t)blockIdx.x * nw + warp;
    if (p >= P) return;
    uint16_t *table = tables + (size_t)warp * tab;
    table_reset(table, tab, lane);
    Canon cn{table, 0};
    for (int base = 0; base < N; base += 32) {
        const int i = base + lane;
        const bool valid = i < N;
        const uint32_t s = valid ? (uint32_t)lab[p * N + i] : 0u;
        const uint32_t c = cn.step(s, valid, lane);
        if (valid) lab[p * N + i] = (int32_t)c;
    }
}

// ---------------------------------------------------------------------------
// k_stats: best (lowest index on ties), mean, stall counter, termination
// flag, best-ever labels, history (Alg. 1; Q16, Q17).  Each CTA
// reduces a fixed contiguous slice; the last CTA to finish reduces the
// partials in CTA order (deterministic) and updates the state.
// mode 0: single island, update stall every generation
// mode 1: multi-island non-migration generation: statistics only
// mode 2: multi-island migration generation: stall on the (global) best
// ---------------------------------------------------------------------------
constexpr int STATS_T = 1024, STATS_PER_CTA = 4096, STATS_MAXG = 1024;

__device__ __forceinline__ void stats_reduce(double &best, int &bi, double &sum, double *sb, int *si,
                                             double *ss) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ob = __shfl_xor_sync(0xFFFFFFFFu, best, off);
        const int oi = __shfl_xor_sync(0xFFFFFFFFu, bi, off);
        sum += __shfl_xor_sync(0xFFFFFFFFu, sum, off);
        if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    if (lane == 0) {
        sb[warp] = best;
        si[warp] = bi;
        ss[warp] = sum;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        best = lane < nw ? sb[lane] : -1.0;
        bi = lane < nw ? si[lane] : 0x7FFFFFFF;
        sum = lane < nw ? ss[lane] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ob = __shfl_xor_sync(0xFFFFFFFFu, best, off);
            const int oi = __shfl_xor_sync(0xFFFFFFFFu, bi, off);
            sum += __shfl_xor_sync(0xFFFFFFFFu, sum, off);
            if (ob > best || (ob == best && oi < bi)) {
                best = ob;
                bi = oi;
            }
        }
    }
}

__global__ void __launch_bounds__(STATS_T)
k_stats(const double *__restrict__ L, int64_t P, const uint16_t *CM0, const uint16_t *CM1,
        int ldn, int N, pga::DevState *st, uint16_t *best_labels, double *history,
        int hist_cap, double tol, int stall_gens, int max_gens, int mode, int migrate_every,
        double *part, uint32_t *counter, int64_t per) {
    __shared__ double sb[32], ss[32];
    __shared__ int si[32];
    __shared__ int s_improved, s_bi, s_last;
    pdl_wait();
    pdl_trigger();
    if (st->done) return;
    const int tid = threadIdx.x;
    double best = -1.0, sum = 0.0;
    int bi = 0x7FFFFFFF;
    const int64_t lo = (int64_t)blockIdx.x * per, hi = min(P, lo + per);
    for (int64_t i = lo + tid; i < hi; i += blockDim.x) {
        const double v = L[i];
        sum += v;
        if (v > best) {  // ascending i per thread -> first max kept
            best = v;
            bi = (int)i;
        }
    }
    stats_reduce(best, bi, sum, sb, si, ss);
    if (gridDim.x > 1) {
        if (tid == 0) {
            part[3 * blockIdx.x] = best;
            part[3 * blockIdx.x + 1] = sum;
            part[3 * blockIdx.x + 2] = (double)bi;   // exact: |bi| < 2^31
            __threadfence();
            s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        // partials in CTA order: thread t takes CTA t (<= STATS_MAXG), then the same tree
        best = -1.0;
        sum = 0.0;
        bi = 0x7FFFFFFF;
        if (tid < (int)gridDim.x) {
            const volatile double *vp = part;
            best = vp[3 * tid];
            sum = vp[3 * tid + 1];
            bi = (int)vp[3 * tid + 2];
        }
        __syncthreads();
        stats_reduce(best, bi, sum, sb, si, ss);
        if (tid == 0) *counter = 0u;
    }
    if (tid == 0) {
        const int g = st->gen;
        st->best = best;
        st->best_idx = bi;
        st->mean = sum / (double)P;
        if (g < hist_cap) history[g] = best;
        if (mode == 0) {
            if (g > 0) st->stall = (best - st->prev_best < tol) ? st->stall + 1 : 0;
            st->prev_best = best;
        } else if (mode == 2) {
            if (g + 1 > migrate_every)
                st->stall = (best - st->prev_best < tol) ? st->stall + migrate_every : 0;
            st->prev_best = best;
        }
        int done = 0;
        if (tol >= 0.0 && st->stall >= stall_gens) {
            done = 1;
            st->reason = PGA_REASON_STALLED;
        }
        if (g + 1 >= max_gens) done = 1;
        st->done = done;
        const int improved = (best > st->best_ever) ? 1 : 0;
        if (improved) st->best_ever = best;
        s_improved = improved;
        s_bi = bi;               // broadcast the argmax
    }
    __syncthreads();
    if (s_improved) {
        const uint16_t *CM = (st->gen & 1) ? CM1 : CM0;
        const int b = s_bi;
        for (int i = tid; i < N; i += blockDim.x) best_labels[i] = CM[(int64_t)b * ldn + i];
    }
}

// ---------------------------------------------------------------------------
// selection
// ---------------------------------------------------------------------------

// SUS (Q9) without a search: the M pointers start + m * step are sorted and
// evenly spaced, so individual i (wheel segment [prefix[i-1], prefix[i])) owns
// exactly the pointers m in [ceil((lo - start) / step), ceil((hi - start) /
// step)) -- the same min{i : prefix[i] > ptr} as a binary search, in exact
// u64 arithmetic.  Thread t: the mates slot sigma[t] (t < M, fused) and the
// pointers of individual t (t < P).
__device__ __forceinline__ uint64_t sus_first(uint64_t x, uint64_t start, uint64_t step) {
    return x <= start ? 0ull : (x - start + step - 1) / step;
}

// ---------------------------------------------------------------------------
// SUS for P > SMALL_GA_P without a library scan: two kernels over index
// blocks of SCAN_T individuals.  k_qsum: q_i = floor(2^B w_i / w_max) in
// index order (w from the rank the last merge level wrote, or from L) and
// the block's sum.  k_sus2: the block's exclusive base (sum of the earlier
// block sums) and the total Q from the block sums, an inclusive block scan
// of q, and every individual's SUS pointer range (as k_sus), plus the mate
// slots (Q10).  All integer (u64) arithmetic: the same prefix, bit for bit,
// as any other summation order.
// ---------------------------------------------------------------------------
constexpr int SCAN_T = 1024;

__device__ __forceinline__ uint64_t block_sum_u64(uint64_t v, uint64_t *ws) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, off);
    __syncthreads();                      // ws may still be read from a previous call
    if (lane == 0) ws[wid] = v;
    __syncthreads();
    uint64_t t = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += ws[k];
    return t;
}

__global__ void __launch_bounds__(SCAN_T) k_qsum(const double *__restrict__ L, const int32_t *__restrict__ order,
                                                 const int32_t *__restrict__ rank, int64_t P, int scaling,
                                                 uint64_t *q, uint64_t *bsum, const int32_t *done) {
    pdl_wait();
    pdl_trigger();
    if (done && *done) return;
    __shared__ uint64_t ws[SCAN_T / 32];
    const int64_t i = (int64_t)blockIdx.x * SCAN_T + threadIdx.x;
    uint64_t qi = 0;
    if (i < P) {
        const int B = 62 - ceil_log2_d(P);
        double w, wmax;
        if (scaling == PGA_SCALE_RANK) {
            w = 1.0 / sqrt((double)(rank[i] + 1));
            wmax = 1.0;
        } else {
            w = L[i];
            wmax = L[order[0]];
        }
        if (wmax > 0.0) {
            const double x = w / wmax;
            if (x > 0.0) qi = (uint64_t)floor(ldexp(x, B));
        }
        q[i] = qi;
    }
    const uint64_t t = block_sum_u64(qi, ws);
    if (threadIdx.x == 0) bsum[blockIdx.x] = t;
}

template <int T>
__global__ void __launch_bounds__(T) k_sus2(const uint64_t *__restrict__ q, const uint64_t *__restrict__ bsum,
                                                 int nbq, const double *__restrict__ L,
                                                 const int32_t *__restrict__ order, int64_t P, int64_t M,
                                                 int scaling, uint64_t seed, uint32_t gen, uint32_t island,
                                                 int32_t *sel, const int32_t *done, const int32_t *gen_ptr,
                                                 int32_t *sigma) {
    pdl_wait();
    pdl_trigger();
    if (done && *done) return;
    __shared__ uint64_t ws[T / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t t = (int64_t)blockIdx.x * T + tid;
    if (gen_ptr) gen = (uint32_t)*gen_ptr;
    if (sigma && t < M) sigma[t] = feistel_slot(t, M, seed, gen, island);   // mates fused (Q10)
    const double wmax = (scaling == PGA_SCALE_RANK) ? 1.0 : L[order[0]];
    if (!(wmax > 0.0)) {   // all-zero fitness: uniform fallback; block-uniform
        if (t < M) {
            const U4 u = draw(seed, pga::TAG_SUS, island, gen, (uint32_t)t, 0u);
            sel[t] = (int32_t)scale_u32(u.x, (uint32_t)P);
        }
        return;
    }
    // base of this block and the total Q from the block sums
    uint64_t a = 0, b = 0;
    for (int k = tid; k < nbq; k += T) {
        const uint64_t v = bsum[k];
        b += v;
        if (k < (int)blockIdx.x) a += v;
    }
    const uint64_t base = block_sum_u64(a, ws);
    const uint64_t Q = block_sum_u64(b, ws);
    // inclusive scan of q over the block
    const uint64_t qi = t < P ? q[t] : 0ull;
    uint64_t incl = qi;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += o;
    }
    __syncthreads();
    if (lane == 31) ws[wid] = incl;
    __syncthreads();
    uint64_t wbase = 0;
    for (int k = 0; k < wid; ++k) wbase += ws[k];
    if (t >= P) return;
    const uint64_t hi = base + wbase + incl, lo = hi - qi;
    const uint64_t step = Q / (uint64_t)M;
    const U4 u = draw(seed, pga::TAG_SUS, island, gen, 0u, 0xFFFFFFFFu);
    const uint64_t x = ((uint64_t)u.x << 32) | (uint64_t)u.y;
    const uint64_t start = __umul64hi(x, step);
    const int64_t m0 = (int64_t)min(sus_first(lo, start, step), (uint64_t)M);
    const int64_t m1 = (int64_t)min(sus_first(hi, start, step), (uint64_t)M);
    PGA_DCHECK(hi >= lo && hi <= Q);
    for (int64_t m = m0; m < m1; ++m) sel[m] = (int32_t)t;
}

__global__ void k_tournament(const double *__restrict__ L, int64_t P, int64_t M, int k,
                             uint64_t seed, uint32_t gen, uint32_t island, int32_t *sel,
                             const int32_t *done, const int32_t *gen_ptr, int32_t *sigma) {
    pdl_wait();
    pdl_trigger();
    if (done && *done) return;
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    if (gen_ptr) gen = (uint32_t)*gen_ptr;
    if (sigma) sigma[m] = feistel_slot(m, M, seed, gen, island);   // mates fused (Q10)
    const U4 u = draw(seed, pga::TAG_TOUR, island, gen, (uint32_t)m, 0u);
    int best = (int)scale_u32(u.x, (uint32_t)P);
    for (int t = 1; t < k; ++t) {
        const int c = (int)scale_u32(word(u, t), (uint32_t)P);
        if (L[c] > L[best] || (L[c] == L[best] && c < best)) best = c;
    }
    sel[m] = best;
}

// Mutation masks of one generation (Q13, Q27): gene i of child slot o
// mutates iff Philox(MUT; i >> 2, p_off + o)[i & 3] < thr(p_m) -- the same
// draws the breed would make, one bit per gene, [Pcap][mw] 32-bit words,
// thread per word (8 Philox blocks).  They depend only on (seed, generation,
// island, slot), so the GA computes them on its side stream beside the
// fitness pass (launch_mates_fork); elites (o < E) are never mutated.
__global__ void k_mutmask(RoundKeys rk, uint32_t island, const int32_t *gen_ptr, const int32_t *done, int64_t P,
                          int N, int E, int64_t p_off, uint64_t thr_m, int mw, uint32_t *mask) {
    if (done && *done) return;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t o = t / mw;
    const int w = (int)(t - o * mw);
    if (o >= P || o < E) return;
    const uint32_t gen = (uint32_t)*gen_ptr;
    const uint32_t og = (uint32_t)(p_off + o);
    uint32_t bits = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int blk = 8 * w + k;
        if (4 * blk < N) {
            const U4 u = draw_rk(rk, pga::TAG_MUT, island, gen, (uint32_t)blk, og);
            bits |= (((uint64_t)u.x < thr_m ? 1u : 0u) | ((uint64_t)u.y < thr_m ? 2u : 0u) |
                     ((uint64_t)u.z < thr_m ? 4u : 0u) | ((uint64_t)u.w < thr_m ? 8u : 0u)) << (4 * k);
        }
    }
    mask[o * mw + w] = bits;
}

// Mate pairing (Q10): sigma = keyed Feistel permutation of the M slots
// (4 rounds, round function Philox(PERM; R, round)[0], cycle-walking).
__global__ void k_mates(int64_t M, uint64_t seed, uint32_t gen, uint32_t island, int32_t *sigma,
                        const int32_t *done, const int32_t *gen_ptr) {
    if (done && *done) return;
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    if (gen_ptr) gen = (uint32_t)*gen_ptr;
    sigma[m] = feistel_slot(m, M, seed, gen, island);
}

// ---------------------------------------------------------------------------
// k_select_small: P <= SMALL_P in ONE CTA (what the multi-kernel path does
// with ~8 launches): order by (L desc, idx asc) via a shared-memory bitonic
// sort, rank scaling, exact u64 prefix, SUS or tournament, Feistel mates.
// what: bit 0 = order, bit 1 = selection + mates.
// ---------------------------------------------------------------------------
constexpr int SMALL_P = 4096, SMALL_T = 1024;

// (ka, va) < (kb, vb) lexicographically = the 96-bit number ka:va below
// kb:vb: the borrow out of one subtraction chain (4 instructions instead of
// two 64-bit compares, an equality test and the index compare)
__device__ __forceinline__ bool kv_less(uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
#ifdef PGA_KV_PLAIN
    return ka < kb || (ka == kb && va < vb);
#else
    uint32_t r;
    asm("{\n\t.reg .u32 t;\n\t"
        "sub.cc.u32 t, %1, %4;\n\t"
        "subc.cc.u32 t, %2, %5;\n\t"
        "subc.cc.u32 t, %3, %6;\n\t"
        "subc.u32 %0, 0, 0;\n\t}"
        : "=r"(r)
        : "r"(va), "r"((uint32_t)ka), "r"((uint32_t)(ka >> 32)), "r"(vb), "r"((uint32_t)kb),
          "r"((uint32_t)(kb >> 32)));
    return r != 0u;
#endif
}


__global__ void __launch_bounds__(SMALL_T)
k_select_small(int what, const double *__restrict__ L, int P, int M, int selection, int tour_k, int scaling,
               uint64_t seed, uint32_t gen, uint32_t island, const int32_t *gen_ptr, int32_t *order,
               int32_t *sel, int32_t *sigma, const int32_t *done) {
    pdl_wait();
    pdl_trigger();
    if (done && *done) return;
    extern __shared__ __align__(16) unsigned char ssm[];
    using BRS0 = cub::BlockRadixSort<uint64_t, SMALL_T, SMALL_P / SMALL_T, uint32_t>;
    constexpr size_t SK_BYTES = (size_t)SMALL_P * 8 > sizeof(typename BRS0::TempStorage)
                                    ? (size_t)SMALL_P * 8 : sizeof(typename BRS0::TempStorage);
    uint64_t *sk = reinterpret_cast<uint64_t *>(ssm);               // sort temp storage, then prefix
    double *sL = reinterpret_cast<double *>(ssm + SK_BYTES);        // [SMALL_P]
    uint32_t *sv = reinterpret_cast<uint32_t *>(sL + SMALL_P);      // [SMALL_P]
    int32_t *srank = reinterpret_cast<int32_t *>(sv + SMALL_P);     // [SMALL_P]
    __shared__ uint64_t wsum[SMALL_T / 32];
    __shared__ int32_t s_top;
    const int tid = threadIdx.x;
    if (gen_ptr) gen = (uint32_t)*gen_ptr;
    if (P <= SMALL_T) {
        // small: bitonic network on n2 <= 1024 items (one pair per thread per stage)
        int n2 = 2;
        while (n2 < P) n2 <<= 1;
        uint32_t *svv = sv;
        uint64_t *skk = reinterpret_cast<uint64_t *>(srank + SMALL_P);   // scratch after srank
        for (int t = tid; t < n2; t += SMALL_T) {
            if (t < P) {
                double x = L[t];
                if (x == 0.0) x = 0.0;
                sL[t] = x;
                skk[t] = ~(uint64_t)__double_as_longlong(x);
                svv[t] = (uint32_t)t;
            } else {
                skk[t] = ~0ull;
                svv[t] = 0xFFFFFFFFu;
            }
        }
        __syncthreads();
        for (int size = 2; size <= n2; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                const int t = tid;
                if (t < n2 / 2) {
                    const int i = 2 * t - (t & (stride - 1)), j = i + stride;
                    const bool up = (i & size) == 0;
                    const uint64_t ki = skk[i], kj = skk[j];
                    const uint32_t vi = svv[i], vj = svv[j];
                    if (kv_less(kj, vj, ki, vi) == up) {
                        skk[i] = kj; skk[j] = ki;
                        svv[i] = vj; svv[j] = vi;
                    }
                }
                __syncthreads();
            }
    } else {
        // stable in-CTA radix sort of (key = ~bits(L), value = index); items
        // are loaded in index order (blocked), so equal keys stay in index order
        using BRS = cub::BlockRadixSort<uint64_t, SMALL_T, SMALL_P / SMALL_T, uint32_t>;
        uint64_t kk[SMALL_P / SMALL_T];
        uint32_t vv[SMALL_P / SMALL_T];
#pragma unroll
        for (int k = 0; k < SMALL_P / SMALL_T; ++k) {
            const int t = tid * (SMALL_P / SMALL_T) + k;
            if (t < P) {
                double x = L[t];
                if (x == 0.0) x = 0.0;
                sL[t] = x;
                kk[k] = ~(uint64_t)__double_as_longlong(x);
                vv[k] = (uint32_t)t;
            } else {
                kk[k] = ~0ull;
                vv[k] = 0xFFFFFFFFu;
            }
        }
        {
            typename BRS::TempStorage &ts = *reinterpret_cast<typename BRS::TempStorage *>(sk);
            BRS(ts).Sort(kk, vv);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < SMALL_P / SMALL_T; ++k) sv[tid * (SMALL_P / SMALL_T) + k] = vv[k];
        __syncthreads();
    }
    for (int r = tid; r < P; r += SMALL_T) {
        srank[sv[r]] = r + 1;
        if (what & 1) order[r] = (int32_t)sv[r];
    }
    if (tid == 0) s_top = (int32_t)sv[0];
    __syncthreads();
    if (!(what & 2)) return;
    if (selection == PGA_SEL_TOURNAMENT) {
        for (int m = tid; m < M; m += SMALL_T) {
            const U4 u = draw(seed, pga::TAG_TOUR, island, gen, (uint32_t)m, 0u);
            int best = (int)scale_u32(u.x, (uint32_t)P);
            for (int t = 1; t < tour_k; ++t) {
                const int c = (int)scale_u32(word(u, t), (uint32_t)P);
                if (sL[c] > sL[best] || (sL[c] == sL[best] && c < best)) best = c;
            }
            sel[m] = best;
        }
    } else {
        const double wmax = (scaling == PGA_SCALE_RANK) ? 1.0 : sL[s_top];
        if (!(wmax > 0.0)) {
            for (int m = tid; m < M; m += SMALL_T) {
                const U4 u = draw(seed, pga::TAG_SUS, island, gen, (uint32_t)m, 0u);
                sel[m] = (int32_t)scale_u32(u.x, (uint32_t)P);
            }
        } else {
            const int B = 62 - ceil_log2_d(P);
            // q_i (index order) and an inclusive block scan: thread t owns
            // items 4t .. 4t+3 (P <= 4 * SMALL_T)
            uint64_t q[4], run = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * tid + k;
                uint64_t qi = 0;
                if (i < P) {
                    const double w = (scaling == PGA_SCALE_RANK) ? 1.0 / sqrt((double)srank[i]) : sL[i];
                    const double x = w / wmax;
                    if (x > 0.0) qi = (uint64_t)floor(ldexp(x, B));
                }
                run += qi;
                q[k] = run;
            }
            const int lane = tid & 31, wid = tid >> 5;
            uint64_t incl = run;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, incl, off);
                if (lane >= off) incl += o;
            }
            if (lane == 31) wsum[wid] = incl;
            __syncthreads();
            if (wid == 0) {
                uint64_t v = wsum[lane];
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, v, off);
                    if (lane >= off) v += o;
                }
                wsum[lane] = v;
            }
            __syncthreads();
            const uint64_t base = (incl - run) + (wid ? wsum[wid - 1] : 0ull);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * tid + k;
                if (i < P) sk[i] = base + q[k];
            }
            __syncthreads();
            const uint64_t Q = sk[P - 1];
            const uint64_t step = Q / (uint64_t)M;
            const U4 u = draw(seed, pga::TAG_SUS, island, gen, 0u, 0xFFFFFFFFu);
            const uint64_t x = ((uint64_t)u.x << 32) | (uint64_t)u.y;
            const uint64_t start = __umul64hi(x, step);
            for (int m = tid; m < M; m += SMALL_T) {
                const uint64_t ptr = start + (uint64_t)m * step;
                int lo = 0, hi = P - 1;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (sk[mid] > ptr) hi = mid;
                    else lo = mid + 1;
                }
                sel[m] = lo;
            }
        }
    }
    for (int m = tid; m < M; m += SMALL_T) sigma[m] = feistel_slot(m, M, seed, gen, island);
}

// ---------------------------------------------------------------------------
// Order (isolate fittest) for P > 4096: (1) runs of RUN items, each
// sorted in one CTA by a shared-memory bitonic network on (key = ~bits(L),
// index) -- a total order, indices being unique; (2) a merge tree: at width
// w every item moves to (start of its 2w block) + (its offset in its run) +
// (number of items of the sibling run before it), found by binary search.
// The last level writes the indices to order.  1 + ceil(log2(P / RUN))
// launches, each spread over the whole GPU.
// ---------------------------------------------------------------------------
#ifndef PGA_SORT_RUN
#define PGA_SORT_RUN 512
#endif
// bitonic runs in shared memory (RUN * 12 B); 512 measured best of 256..4096 with the
// borrow-chain compare (C4 0.4878 -> 0.4845 ms per generation against 1024; 256: 0.4858)
constexpr int RUN = PGA_SORT_RUN, RUN_T = RUN;   // one thread per item
static_assert(RUN <= 1024, "one CTA thread per run item");

// compare-exchange of a bitonic stage with the partner lane (stride < 32):
// keep the smaller (key, index) when keep_min, else the larger
__device__ __forceinline__ void cs_exchange(uint64_t &k, uint32_t &v, int partner_lane_xor, bool keep_min) {
    const uint64_t ok = __shfl_xor_sync(0xFFFFFFFFu, k, partner_lane_xor);
    const uint32_t ov = __shfl_xor_sync(0xFFFFFFFFu, v, partner_lane_xor);
    const bool other_less = kv_less(ok, ov, k, v);
    if (other_less == keep_min) {
        k = ok;
        v = ov;
    }
}

// ---------------------------------------------------------------------------
// Isolate fittest + rank scaling (Alg. 1) for SMALL_GA_P < P <=
// RANKC_MAXP, spread over the whole GPU.  The position of i in the (L desc,
// index asc) order is the number of j before it.  CTA (x, y) sorts chunk y
// of RS_T individuals in shared memory (bitonic, one item per thread) and
// each of the RS_T * IPT individuals i of tile x counts the chunk's items before
// it by a binary search; the counts are added into acc[i] (integer atomics:
// the sum is order-free).  The last CTA of tile x to finish (threadfence +
// per-tile counter) reads and re-zeroes acc, writes rank and order and,
// for SUS with rank scaling (Table 3), forms q_i = qtab[rank_i] =
// floor(2^B / sqrt(rank_i + 1)), publishes the tile's sum, waits until all
// tiles have published theirs (the finalising CTAs are running: at most
// RS_MAXTILES of them wait, every other CTA has finished or will), and
// writes the tile's SUS pointer ranges from its base, Q and a block scan --
// the exact u64 prefix of k_qsum + k_sus2, without their launches.  A sort of a few thousand items in one CTA or one
// cluster is a chain of dependent steps on a handful of SMs; here each CTA's
// chain is one 512-item sort and one or two 10-step searches per thread.
// ---------------------------------------------------------------------------
#ifndef PGA_RS_T
#define PGA_RS_T 512
#endif
// chunk RS_T; tile RS_T * IPT individuals: IPT = 1 up to P = 8192 (16 x 16
// CTAs keep every SM busy: island-load 8 0.1130 -> 0.1111 ms), IPT = 2
// above (fewer chunk sorts: island-load 4 0.1921 -> 0.1810 ms)
constexpr int RS_T = PGA_RS_T;
constexpr int RS_MAXTILES = 32;   // per-tile counters, then the SUS arrive / depart counters
static_assert(pga::RANKC_MAXP <= (int64_t)RS_T * RS_MAXTILES, "tile counters");

__device__ __forceinline__ uint64_t order_key(double x) {
    if (x == 0.0) x = 0.0;   // -0 ties +0
    return ~(uint64_t)__double_as_longlong(x);
}

template <int RS_IPT>
__global__ void __launch_bounds__(RS_T) k_rank_sel(const double *__restrict__ L, int P,
                                                   const uint64_t *__restrict__ qtab, int32_t *__restrict__ acc,
                                                   uint32_t *ctr, int32_t *__restrict__ order,
                                                   int32_t *__restrict__ rank, bool q, uint64_t *bsum, int M,
                                                   uint64_t seed, uint32_t island, const int32_t *gen_ptr,
                                                   int32_t *__restrict__ sel) {
    // no early exit on the done flag: the statistics may raise it during
    // this launch (side stream), and every CTA must reach the counter
    constexpr int RS_TILE = RS_T * RS_IPT;
    pdl_wait();
    pdl_trigger();
    __shared__ uint64_t sk[RS_T];
    __shared__ uint32_t sv[RS_T];
    __shared__ uint64_t ws[RS_T / 32];
    __shared__ int s_last;
    const int tid = threadIdx.x;
    // ---- this CTA's chunk, sorted by (key, index)
    {
        const int j = blockIdx.y * RS_T + tid;
        uint64_t k = ~0ull;
        uint32_t v = 0xFFFFFFFFu;   // padding: after every individual
        if (j < P) {
            k = order_key(L[j]);
            v = (uint32_t)j;
        }
        for (int size = 2; size <= RS_T; size <<= 1) {
            const bool up = (tid & size) == 0;
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                const bool lower = (tid & stride) == 0;
                if (stride < 32) {
                    cs_exchange(k, v, stride, lower == up);
                } else {
                    __syncthreads();
                    sk[tid] = k;
                    sv[tid] = v;
                    __syncthreads();
                    const uint64_t ok = sk[tid ^ stride];
                    const uint32_t ov = sv[tid ^ stride];
                    if (kv_less(ok, ov, k, v) == (lower == up)) {
                        k = ok;
                        v = ov;
                    }
                }
            }
        }
        __syncthreads();
        sk[tid] = k;
        sv[tid] = v;
        __syncthreads();
    }
    // ---- items of the chunk before individual i: lower bound of (key_i, i)
#pragma unroll
    for (int k = 0; k < RS_IPT; ++k) {
        const int i = blockIdx.x * RS_TILE + k * RS_T + tid;
        if (i < P) {
            const uint64_t ki = order_key(L[i]);
            int lo = 0;   // lower bound in [0, RS_T]
#pragma unroll
            for (int h = RS_T / 2; h > 0; h >>= 1)
                if (kv_less(sk[lo + h - 1], sv[lo + h - 1], ki, (uint32_t)i)) lo += h;
            lo += (int)kv_less(sk[lo], sv[lo], ki, (uint32_t)i);   // lo <= RS_T - 1 here
            if (lo) atomicAdd(acc + i, lo);
        }
    }
    // ---- the last CTA of tile x (all chunks counted): rank, order, q_i and
    // the tile's sum of q (k_sus2 scans the tile sums); accumulators and
    // counter re-zeroed
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(ctr + blockIdx.x, 1u) == gridDim.y - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    uint64_t qs = 0, qk[RS_IPT];
#pragma unroll
    for (int k = 0; k < RS_IPT; ++k) {
        qk[k] = 0;
        const int i = blockIdx.x * RS_TILE + k * RS_T + tid;
        if (i < P) {
            const int32_t r = __ldcg(acc + i);
            PGA_DCHECK(r >= 0 && r < P);
            acc[i] = 0;
            rank[i] = r;
            order[r] = i;
            if (q) {
                qk[k] = qtab[r];
                qs += qk[k];
            }
        }
    }
    if (tid == 0) ctr[blockIdx.x] = 0u;
    if (!q) return;
    // ---- SUS (as k_sus2): publish the tile's sum of q, wait for every
    // tile's (the nb finalising CTAs are running: their tiles' other CTAs
    // have finished), then the tile's base, Q, a block scan of q in index
    // order and each individual's pointer range
    const int nb = (int)gridDim.x;
    uint32_t *arrive = ctr + RS_MAXTILES, *depart = arrive + 1;
    const uint64_t tsum = block_sum_u64(qs, ws);
    if (tid == 0) {
        bsum[blockIdx.x] = tsum;
        __threadfence();
        atomicAdd(arrive, 1u);
        while (*reinterpret_cast<volatile uint32_t *>(arrive) < (uint32_t)nb) __nanosleep(64);
        __threadfence();
    }
    __syncthreads();
    uint64_t a = 0, b = 0;
    for (int k = tid; k < nb; k += RS_T) {
        const uint64_t v = __ldcg(bsum + k);
        b += v;
        if (k < (int)blockIdx.x) a += v;
    }
    const uint64_t base = block_sum_u64(a, ws);
    const uint64_t Q = block_sum_u64(b, ws);
    if (tid == 0 && atomicAdd(depart, 1u) == (uint32_t)nb - 1) {   // the last to read arrive
        *arrive = 0u;
        *depart = 0u;
    }
    const uint32_t gen = (uint32_t)*gen_ptr;
    const uint64_t step = Q / (uint64_t)M;
    const U4 u = draw(seed, pga::TAG_SUS, island, gen, 0u, 0xFFFFFFFFu);
    const uint64_t start = __umul64hi(((uint64_t)u.x << 32) | (uint64_t)u.y, step);
    const int lane = tid & 31, wid = tid >> 5;
    uint64_t run = base;
#pragma unroll
    for (int k = 0; k < RS_IPT; ++k) {
        const int i = blockIdx.x * RS_TILE + k * RS_T + tid;
        uint64_t incl = qk[k];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, incl, off);
            if (lane >= off) incl += o;
        }
        __syncthreads();
        if (lane == 31) ws[wid] = incl;
        __syncthreads();
        uint64_t wb = 0, tot = 0;
        for (int w = 0; w < RS_T / 32; ++w) {
            const uint64_t t = ws[w];
            if (w < wid) wb += t;
            tot += t;
        }
        if (i < P) {
            const uint64_t hi = run + wb + incl, lo = hi - qk[k];
            const int m0 = (int)min(sus_first(lo, start, step), (uint64_t)M);
            const int m1 = (int)min(sus_first(hi, start, step), (uint64_t)M);
            for (int m = m0; m < m1; ++m) sel[m] = i;
        }
        run += tot;
    }
}

// q by rank for k_rank_sel: qtab[r] = floor(2^B / sqrt(r + 1)) (k_qsum's
// formula with w_max = 1), B = 62 - ceil(log2 P)
__global__ void k_qtab(int P, uint64_t *qtab) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= P) return;
    const int B = 62 - ceil_log2_d(P);
    const double x = 1.0 / sqrt((double)(r + 1));
    qtab[r] = x > 0.0 ? (uint64_t)floor(ldexp(x, B)) : 0ull;
}

// One thread per item: bitonic stages with stride < 32 run as warp shuffles
// (no barrier), larger strides exchange through shared memory.
__global__ void __launch_bounds__(RUN_T)
k_sort_runs(const double *__restrict__ L, int64_t P, uint64_t *keys, int32_t *idx, const int32_t *done) {
    pdl_wait();
    pdl_trigger();
    if (done && *done) return;
    __shared__ uint64_t sk[RUN];
    __shared__ uint32_t sv[RUN];
    const int tid = threadIdx.x;
    const int64_t i = (int64_t)blockIdx.x * RUN + tid;
    uint64_t k = ~0ull;
    uint32_t v = 0xFFFFFFFFu;
    if (i < P) {
        double x = L[i];
        if (x == 0.0) x = 0.0;
        k = ~(uint64_t)__double_as_longlong(x);
        v = (uint32_t)i;
    }
    for (int size = 2; size <= RUN; size <<= 1) {
        const bool up = (tid & size) == 0;
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const bool lower = (tid & stride) == 0;
            if (stride < 32) {
                cs_exchange(k, v, stride, lower == up);
            } else {
                __syncthreads();
                sk[tid] = k;
                sv[tid] = v;
                __syncthreads();
                const uint64_t ok = sk[tid ^ stride];
                const uint32_t ov = sv[tid ^ stride];
                if (kv_less(ok, ov, k, v) == (lower == up)) {
                    k = ok;
                    v = ov;
                }
            }
        }
    }
    if (i < P) {
        keys[i] = k;
        idx[i] = (int32_t)v;
    }
}

// one merge level at run width w: (ks, is) -> (kd, id); kd may be null (last level)
// One merge level.  A CTA's 256 items lie in one run (w is a multiple of
// 256), so their ranks in the sibling run are monotone and cover one
// contiguous range.  Rank = number of sibling items before the item in
// (key, index) order: (1) a sample of every MS-th sibling item is staged in
// shared memory (one coalesced round trip) and searched there, which bounds
// the rank to a window of MS; (2) the union of the CTA's windows is staged in
// shared memory and each item finishes its search there.  Spans too large
// to stage fall back to searches in global memory.  The result is the same
// permutation as a plain per-item binary search.
#ifndef PGA_MERGE_T
#define PGA_MERGE_T 256
#endif
#ifndef PGA_MERGE_MS
#define PGA_MERGE_MS 64
#endif
constexpr int MERGE_T = PGA_MERGE_T, MERGE_MS = PGA_MERGE_MS, MERGE_CAP = 2048;
static_assert(RUN % MERGE_T == 0, "a CTA of the merge must lie in one run");

__device__ __forceinline__ bool key_before(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return kv_less(ka, ia, kb, ib);
}

// WAY-way merge level (WAY = 2 or 4): runs of width w are merged in groups
// of WAY into runs of width WAY * w.  An item's new position = group start +
// its offset in its own run + the number of items before it in each sibling
// run.  All siblings are searched at once: their samples are staged in one
// round trip, then their windows in a second one.
template <int WAY>
__global__ void __launch_bounds__(MERGE_T) k_merge_level(const uint64_t *__restrict__ ks,
                                                         const int32_t *__restrict__ is, int64_t P, int64_t w,
                                                         uint64_t *kd, int32_t *id, int32_t *rank_out,
                                                         const int32_t *done) {
    constexpr int NSIB = WAY - 1, CAP = MERGE_CAP / (WAY == 2 ? 1 : 2);
    pdl_wait();
    pdl_trigger();
    if (done && *done) return;
    __shared__ uint64_t sk[NSIB][CAP];
    __shared__ uint32_t si[NSIB][CAP];
    __shared__ int s_lo[NSIB], s_hi[NSIB];   // positions fit 32 bits (P <= 2^31)
    const int tid = threadIdx.x;
    const int c0 = (int)blockIdx.x * MERGE_T;
    if (c0 >= P) return;
    const int g = c0 + tid;
    const bool valid = g < P;
    const int W = (int)w, blk = c0 / (WAY * W) * (WAY * W), Pi = (int)P;
    const int q = (c0 - blk) / W;                            // own run in the group
    const int off = c0 - blk - q * W + tid;
    const int last = min(MERGE_T, Pi - c0) - 1;            // last valid thread
    const uint64_t ke = valid ? ks[g] : ~0ull;
    const uint32_t ie = valid ? (uint32_t)is[g] : 0xFFFFFFFFu;
    int sib[NSIB], slen[NSIB], ns[NSIB], lo[NSIB], hi[NSIB];
#pragma unroll
    for (int j = 0; j < NSIB; ++j) {
        const int r = j < q ? j : j + 1;
        sib[j] = blk + r * W;
        slen[j] = max(0, min(W, Pi - sib[j]));
        ns[j] = (slen[j] + MERGE_MS - 1) / MERGE_MS;
        lo[j] = 0;
        hi[j] = slen[j];
    }
    // (1) samples of every sibling, one round trip
#pragma unroll
    for (int j = 0; j < NSIB; ++j)
        if (ns[j] > 0 && ns[j] <= CAP)
            for (int t = tid; t < ns[j]; t += MERGE_T) {
                sk[j][t] = __ldg(ks + sib[j] + t * MERGE_MS);
                si[j][t] = (uint32_t)__ldg(is + sib[j] + t * MERGE_MS);
            }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NSIB; ++j)
        if (ns[j] > 0 && ns[j] <= CAP) {
            int a = 0, b = ns[j];                     // samples before the item
            while (a < b) {
                const int m = (a + b) >> 1;
                if (key_before(sk[j][m], si[j][m], ke, ie)) a = m + 1;
                else b = m;
            }
            lo[j] = a > 0 ? (a - 1) * MERGE_MS + 1 : 0;
            hi[j] = min(slen[j], a * MERGE_MS);
        }
    __syncthreads();                                  // samples read: the buffers are reused
    // (2) the CTA's span of windows in every sibling, staged when it fits
#pragma unroll
    for (int j = 0; j < NSIB; ++j) {
        if (tid == 0) s_lo[j] = lo[j];
        if (tid == last) s_hi[j] = hi[j];
    }
    __syncthreads();
    int Lo[NSIB], Hi[NSIB];
#pragma unroll
    for (int j = 0; j < NSIB; ++j) {
        Lo[j] = s_lo[j];
        Hi[j] = s_hi[j];
        if (!valid) lo[j] = hi[j] = Lo[j];            // beyond P: no search
        if (Hi[j] - Lo[j] <= CAP)
            for (int p = Lo[j] + tid; p < Hi[j]; p += MERGE_T) {
                sk[j][p - Lo[j]] = __ldg(ks + sib[j] + p);
                si[j][p - Lo[j]] = (uint32_t)__ldg(is + sib[j] + p);
            }
    }
    __syncthreads();
    int pos = blk + off;
#pragma unroll
    for (int j = 0; j < NSIB; ++j) {
        int l = lo[j], h = hi[j];
        if (Hi[j] - Lo[j] <= CAP) {
            while (l < h) {
                const int m = (l + h) >> 1;
                if (key_before(sk[j][m - Lo[j]], si[j][m - Lo[j]], ke, ie)) l = m + 1;
                else h = m;
            }
        } else {
            const uint64_t *k_g = ks + sib[j];
            const int32_t *i_g = is + sib[j];
            while (l < h) {
                const int m = (l + h) >> 1;
                if (key_before(__ldg(k_g + m), (uint32_t)__ldg(i_g + m), ke, ie)) l = m + 1;
                else h = m;
            }
        }
        pos += l;
    }
    if (!valid) return;
    PGA_DCHECK(pos >= 0 && pos < P);
    if (kd) kd[pos] = ke;
    id[pos] = (int32_t)ie;
    if (rank_out) rank_out[ie] = (int32_t)pos;   // last level: rank (0-based) of individual ie
}

// ---------------------------------------------------------------------------
// k_select_cluster (SMALL_GA_P < P <= CSEL_MAXP): isolate fittest, scaling
// and selection of one island in ONE launch of a 16-CTA thread-block cluster
// (distributed shared memory) -- what the multi-kernel path does with a run
// sort, a merge tree, q sums and a scan (five or more latency-bound launches
// at these sizes).  The mate slots are computed off the critical path (a
// parallel graph branch, launch_mates_fork).
//   1. CTA c holds individuals [c R, (c + 1) R) (R a power of two <= CSEL_T,
//      one per thread) and sorts them by (key = ~bits(L), index): a bitonic
//      network, strides < 32 by warp shuffles, larger ones in shared memory.
//   2. Global rank = local position + the number of items of every other
//      run before it: the other runs are copied in (DSMEM, 16-byte vectors)
//      and searched locally, all runs in lockstep (branch-free bisection).
//   3. order[rank] = index, rank[index] = rank (global memory).
//   4. SUS: q_i in index order from the rank (RANK) or L (NONE), a block
//      scan, the CTA's base from the other CTAs' totals (DSMEM), pointer
//      ranges per individual; or tournament.
// The same integers as the multi-kernel path (bit-exact).
// ---------------------------------------------------------------------------
constexpr int CSEL_T = 1024, CSEL_CL = 16, CSEL_MAXR = CSEL_T / 2;   // >= 2 threads per item in the rank search
constexpr int CSEL_RPT = (CSEL_CL - 1 + 1) / 2;                       // other runs per search thread (at most)
constexpr int CSEL_MAXP = CSEL_CL * CSEL_MAXR;

__host__ __device__ __forceinline__ int csel_run(int P) {
    int r = 64;
    while (r * CSEL_CL < P) r <<= 1;
    return r;
}

static size_t csel_smem(int R) {
    // own run: sk sL sx si srank spos; copies of the other runs' keys and indices
    return (size_t)R * (8 + 8 + 8 + 4 + 4 + 4) + (size_t)(CSEL_CL - 1) * R * 12 + 256;
}

__global__ void __launch_bounds__(CSEL_T, 1)
k_select_cluster(int what, const double *__restrict__ L, int P, int R, int M, int selection, int tour_k,
                 int scaling, uint64_t seed, uint32_t gen, uint32_t island, const int32_t *gen_ptr,
                 int32_t *order, int32_t *rank_out, int32_t *sel, const int32_t *done) {
    namespace cg = cooperative_groups;
    pdl_wait();
    pdl_trigger();
    if (done && *done) return;                     // grid-uniform
    cg::cluster_group cl = cg::this_cluster();
    const int c = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    extern __shared__ __align__(16) unsigned char csm[];
    uint64_t *sk = reinterpret_cast<uint64_t *>(csm);          // [R] sorted keys
    double *sL = reinterpret_cast<double *>(sk + R);           // [R] L by local index
    uint64_t *sx = reinterpret_cast<uint64_t *>(sL + R);       // [R] exchange buffer (sort)
    uint64_t *ok_ = sx + R;                                     // [(CL-1) R] other runs' keys
    uint32_t *si = reinterpret_cast<uint32_t *>(ok_ + (CSEL_CL - 1) * R);   // [R] sorted indices
    int32_t *srank = reinterpret_cast<int32_t *>(si + R);     // [R] global rank by local index
    uint32_t *oi_ = reinterpret_cast<uint32_t *>(srank + R);  // [(CL-1) R] other runs' indices
    int32_t *spos = reinterpret_cast<int32_t *>(oi_ + (CSEL_CL - 1) * R);   // [R] global rank accumulators
    __shared__ uint64_t ws[CSEL_T / 32];
    __shared__ uint64_t s_tot, s_first_key;
    __shared__ uint32_t s_first_idx;
    if (gen_ptr) gen = (uint32_t)*gen_ptr;
    const int base = c * R;
    const bool act = tid < R;

    // (1) load and sort the run: thread t holds position t
    uint64_t k = ~0ull;
    uint32_t v = 0xFFFFFFFFu;
    if (act) {
        const int i = base + tid;
        double x = 0.0;
        if (i < P) {
            x = L[i];
            if (x == 0.0) x = 0.0;
            k = ~(uint64_t)__double_as_longlong(x);
            v = (uint32_t)i;
        }
        sL[tid] = x;
    }
    for (int size = 2; size <= R; size <<= 1) {
        const bool up = (tid & size) == 0;
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const bool lower = (tid & stride) == 0;    // this thread holds the lower position
            if (stride < 32) {
                if (act) cs_exchange(k, v, stride, lower == up);
                else { __shfl_xor_sync(0xFFFFFFFFu, k, stride); __shfl_xor_sync(0xFFFFFFFFu, v, stride); }
            } else {
                __syncthreads();
                if (act) {
                    sx[tid] = k;
                    si[tid] = v;
                }
                __syncthreads();
                if (act) {
                    const uint64_t ok = sx[tid ^ stride];
                    const uint32_t ov = si[tid ^ stride];
                    if (kv_less(ok, ov, k, v) == (lower == up)) {
                        k = ok;
                        v = ov;
                    }
                }
            }
        }
    }
    __syncthreads();
    if (act) {
        sk[tid] = k;
        si[tid] = v;
    }
    if (tid == 0) {
        s_first_key = k;
        s_first_idx = v;
    }
    cl.sync();                                     // every run sorted and visible

    // (2) global ranks: copy the other runs (DSMEM, 16-byte vectors), then
    // search all of them locally, in lockstep
    {
        const int nv = R / 2;                      // 16-byte vectors of keys per run
        for (int j = tid; j < (CSEL_CL - 1) * nv; j += CSEL_T) {
            const int r = j / nv, cr = r < c ? r : r + 1, q = j - r * nv;
            reinterpret_cast<ulonglong2 *>(ok_ + r * R)[q] =
                reinterpret_cast<const ulonglong2 *>(cl.map_shared_rank(sk, cr))[q];
        }
        const int nw = R / 4;                      // 16-byte vectors of indices per run
        for (int j = tid; j < (CSEL_CL - 1) * nw; j += CSEL_T) {
            const int r = j / nw, cr = r < c ? r : r + 1, q = j - r * nw;
            reinterpret_cast<uint4 *>(oi_ + r * R)[q] = reinterpret_cast<const uint4 *>(cl.map_shared_rank(si, cr))[q];
        }
    }
    for (int t = tid; t < R; t += CSEL_T) spos[t] = t;   // own position
    __syncthreads();
    {   // thread t searches for item t % R in the runs t / R, t / R + tpi, ...
        const int tpi = CSEL_T / R, it = tid % R, h = tid / R;
        const uint64_t ke = sk[it];
        const uint32_t ve = si[it];
        if (ve != 0xFFFFFFFFu) {                   // padding sorts last
            int lo[CSEL_RPT];
#pragma unroll
            for (int q = 0; q < CSEL_RPT; ++q) lo[q] = 0;
            // branch-free binary search for the first position not before (ke, ve)
            for (int half = R >> 1; half > 0; half >>= 1) {
#pragma unroll
                for (int q = 0; q < CSEL_RPT; ++q) {
                    const int r = h + q * tpi;
                    if (r < CSEL_CL - 1) {
                        const int m = lo[q] + half - 1;
                        if (kv_less(ok_[r * R + m], oi_[r * R + m], ke, ve)) lo[q] += half;
                    }
                }
            }
            int sum = 0;
#pragma unroll
            for (int q = 0; q < CSEL_RPT; ++q) {
                const int r = h + q * tpi;
                if (r < CSEL_CL - 1) {
                    if (lo[q] == R - 1 && kv_less(ok_[r * R + R - 1], oi_[r * R + R - 1], ke, ve)) lo[q] = R;
                    sum += lo[q];
                }
            }
            atomicAdd(spos + it, sum);
        }
    }
    __syncthreads();
    if (act && v != 0xFFFFFFFFu) {
        const int rank = spos[tid];
        PGA_DCHECK(rank >= 0 && rank < P && (int)v - base >= 0 && (int)v - base < R);
        if (what & 1) order[rank] = (int32_t)v;
        if (rank_out) rank_out[v] = rank;
        srank[v - base] = rank;
    }
    __syncthreads();
    if (!(what & 2)) {
        cl.sync();                                 // no CTA leaves while others read its runs
        return;
    }

    // (4) selection
    if (selection == PGA_SEL_TOURNAMENT) {
        for (int m = c * CSEL_T + tid; m < M; m += CSEL_CL * CSEL_T) {
            const U4 u = draw(seed, pga::TAG_TOUR, island, gen, (uint32_t)m, 0u);
            int best = (int)scale_u32(u.x, (uint32_t)P);
            for (int t = 1; t < tour_k; ++t) {
                const int cc = (int)scale_u32(word(u, t), (uint32_t)P);
                if (L[cc] > L[best] || (L[cc] == L[best] && cc < best)) best = cc;
            }
            sel[m] = best;
        }
        cl.sync();
        return;
    }
    // w_max: the globally first item (smallest key, then index) of the runs
    double wmax = 1.0;
    if (scaling != PGA_SCALE_RANK) {
        uint64_t bk = ~0ull;
        uint32_t bi = 0xFFFFFFFFu;
        for (int r = 0; r < CSEL_CL; ++r) {
            const uint64_t k_ = *cl.map_shared_rank(&s_first_key, r);
            const uint32_t i_ = *cl.map_shared_rank(&s_first_idx, r);
            if (kv_less(k_, i_, bk, bi)) {
                bk = k_;
                bi = i_;
            }
        }
        wmax = L[bi];
        if (wmax == 0.0) wmax = 0.0;
    }
    if (!(wmax > 0.0)) {                           // all-zero fitness: uniform fallback
        for (int m = c * CSEL_T + tid; m < M; m += CSEL_CL * CSEL_T) {
            const U4 u = draw(seed, pga::TAG_SUS, island, gen, (uint32_t)m, 0u);
            sel[m] = (int32_t)scale_u32(u.x, (uint32_t)P);
        }
        cl.sync();
        return;
    }
    const int B = 62 - ceil_log2_d(P);
    uint64_t qi = 0;
    if (act && base + tid < P) {
        const double w = (scaling == PGA_SCALE_RANK) ? 1.0 / sqrt((double)(srank[tid] + 1)) : sL[tid];
        const double x = w / wmax;
        if (x > 0.0) qi = (uint64_t)floor(ldexp(x, B));
    }
    uint64_t incl = qi;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) ws[wid] = incl;
    __syncthreads();
    uint64_t wbase = 0;
    for (int kk = 0; kk < wid; ++kk) wbase += ws[kk];
    if (tid == CSEL_T - 1) s_tot = wbase + incl;   // the CTA's total
    cl.sync();                                     // totals visible
    uint64_t cbase = 0, Q = 0;
    for (int r = 0; r < CSEL_CL; ++r) {
        const uint64_t t_ = *cl.map_shared_rank(&s_tot, r);
        Q += t_;
        if (r < c) cbase += t_;
    }
    if (act && base + tid < P) {
        const uint64_t step = Q / (uint64_t)M;
        const U4 u = draw(seed, pga::TAG_SUS, island, gen, 0u, 0xFFFFFFFFu);
        const uint64_t x = ((uint64_t)u.x << 32) | (uint64_t)u.y;
        const uint64_t start = __umul64hi(x, step);
        const uint64_t hi = cbase + wbase + incl, lo = hi - qi;
        const int64_t m0 = (int64_t)min(sus_first(lo, start, step), (uint64_t)M);
        const int64_t m1 = (int64_t)min(sus_first(hi, start, step), (uint64_t)M);
        for (int64_t m = m0; m < m1; ++m) sel[m] = base + tid;
    }
    cl.sync();                                     // no CTA leaves while others read its totals
}

static size_t select_small_smem() {
    using BRS = cub::BlockRadixSort<uint64_t, SMALL_T, SMALL_P / SMALL_T, uint32_t>;
    const size_t a = (size_t)SMALL_P * 8 > sizeof(typename BRS::TempStorage) ? (size_t)SMALL_P * 8
                                                                             : sizeof(typename BRS::TempStorage);
    return a + (size_t)SMALL_P * (8 + 4 + 4) + (size_t)SMALL_T * 8;   // + bitonic key scratch
}

// ---------------------------------------------------------------------------
// k_breed: warp per output slot o.  o < E: copy elite order[o];
// else child c of pair k = (o - E) / 2.  Crossover, mutation, canonicalise,
// write both layouts (and an optional int32 copy for the test hook).
// ---------------------------------------------------------------------------
struct BreedArgs {
    const uint16_t *cm_in0, *cm_in1;   // parents (chromosome-major), by gen parity
    uint16_t *cm_out0, *cm_out1;       // children written to the other buffer
    uint16_t *gm_out0, *gm_out1;
    const int32_t *i32_in;             // hook: int32 parents [P][N] (instead of cm_in)
    int32_t *i32_out;                  // hook: int32 children [P][N]
    const uint16_t *top16;             // KB top labels (0xFFFF none)
    const int32_t *top32;              // hook: int32 tops (-1 none)
    const int32_t *order, *sel, *sigma;
    int64_t P, Pcap, p_off;
    int N, ldn, E;
    uint64_t thr_c, thr_m, thr_kb;
    uint64_t seed;
    uint32_t gen, island;
    const int32_t *done, *gen_ptr;
    const int32_t *gm_skip;            // != 0: the label-sparse pass owns the gene-major copy (f2)
    RoundKeys rk;                      // Philox round keys of `seed` (in the parameter constant bank)
    const uint32_t *mmask;             // GA, P > SMALL_GA_P: precomputed mutation masks [Pcap][mw] (k_mutmask)
    int mw;                            // words per child: ceil(N / 32)
    pga::DevState *adv_st;             // GA: advance st->gen once the grid is done (null: hooks)
    uint32_t *adv_ctr;                 // CTA counter for that (reset by the last CTA)
};

// The generation counter advances once the whole breed grid is done: the
// last CTA to finish does it (every CTA read the generation at its start),
// which replaces a separate one-thread k_advance launch.
__device__ __forceinline__ void breed_advance(const BreedArgs &a) {
    if (!a.adv_st) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(a.adv_ctr, 1u) == gridDim.x - 1) {
            *a.adv_ctr = 0u;
            if (!a.adv_st->done) a.adv_st->gen += 1;
        }
    }
}


__device__ __forceinline__ int parent_top(const BreedArgs &a, int64_t p) {
    if (a.top32) return a.top32[p];
    const uint16_t t = a.top16[p];
    return t == 0xFFFF ? -1 : (int)t;
}

// CTA = BW warps x BC children (BS = BW*BC consecutive output slots).  Genes
// are processed in chunks of 128: each lane draws ONE Philox block for 4
// consecutive genes (the oracle's layout Philox(MUT; i>>2, o)[i&3]) and the
// 4-bit mutation mask is redistributed with one shuffle per 32 genes; the
// children's canonical genes go to CM directly (coalesced) and through a
// shared-memory tile [128][BS] to the gene-major layout (BS*2-byte rows).
constexpr int BW = 16, BC = 1, BS = BW * BC, GCH = 128;
constexpr int TS = BS + 2;   // tile row stride (u16): 36 B, odd multiple of 4 B -> conflict-free

struct ChildPlan {
    int64_t pa, pb;
    int mode, kb_top, cut;
    bool mutate, valid;
    uint32_t og;
};

__device__ __forceinline__ ChildPlan plan_child(const BreedArgs &a, int64_t o, uint32_t gen) {
    ChildPlan c{};
    c.valid = o < a.P;
    if (!c.valid) return c;
    c.og = (uint32_t)(a.p_off + o);
    if (o < a.E) {
        c.pa = a.order[o];
        c.mode = 0;
        c.mutate = false;
        return c;
    }
    const int64_t k = (o - a.E) >> 1;
    const int child = (int)((o - a.E) & 1);
    const int64_t ia = a.sel[a.sigma[2 * k]], ib = a.sel[a.sigma[2 * k + 1]];
    c.pa = child ? ib : ia;   // the parent whose genes the child keeps
    c.pb = child ? ia : ib;   // the other parent
    const U4 x = draw_rk(a.rk, pga::TAG_XO, a.island, gen, (uint32_t)k, 0u);
    c.kb_top = -1;
    if ((uint64_t)x.x >= a.thr_c) {
        c.mode = 0;
    } else if ((uint64_t)x.y < a.thr_kb) {
        c.mode = 1;
        c.kb_top = parent_top(a, c.pb);
    } else {
        c.mode = 2;
        c.cut = 1 + (int)scale_u32(x.z, (uint32_t)(a.N - 1));
    }
    c.mutate = a.thr_m != 0;
    return c;
}

template <bool HOOK>
__global__ void __launch_bounds__(BW * 32, 3) k_breed(BreedArgs a) {
    pdl_wait();
    pdl_trigger();
    if (a.done && *a.done) return;
    extern __shared__ uint16_t sm16[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int N = a.N;
    const uint32_t gen = a.gen_ptr ? (uint32_t)*a.gen_ptr : a.gen;
    const int par = a.gen_ptr ? (int)(gen & 1u) : 0;
    const uint16_t *cm_in = par ? a.cm_in1 : a.cm_in0;
    uint16_t *cm_out = par ? a.cm_out0 : a.cm_out1;
    uint16_t *gm_out = par ? a.gm_out0 : a.gm_out1;
    uint16_t *tile = sm16;                               // 2 x [GCH][TS]
    uint16_t *tables = sm16 + 2 * GCH * TS;              // [BS][N+1]
    const int64_t o0 = (int64_t)blockIdx.x * BS;

    ChildPlan cp[BC];
    Canon cn[BC];
#pragma unroll
    for (int c = 0; c < BC; ++c) {
        const int slot = warp * BC + c;
        cp[c] = plan_child(a, o0 + slot, gen);
        cn[c].table = tables + (size_t)slot * breed_tab(N);
        cn[c].next = 0;
        table_reset16(cn[c].table, N + 1, lane);
    }
    for (int base = 0; base < N; base += GCH) {
        const int tb = ((base / GCH) & 1) * GCH * TS;     // double-buffered tile
#pragma unroll
        for (int c = 0; c < BC; ++c) {
            const ChildPlan &p = cp[c];
            const int slot = warp * BC + c;
            // batch this chunk's parent loads (memory-level parallelism)
            uint32_t ga[GCH / 32], gb[GCH / 32];
#pragma unroll
            for (int sc = 0; sc < GCH / 32; ++sc) {
                const int i = base + 32 * sc + lane;
                const bool valid = p.valid && i < N;
                if (HOOK) {
                    ga[sc] = valid ? (uint32_t)a.i32_in[p.pa * N + i] : 0u;
                    gb[sc] = (valid && p.mode != 0) ? (uint32_t)a.i32_in[p.pb * N + i] : 0u;
                } else {
                    ga[sc] = valid ? (uint32_t)cm_in[p.pa * a.ldn + i] : 0u;
                    gb[sc] = (valid && p.mode != 0) ? (uint32_t)cm_in[p.pb * a.ldn + i] : 0u;
                }
            }
            // mutation mask of genes base+4*lane .. base+4*lane+3
            uint32_t mbits = 0;
            if (p.valid && p.mutate && base + 4 * lane < N) {
                if (a.mmask) {
                    const uint32_t wv = a.mmask[(o0 + slot) * a.mw + (base >> 5) + (lane >> 3)];
                    mbits = (wv >> (4 * (lane & 7))) & 0xFu;
                } else {
                    const U4 u = draw_rk(a.rk, pga::TAG_MUT, a.island, gen, (uint32_t)((base >> 2) + lane), p.og);
                    mbits = ((uint64_t)u.x < a.thr_m ? 1u : 0u) | ((uint64_t)u.y < a.thr_m ? 2u : 0u) |
                            ((uint64_t)u.z < a.thr_m ? 4u : 0u) | ((uint64_t)u.w < a.thr_m ? 8u : 0u);
                }
            }
            uint32_t sv[GCH / 32];
            unsigned mm[GCH / 32];
#pragma unroll
            for (int sc = 0; sc < GCH / 32; ++sc) {
                const int i = base + 32 * sc + lane;
                const bool valid = p.valid && i < N;
                const uint32_t mb = __shfl_sync(0xFFFFFFFFu, mbits, 8 * sc + (lane >> 2));
                uint32_t s = ga[sc];
                if (p.mode == 1) {
                    if (p.kb_top >= 0 && (int)gb[sc] == p.kb_top) s = (uint32_t)N;
                } else if (p.mode == 2) {
                    if (i >= p.cut) s = gb[sc];
                }
                if (valid && ((mb >> (lane & 3)) & 1u)) {
                    const U4 v = draw_rk(a.rk, pga::TAG_MUTV, a.island, gen, (uint32_t)(i >> 2), p.og);
                    s = scale_u32(word(v, i & 3), (uint32_t)N);
                }
                sv[sc] = s;
            }
            // the four group masks are independent: issue them back to back
#pragma unroll
            for (int sc = 0; sc < GCH / 32; ++sc) {
                const bool valid = p.valid && base + 32 * sc + lane < N;
                mm[sc] = __match_any_sync(0xFFFFFFFFu, valid ? sv[sc] : (0x10000u + (uint32_t)lane));
            }
#pragma unroll
            for (int sc = 0; sc < GCH / 32; ++sc) {
                const int i = base + 32 * sc + lane;
                const bool valid = p.valid && i < N;
                const uint32_t cv = cn[c].assign(sv[sc], valid, lane, mm[sc]);
                if (valid) {
                    if (HOOK) a.i32_out[(o0 + slot) * N + i] = (int32_t)cv;
                    else cm_out[(o0 + slot) * a.ldn + i] = (uint16_t)cv;
                }
                if (!HOOK) tile[tb + (32 * sc + lane) * TS + slot] = (uint16_t)cv;
            }
        }
        __syncthreads();     // tile[tb] complete; the other half is free again
        if (!HOOK) {
            // gene-major rows: genes base..base+127, slots o0..o0+BS-1
            for (int e = threadIdx.x; e < GCH * (BS / 2); e += BW * 32) {
                const int g = e / (BS / 2), pr = e - g * (BS / 2);
                const int i = base + g;
                const int64_t o = o0 + 2 * pr;
                if (i < N && o < a.P) {
                    const uint32_t two = *reinterpret_cast<const uint32_t *>(&tile[tb + g * TS + 2 * pr]);
                    if (o + 1 < a.P) *reinterpret_cast<uint32_t *>(&gm_out[(int64_t)i * a.Pcap + o]) = two;
                    else gm_out[(int64_t)i * a.Pcap + o] = (uint16_t)(two & 0xFFFF);
                }
            }
        }
    }
    breed_advance(a);
}

// ---------------------------------------------------------------------------
// k_breed2 (N <= BREED2_MAXN): the same operators and outputs as k_breed with
// a canonicalisation that has no dependency chain across gene chunks, and the
// child's labels held in registers from crossover to the store.  Lane l owns
// the gene pairs (128 b + 64 h + 2 l, +1) of its warp's child (NB = ceil(N /
// 128) chunks b, h = 0, 1: one 32-bit word per pair).
// Phase 1: crossover + mutation -> pre-canonical pair words.
// Phase 2 (canonical form, Q7): (a) first-occurrence positions fp[v] = min i
// by shared atomicMin (order-free, so no chunk waits on another); (b) per
// 64-gene group G two ballots (even / odd genes) mark the genes i with
// fp[s_i] == i, and a running count gives each group's base; (c) canonical(s_i)
// = rank of f = fp[s_i] among the first occurrences = base[G'] + firsts of
// group G' = f >> 6 below f (even genes with lane <= / < (f >> 1) & 31,
// odd genes with lane <).  The canonical pair is one 32-bit store.
// Phase 3 (dense mode only) writes the gene-major rows of the CTA's 16
// children through the shared tile.
// ---------------------------------------------------------------------------
constexpr int BREED2_MAXN = 1024;
#ifndef PGA_B2_MINB
#define PGA_B2_MINB 2
#endif

__host__ __device__ __forceinline__ int breed2_ngrp(int N) { return (N + 63) / 64; }

// tile rows padded to whole 128-gene chunks
__host__ __device__ __forceinline__ int breed2_rows(int N) { return (N + GCH - 1) / GCH * GCH; }

static size_t breed2_smem(int N) {
    const size_t tile = (size_t)breed2_rows(N) * TS * sizeof(uint16_t);
    const size_t fp = (size_t)BS * ((N + 1 + 3) & ~3) * sizeof(uint32_t);
    const size_t grp = (size_t)BS * breed2_ngrp(N) * sizeof(uint4);
    return ((tile + 15) & ~(size_t)15) + ((fp + 15) & ~(size_t)15) + grp + 16;
}

template <bool HOOK, int NB>
__global__ void __launch_bounds__(BW * 32, NB <= 2 ? 3 : PGA_B2_MINB) k_breed2(BreedArgs a) {
    pdl_wait();
    pdl_trigger();
    if (a.done && *a.done) return;
    extern __shared__ __align__(16) unsigned char sm2[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int N = a.N;
    const uint32_t gen = a.gen_ptr ? (uint32_t)*a.gen_ptr : a.gen;
    const int par = a.gen_ptr ? (int)(gen & 1u) : 0;
    const uint16_t *cm_in = par ? a.cm_in1 : a.cm_in0;
    uint16_t *cm_out = par ? a.cm_out0 : a.cm_out1;
    uint16_t *gm_out = par ? a.gm_out0 : a.gm_out1;
    uint16_t *tile = reinterpret_cast<uint16_t *>(sm2);                               // [rows][TS]
    const size_t tile_b = ((size_t)breed2_rows(N) * TS * sizeof(uint16_t) + 15) & ~(size_t)15;
    const int fpn = (N + 1 + 3) & ~3;
    uint32_t *fp = reinterpret_cast<uint32_t *>(sm2 + tile_b) + (size_t)warp * fpn;    // [BS][fpn]
    const size_t fp_b = ((size_t)BS * fpn * sizeof(uint32_t) + 15) & ~(size_t)15;
    uint4 *grp = reinterpret_cast<uint4 *>(sm2 + tile_b + fp_b) + (size_t)warp * breed2_ngrp(N);  // {even, odd, base, -}
    const int64_t o0 = (int64_t)blockIdx.x * BS;
    const int slot = warp;
    const int64_t o = o0 + slot;
    // precomputed mutation-mask words (k_mutmask) depend only on the child
    // index: their loads are issued before the plan's dependent chain
    // (sigma -> sel -> parent labels) instead of after it
    uint32_t mwv[NB];
    {
        const bool mw_on = a.mmask && o < a.P && o >= a.E && a.thr_m != 0;
#pragma unroll
        for (int b = 0; b < NB; ++b)
            mwv[b] = (mw_on && GCH * b + 4 * lane < N) ? a.mmask[o * a.mw + ((GCH * b) >> 5) + (lane >> 3)] : 0u;
    }
    const ChildPlan p = plan_child(a, o, gen);

    // ---- phase 1: crossover + mutation -> pre-canonical pair words.  Both
    // mutation bits of a pair come from one shuffle, and there is at most one
    // MUTV block per pair (both genes share Philox block (g >> 2)).
    uint32_t w[NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int b0 = GCH * b;
        uint32_t ga[2], gb[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g0 = b0 + 64 * h + 2 * lane;
            const bool v0 = p.valid && g0 < N, v1 = p.valid && g0 + 1 < N;
            if (HOOK) {
                ga[h] = (v0 ? (uint32_t)a.i32_in[p.pa * N + g0] : 0u) |
                        ((v1 ? (uint32_t)a.i32_in[p.pa * N + g0 + 1] : 0u) << 16);
                gb[h] = (p.mode != 0) ? ((v0 ? (uint32_t)a.i32_in[p.pb * N + g0] : 0u) |
                                         ((v1 ? (uint32_t)a.i32_in[p.pb * N + g0 + 1] : 0u) << 16)) : 0u;
            } else {
                // ldn is even and g0 is even: the pair is one aligned 32-bit word
                ga[h] = v0 ? *reinterpret_cast<const uint32_t *>(cm_in + p.pa * a.ldn + g0) : 0u;
                gb[h] = (v0 && p.mode != 0) ? *reinterpret_cast<const uint32_t *>(cm_in + p.pb * a.ldn + g0) : 0u;
            }
        }
        uint32_t mbits = 0;
        if (p.valid && p.mutate && b0 + 4 * lane < N) {
            if (a.mmask) {   // precomputed on the side stream (k_mutmask)
                mbits = (mwv[b] >> (4 * (lane & 7))) & 0xFu;
            } else {
                const U4 u = draw_rk(a.rk, pga::TAG_MUT, a.island, gen, (uint32_t)((b0 >> 2) + lane), p.og);
                mbits = ((uint64_t)u.x < a.thr_m ? 1u : 0u) | ((uint64_t)u.y < a.thr_m ? 2u : 0u) |
                        ((uint64_t)u.z < a.thr_m ? 4u : 0u) | ((uint64_t)u.w < a.thr_m ? 8u : 0u);
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g0 = b0 + 64 * h + 2 * lane;
            const uint32_t mb = (__shfl_sync(0xFFFFFFFFu, mbits, 16 * h + (lane >> 1)) >> (2 * (lane & 1))) & 3u;
            uint32_t s[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = g0 + e;
                uint32_t x = (ga[h] >> (16 * e)) & 0xFFFFu;
                const uint32_t y = (gb[h] >> (16 * e)) & 0xFFFFu;
                if (p.mode == 1) {
                    if (p.kb_top >= 0 && (int)y == p.kb_top) x = (uint32_t)N;
                } else if (p.mode == 2) {
                    if (i >= p.cut) x = y;
                }
                s[e] = x;
            }
            if (p.valid && mb) {
                const U4 v = draw_rk(a.rk, pga::TAG_MUTV, a.island, gen, (uint32_t)(g0 >> 2), p.og);
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if ((mb >> e) & 1u) s[e] = scale_u32(word(v, (g0 + e) & 3), (uint32_t)N);
            }
            w[b][h] = s[0] | (s[1] << 16);
        }
    }

    // ---- phase 2: canonical form (Q7), no chain across chunks
    const bool gm = !HOOK && !(a.gm_skip && *a.gm_skip);   // dense mode: gene-major rows wanted
    if (p.valid) {
        {                                             // (a) first occurrences: fp[v] = min i
            uint4 *f4 = reinterpret_cast<uint4 *>(fp);
            const uint4 inf = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
            for (int k = lane; k < fpn / 4; k += 32) f4[k] = inf;
            __syncwarp();
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int g0 = GCH * b + 64 * h + 2 * lane;
                    PGA_DCHECK((w[b][h] & 0xFFFFu) <= (uint32_t)N && (w[b][h] >> 16) <= (uint32_t)N);
                    if (g0 < N) atomicMin(&fp[w[b][h] & 0xFFFFu], (uint32_t)g0);
                    if (g0 + 1 < N) atomicMin(&fp[w[b][h] >> 16], (uint32_t)(g0 + 1));
                }
            __syncwarp();
        }
        uint32_t run = 0;
#pragma unroll
        for (int b = 0; b < NB; ++b)                  // (b) first-occurrence ballots, group bases
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int G = 2 * b + h, g0 = 64 * G + 2 * lane;
                if (64 * G >= N) continue;            // warp-uniform
                const bool f0 = g0 < N && fp[w[b][h] & 0xFFFFu] == (uint32_t)g0;
                const bool f1 = g0 + 1 < N && fp[w[b][h] >> 16] == (uint32_t)(g0 + 1);
                const unsigned be = __ballot_sync(0xFFFFFFFFu, f0), bo = __ballot_sync(0xFFFFFFFFu, f1);
                if (lane == 0) grp[G] = make_uint4(be, bo, run, 0u);
                run += (uint32_t)(__popc(be) + __popc(bo));
            }
        __syncwarp();
#pragma unroll
        for (int b = 0; b < NB; ++b)                  // (c) canonical labels
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int g0 = GCH * b + 64 * h + 2 * lane;
                if (g0 >= N) continue;
                uint32_t cv[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const uint32_t f = (g0 + e < N) ? fp[(w[b][h] >> (16 * e)) & 0xFFFFu] : 0u;
                    const uint4 gr = grp[f >> 6];
                    const uint32_t l = (f >> 1) & 31u, below = (1u << l) - 1u;
                    cv[e] = gr.z + __popc(gr.x & (below | ((f & 1u) << l))) + __popc(gr.y & below);
                }
                if (g0 + 1 >= N) cv[1] = 0u;
                if (HOOK) {
                    a.i32_out[o * N + g0] = (int32_t)cv[0];
                    if (g0 + 1 < N) a.i32_out[o * N + g0 + 1] = (int32_t)cv[1];
                } else {
                    *reinterpret_cast<uint32_t *>(cm_out + o * a.ldn + g0) = cv[0] | (cv[1] << 16);
                    if (gm) {
                        tile[g0 * TS + slot] = (uint16_t)cv[0];
                        tile[(g0 + 1) * TS + slot] = (uint16_t)cv[1];   // rows >= N are padding
                    }
                }
            }
    }
    if (gm) {   // sparse mode: k_fitness_sparse transposes dense blocks itself
        __syncthreads();
        // ---- phase 3: gene-major rows (BS children = 32 B per gene)
        for (int e = threadIdx.x; e < N * (BS / 2); e += BW * 32) {
            const int i = e / (BS / 2), pr = e - i * (BS / 2);
            const int64_t oo = o0 + 2 * pr;
            if (oo < a.P) {
                const uint32_t two = *reinterpret_cast<const uint32_t *>(&tile[i * TS + 2 * pr]);
                if (oo + 1 < a.P) *reinterpret_cast<uint32_t *>(&gm_out[(int64_t)i * a.Pcap + oo]) = two;
                else gm_out[(int64_t)i * a.Pcap + oo] = (uint16_t)(two & 0xFFFF);
            }
        }
    }
    breed_advance(a);
}

// one instantiation per chunk count NB = ceil(N / 128) (labels stay in registers)
template <bool HOOK>
static cudaError_t launch_breed2(const BreedArgs &a, int64_t P, int N, cudaStream_t s) {
    const unsigned grid = (unsigned)((P + BS - 1) / BS);
    const size_t sm = breed2_smem(N);
    switch ((N + GCH - 1) / GCH) {
#define PGA_B2(nb) case nb: return pga::launch_pdl(k_breed2<HOOK, nb>, dim3(grid), dim3(BW * 32), sm, s, a);
        PGA_B2(1) PGA_B2(2) PGA_B2(3) PGA_B2(4) PGA_B2(5) PGA_B2(6) PGA_B2(7) PGA_B2(8)
#undef PGA_B2
    }
    return cudaErrorInvalidValue;
}

template <bool HOOK>
static cudaError_t prepare_breed2(int N) {
    const int sm = (int)breed2_smem(N);
    switch ((N + GCH - 1) / GCH) {
#define PGA_B2(nb) case nb: return cudaFuncSetAttribute(k_breed2<HOOK, nb>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        PGA_B2(1) PGA_B2(2) PGA_B2(3) PGA_B2(4) PGA_B2(5) PGA_B2(6) PGA_B2(7) PGA_B2(8)
#undef PGA_B2
    }
    return cudaSuccess;
}

// k_set_pop: int32 1-based labels (validated on the host) -> canonical
// u16 in both layouts of buffer `par`.
__global__ void k_set_pop(const int32_t *__restrict__ lab, int64_t P, int N, int ldn, int64_t Pcap,
                          uint16_t *CM, uint16_t *GM) {
    extern __shared__ uint16_t tables[];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t p = (int64_t)blockIdx.x * nw + warp;
    if (p >= P) return;
    uint16_t *table = tables + (size_t)warp * (N + 1);
    table_reset(table, N + 1, lane);
    Canon cn{table, 0};
    for (int base = 0; base < N; base += 32) {
        const int i = base + lane;
        const bool valid = i < N;
        const uint32_t s = valid ? (uint32_t)(lab[p * N + i] - 1) : 0u;
        const uint32_t c = cn.step(s, valid, lane);
        if (valid) {
            CM[p * ldn + i] = (uint16_t)c;
            GM[(int64_t)i * Pcap + p] = (uint16_t)c;
        }
    }
}


// ---------------------------------------------------------------------------
// migration (Q21).  Record: fp64 L | u16 top | u16 pad[3] | u16 labels[N],
// padded to a multiple of 16 bytes.
// ---------------------------------------------------------------------------
__global__ void k_export(const double *__restrict__ L, const uint16_t *__restrict__ top,
                         const int32_t *__restrict__ order, const uint16_t *CM0,
                         const uint16_t *CM1, const pga::DevState *st, int ldn, int N, int Em,
                         int64_t rec_bytes, unsigned char *out) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x;
    if (r >= Em || st->done) return;   // stopped: the population is final (every island agrees, Q28)
    const uint16_t *CM = (st->gen & 1) ? CM1 : CM0;
    const int p = order[r];
    unsigned char *rec = out + (int64_t)r * rec_bytes;
    if (threadIdx.x == 0) {
        *reinterpret_cast<double *>(rec) = L[p];
        reinterpret_cast<uint16_t *>(rec + 8)[0] = top[p];
    }
    uint16_t *lab = reinterpret_cast<uint16_t *>(rec + 16);
    for (int i = threadIdx.x; i < N; i += blockDim.x) lab[i] = CM[(int64_t)p * ldn + i];
}

// one block: choose the global top Em of G*Em candidates by (L desc, island
// asc, rank asc), then replace this island's Em worst (order[P-1-r]).
__global__ void k_import(const unsigned char *__restrict__ in, int G, int Em, int64_t rec_bytes,
                         const int32_t *__restrict__ order, int64_t P, double *L, uint16_t *top,
                         uint16_t *CM0, uint16_t *CM1, uint16_t *GM0, uint16_t *GM1,
                         const pga::DevState *st, int ldn, int N, int64_t Pcap) {
    __shared__ int chosen[256];
    pdl_wait();
    pdl_trigger();
    if (st->done) return;   // stopped: the population is final (every island agrees, Q28)
    const int total = G * Em;
    if (threadIdx.x == 0) {
        // selection by repeated scans (total <= 8 * 256); strict '>' keeps
        // the earliest (island, rank) among equal L.
        unsigned char used[2048];
        for (int j = 0; j < total; ++j) used[j] = 0;
        for (int r = 0; r < Em; ++r) {
            int b = -1;
            double bl = 0.0;
            for (int j = 0; j < total; ++j) {
                if (used[j]) continue;
                const double v = *reinterpret_cast<const double *>(in + (int64_t)j * rec_bytes);
                if (b < 0 || v > bl) {
                    b = j;
                    bl = v;
                }
            }
            used[b] = 1;
            chosen[r] = b;
        }
    }
    __syncthreads();
    const int par = st->gen & 1;
    uint16_t *CM = par ? CM1 : CM0;
    uint16_t *GM = par ? GM1 : GM0;
    for (int r = 0; r < Em; ++r) {
        const unsigned char *rec = in + (int64_t)chosen[r] * rec_bytes;
        const int64_t w = order[P - 1 - r];
        const uint16_t *lab = reinterpret_cast<const uint16_t *>(rec + 16);
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            CM[w * ldn + i] = lab[i];
            GM[(int64_t)i * Pcap + w] = lab[i];
        }
        if (threadIdx.x == 0) {
            L[w] = *reinterpret_cast<const double *>(rec);
            top[w] = reinterpret_cast<const uint16_t *>(rec + 8)[0];
        }
    }
}

}  // namespace

PGA_VIOL_READER(viol_ga)

namespace pga {

// k_select_cluster can be co-scheduled on this device (prepare_select_small)
static bool g_csel_ok = false;

// A/B switches for measurement: getenv_flag(name, d) is d unless the variable
// is set (then true for "1", false for "0").
static bool getenv_flag(const char *name, bool d) {
    const char *e = std::getenv(name);
    if (!e || !e[0]) return d;
    return e[0] != '0';
}

// Mutation masks precomputed on the side stream, beside the fitness pass,
// only while that pass leaves SMs idle (P <= MUTMASK_MAXP: an 8-GPU island of
// C4).  At C4's P = 65536 the pass fills the GPU and the mask kernel steals its
// issue slots: 0.5498 vs 0.5285 ms per generation (breed -11 us, sparse pass
// +31 us); at P = 8192 0.1315 vs 0.1328 ms.  PGA_NO_MUTMASK=1 / =0 forces it.
constexpr int64_t MUTMASK_MAXP = 8192;
static bool mutmask_use(int64_t P) { return getenv_flag("PGA_MUTMASK_FORCE", false) || (P <= MUTMASK_MAXP && !getenv_flag("PGA_NO_MUTMASK", false)); }

static size_t breed_smem(int N) { return ((size_t)2 * GCH * TS + (size_t)BS * breed_tab(N)) * sizeof(uint16_t); }

static int breed_warps(int N) {
    const size_t per = (size_t)(N + 1) * sizeof(uint16_t);
    int w = (int)((48 * 1024) / per);
    return w < 1 ? 1 : (w > 8 ? 8 : w);
}

int launch_canonicalize_i32(int32_t *lab, int64_t P, int32_t N, cudaStream_t s) {
    const int tab = 2 * N + 1;
    int w = (int)((48 * 1024) / ((size_t)tab * 2));
    w = w < 1 ? 1 : (w > 8 ? 8 : w);
    k_canon_i32<<<(unsigned)((P + w - 1) / w), 32 * w, (size_t)w * tab * 2, s>>>(lab, P, N, tab);
    PGA_LAUNCHED();
    return PGA_OK;
}

int launch_init_raw(uint64_t seed, int N, int ldn, int64_t P, int64_t Pcap, int64_t p_off,
                    uint32_t island, uint16_t *CM, uint16_t *GM, int32_t *out32, cudaStream_t s) {
    const int w = breed_warps(N);
    k_init<<<(unsigned)((P + w - 1) / w), 32 * w, (size_t)w * (N + 1) * 2, s>>>(
        seed, N, ldn, P, Pcap, p_off, island, CM, GM, out32);
    PGA_LAUNCHED();
    return PGA_OK;
}

int prepare_breed(int N) {
    PGA_CUDA(cudaFuncSetAttribute(k_breed<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)breed_smem(N)));
    PGA_CUDA(cudaFuncSetAttribute(k_breed<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)breed_smem(N)));
    if (N <= BREED2_MAXN) {
        PGA_CUDA(prepare_breed2<true>(N));
        PGA_CUDA(prepare_breed2<false>(N));
    }
    return PGA_OK;
}

int launch_set_pop(pga_ctx *c, const int32_t *lab32, int par, cudaStream_t s) {
    const int w = breed_warps(c->N);
    k_set_pop<<<(unsigned)((c->P + w - 1) / w), 32 * w, (size_t)w * (c->N + 1) * 2, s>>>(
        lab32, c->P, c->N, c->ldn, c->Pcap, c->pop[par], c->popT[par]);
    PGA_LAUNCHED();
    return PGA_OK;
}

int launch_init(pga_ctx *c, uint64_t seed, cudaStream_t s) {
    return launch_init_raw(seed, c->N, c->ldn, c->P, c->Pcap, (int64_t)c->p.island * c->P,
                           (uint32_t)c->p.island, c->pop[0], c->popT[0], nullptr, s);
}

int launch_stats(pga_ctx *c, int mode, cudaStream_t s) {
    int64_t g = (c->P + STATS_PER_CTA - 1) / STATS_PER_CTA;
    if (g > STATS_MAXG) g = STATS_MAXG;
    const int64_t per = (c->P + g - 1) / g;
    PGA_LAUNCH_PDL(k_stats, dim3((unsigned)g), dim3(STATS_T), 0, s, (const double *)c->L, c->P,
                   (const uint16_t *)c->pop[0], (const uint16_t *)c->pop[1], (int)c->ldn, (int)c->N, c->st,
                   c->best_labels, c->history, (int)c->hist_cap, c->p.tol, (int)c->p.stall_gens,
                   (int)c->p.max_gens, mode, (int)c->p.migrate_every, c->stats_part, c->stats_ctr, per);
    return PGA_OK;
}

// order = indices by (L desc, idx asc); rank[i] = position of individual i
static int sort_order(const double *L, int64_t P, int32_t *order, int32_t *rank, uint64_t *keys_in,
                      uint64_t *keys_out, int32_t *idx_in, int32_t *idx_tmp, const int32_t *done,
                      cudaStream_t s) {
    const int nruns = (int)((P + RUN - 1) / RUN);
    uint64_t *kA = keys_out, *kB = keys_in;
    int32_t *iA = idx_in, *iB = idx_tmp;
    PGA_LAUNCH_PDL(k_sort_runs, dim3(nruns), dim3(RUN_T), 0, s, L, P, kA, iA, done);
    const unsigned nb = (unsigned)((P + MERGE_T - 1) / MERGE_T);
    if (nruns == 1) {   // one run: copy its indices out through a width-P "merge"
        PGA_LAUNCH_PDL(k_merge_level<2>, dim3(nb), dim3(MERGE_T), 0, s, (const uint64_t *)kA, (const int32_t *)iA,
                       P, P, (uint64_t *)nullptr, order, rank, done);
        return PGA_OK;
    }
    // 4-way levels while two more doublings are needed, a 2-way level last
    // (P = 65536: three levels instead of six)
    for (int64_t w = RUN; w < P;) {
        const int way = (2 * w < P) ? 4 : 2;
        const bool last = (int64_t)way * w >= P;
        if (way == 4)
            PGA_LAUNCH_PDL(k_merge_level<4>, dim3(nb), dim3(MERGE_T), 0, s, (const uint64_t *)kA,
                           (const int32_t *)iA, P, w, last ? (uint64_t *)nullptr : kB, last ? order : iB,
                           last ? rank : (int32_t *)nullptr, done);
        else
            PGA_LAUNCH_PDL(k_merge_level<2>, dim3(nb), dim3(MERGE_T), 0, s, (const uint64_t *)kA,
                           (const int32_t *)iA, P, w, last ? (uint64_t *)nullptr : kB, last ? order : iB,
                           last ? rank : (int32_t *)nullptr, done);
        w *= way;
        uint64_t *tk = kA;
        kA = kB;
        kB = tk;
        int32_t *ti = iA;
        iA = iB;
        iB = ti;
    }
    return PGA_OK;
}

int prepare_select_small() {
    PGA_CUDA(cudaFuncSetAttribute(k_select_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)select_small_smem()));
    PGA_CUDA(cudaFuncSetAttribute(k_select_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)csel_smem(CSEL_MAXR)));
    PGA_CUDA(cudaFuncSetAttribute(k_select_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    {   // can a 16-CTA cluster of this size be co-scheduled on this device?  If
        // not (a smaller part, MIG), the multi-kernel path serves these P.
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(CSEL_CL);
        cfg.blockDim = dim3(CSEL_T);
        cfg.dynamicSmemBytes = csel_smem(CSEL_MAXR);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CSEL_CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = 0;
        g_csel_ok = cudaOccupancyMaxActiveClusters(&nc, k_select_cluster, &cfg) == cudaSuccess && nc > 0;
        (void)cudaGetLastError();
    }
    return PGA_OK;
}

// order/rank (what & 1) and/or selection + mates (what & 2) in one cluster
// launch, SMALL_GA_P < P <= CSEL_MAXP
static int launch_select_cluster(int what, const double *L, int64_t P, const pga_params &p,
                                 const int32_t *gen_ptr, int32_t *order, int32_t *rank, int32_t *sel,
                                 const int32_t *done, cudaStream_t s) {
    const int64_t M = 2 * ((P - p.elite + 1) / 2);
    const int R = csel_run((int)P);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CSEL_CL);
    cfg.blockDim = dim3(CSEL_T);
    cfg.dynamicSmemBytes = csel_smem(R);
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CSEL_CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    count_launch();
    PGA_CUDA(cudaLaunchKernelEx(&cfg, k_select_cluster, what, L, (int)P, R, (int)M, (int)p.selection,
                                (int)p.tournament_k, (int)p.scaling, p.seed, (uint32_t)0, (uint32_t)p.island,
                                gen_ptr, order, rank, sel, done));
    return PGA_OK;
}

// order (what & 1) and/or selection + mates (what & 2) for P <= SMALL_P
int launch_select_small(int what, const double *L, int64_t P, const pga_params &p, int32_t gen,
                        int32_t island, const int32_t *gen_ptr, int32_t *order, int32_t *sel,
                        int32_t *sigma, const int32_t *done, cudaStream_t s) {
    const int64_t M = 2 * ((P - p.elite + 1) / 2);
    PGA_LAUNCH_PDL(k_select_small, dim3(1), dim3(SMALL_T), select_small_smem(), s, what, L, (int)P, (int)M,
                   (int)p.selection, (int)p.tournament_k, (int)p.scaling, p.seed, (uint32_t)gen, (uint32_t)island,
                   gen_ptr, order, sel, sigma, done);
    return PGA_OK;
}

// Selection for P > SMALL_P (hooks) / P > SMALL_GA_P (GA): order (unless
// `sorted`: the GA sorts in its own step), then tournament or SUS
// (k_qsum + k_sus2) with the mate slots fused.  Scratch: rank (int32 [P]),
// q (u64 [P]; also the sort's index double buffer), bsum (u64 [P / SCAN_T]).
int run_select_ops(const double *L, int64_t P, const pga_params &p, int32_t gen, int32_t island,
                   int32_t *order, int32_t *sel, uint64_t *keys_in, uint64_t *keys_out,
                   int32_t *idx_in, int32_t *rank, uint64_t *q, uint64_t *bsum, const int32_t *done,
                   cudaStream_t s, const int32_t *gen_ptr, bool sorted, int32_t *sigma) {
    const int64_t M = 2 * ((P - p.elite + 1) / 2);
    if (!sorted && P <= SMALL_P)   // one CTA; mates go to scratch (q)
        return launch_select_small(3, L, P, p, gen, island, gen_ptr, order, sel,
                                   reinterpret_cast<int32_t *>(q), done, s);
    int rc;
    if (!sorted) {
        rc = sort_order(L, P, order, rank, keys_in, keys_out, idx_in, reinterpret_cast<int32_t *>(q), done, s);
        if (rc) return rc;
    }
    if (p.selection == PGA_SEL_TOURNAMENT) {
        PGA_LAUNCH_PDL(k_tournament, dim3((unsigned)((M + 255) / 256)), dim3(256), 0, s, L, P, M,
                       (int)p.tournament_k, p.seed, (uint32_t)gen, (uint32_t)island, sel, done, gen_ptr, sigma);
        return PGA_OK;
    }
    const int nbq = (int)((P + SCAN_T - 1) / SCAN_T);
    PGA_LAUNCH_PDL(k_qsum, dim3(nbq), dim3(SCAN_T), 0, s, L, (const int32_t *)order, (const int32_t *)rank, P,
                   (int)p.scaling, q, bsum, done);
    const unsigned nbs = (unsigned)((max(P, M) + SCAN_T - 1) / SCAN_T);
    PGA_LAUNCH_PDL(k_sus2<SCAN_T>, dim3(nbs), dim3(SCAN_T), 0, s, (const uint64_t *)q, (const uint64_t *)bsum, nbq, L,
                   (const int32_t *)order, P, M, (int)p.scaling, p.seed, (uint32_t)gen, (uint32_t)island, sel,
                   done, gen_ptr, sigma);
    return PGA_OK;
}

int run_mates(int64_t M, const pga_params &p, int32_t gen, int32_t island, int32_t *sigma, cudaStream_t s) {
    k_mates<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(M, p.seed, (uint32_t)gen, (uint32_t)island, sigma,
                                                        nullptr, nullptr);
    PGA_LAUNCHED();
    return PGA_OK;
}

static void fill_breed(BreedArgs &a, const pga_params &p, int64_t P, int N) {
    a.thr_c = 0;
    a.P = P;
    a.N = N;
    a.E = p.elite;
    a.seed = p.seed;
    a.rk = round_keys(p.seed);
    a.island = (uint32_t)p.island;
    auto thr = [](double x) -> uint64_t {
        if (x >= 1.0) return (uint64_t)1 << 32;
        if (x <= 0.0) return 0;
        return (uint64_t)llround(x * 4294967296.0);   // Q13: llround(p * 2^32)
    };
    a.thr_c = thr(p.p_crossover);
    a.thr_m = thr(p.p_mutation);
    a.thr_kb = thr(p.p_kb);
}

int launch_breed_hook(const int32_t *pop, const int32_t *top, const int32_t *order, int64_t P,
                      int N, const int32_t *sel, const int32_t *sigma, const pga_params &p,
                      int32_t gen, int32_t island, int64_t p_off, int32_t *next, cudaStream_t s) {
    BreedArgs a{};
    fill_breed(a, p, P, N);
    a.i32_in = pop;
    a.i32_out = next;
    a.top32 = top;
    a.order = order;
    a.sel = sel;
    a.sigma = sigma;
    a.p_off = p_off;
    a.gen = (uint32_t)gen;
    a.island = (uint32_t)island;
    a.ldn = N;
    a.Pcap = P;
    count_launch();
    if (N <= BREED2_MAXN) PGA_CUDA(launch_breed2<true>(a, P, N, s));
    else PGA_CUDA(launch_pdl(k_breed<true>, dim3((unsigned)((P + BS - 1) / BS)), dim3(BW * 32), breed_smem(N), s, a));
    return PGA_OK;
}

// GA generations: one CTA up to 1024 (bitonic); above that the multi-CTA
// path (run sort + merge tree, weights, scan, SUS, mates) is faster than the
// single-CTA block radix sort (pga_op_select still uses it up to SMALL_P)
constexpr int SMALL_GA_P = 1024;
// order fused into the selection launch (one CTA up to SMALL_GA_P, one
// cluster up to CSEL_MAXP); above, the run sort + merge tree is its own step
bool small_select(const pga_ctx *c) {
    return c->P <= SMALL_GA_P || (c->P <= CSEL_MAXP && g_csel_ok && !getenv_flag("PGA_NO_CSEL", false));
}
// Rank + selection in one launch (k_rank_sel) for SMALL_GA_P < P <= RANKC_MAXP
static bool rankc_use(const pga_ctx *c) {
    return c->P > SMALL_GA_P && c->P <= pga::RANKC_MAXP && c->rc_acc && !getenv_flag("PGA_NO_RANKC", false);
}
int prepare_rank_sel(pga_ctx *c) {
    if (!c->rc_acc) return PGA_OK;
    k_qtab<<<(unsigned)((c->P + 255) / 256), 256, 0, c->stream>>>((int)c->P, c->rc_qtab);
    PGA_CUDA(cudaGetLastError());
    return PGA_OK;
}
static int launch_rank_sel(pga_ctx *c, bool sus, cudaStream_t s) {
    const int P = (int)c->P, M = (int)(2 * ((c->P - c->p.elite + 1) / 2));
    const int ipt = P <= 8192 ? 1 : 2, tile = RS_T * ipt;
    const unsigned nb = (unsigned)((P + tile - 1) / tile), nc = (unsigned)((P + RS_T - 1) / RS_T);
    if (ipt == 1)
        PGA_LAUNCH_PDL(k_rank_sel<1>, dim3(nb, nc), dim3(RS_T), 0, s, (const double *)c->L, P,
                       (const uint64_t *)c->rc_qtab, c->rc_acc, reinterpret_cast<uint32_t *>(c->rc_acc + c->Pcap),
                       c->order, c->rank, sus, c->keys_in, M, c->p.seed, (uint32_t)c->p.island,
                       (const int32_t *)&c->st->gen, c->sel);
    else
        PGA_LAUNCH_PDL(k_rank_sel<2>, dim3(nb, nc), dim3(RS_T), 0, s, (const double *)c->L, P,
                       (const uint64_t *)c->rc_qtab, c->rc_acc, reinterpret_cast<uint32_t *>(c->rc_acc + c->Pcap),
                       c->order, c->rank, sus, c->keys_in, M, c->p.seed, (uint32_t)c->p.island,
                       (const int32_t *)&c->st->gen, c->sel);
    return PGA_OK;
}

int launch_sort_order(pga_ctx *c, cudaStream_t s) {
    if (c->P <= SMALL_GA_P)
        return launch_select_small(1, c->L, c->P, c->p, 0, c->p.island, &c->st->gen, c->order, c->sel,
                                   c->sigma, &c->st->done, s);
    if (rankc_use(c)) return launch_rank_sel(c, false, s);
    if (small_select(c))
        return launch_select_cluster(1, c->L, c->P, c->p, &c->st->gen, c->order, c->rank, c->sel,
                                     &c->st->done, s);
    return sort_order(c->L, c->P, c->order, c->rank, c->keys_in, c->keys_out, c->idx_in,
                      reinterpret_cast<int32_t *>(c->q), &c->st->done, s);
}

// Isolate fittest + scaling + selection of a generation (Alg. 1):
// one CTA up to SMALL_GA_P, one thread-block cluster up to CSEL_MAXP, else the
// run sort + merge tree, then SUS (or tournament).  The mate slots come from
// the side stream (launch_mates_fork) for P > SMALL_GA_P.
int launch_select(pga_ctx *c, cudaStream_t s) {
    const pga_params &p = c->p;
    const int32_t *done = &c->st->done;
    const int32_t *genp = &c->st->gen;
    int rc;
    if (c->P <= SMALL_GA_P) {
        rc = launch_select_small(3, c->L, c->P, p, 0, p.island, genp, c->order, c->sel, c->sigma, done, s);
        if (rc) return rc;
    } else if (rankc_use(c)) {
        // SUS with rank scaling (Table 3) completes in the launch; otherwise
        // it leaves order / rank to the tournament or fitness-scaled SUS
        const bool fused = p.selection == PGA_SEL_SUS && p.scaling == PGA_SCALE_RANK;
        rc = launch_rank_sel(c, fused, s);
        if (rc) return rc;
        if (!fused) {
            rc = run_select_ops(c->L, c->P, p, 0, p.island, c->order, c->sel, c->keys_in, c->keys_out,
                                c->idx_in, c->rank, c->q, c->keys_in, done, s, genp, true, nullptr);
            if (rc) return rc;
        }
    } else if (small_select(c)) {
        rc = launch_select_cluster(3, c->L, c->P, p, genp, c->order, c->rank, c->sel, done, s);
        if (rc) return rc;
    } else {
        rc = sort_order(c->L, c->P, c->order, c->rank, c->keys_in, c->keys_out, c->idx_in,
                        reinterpret_cast<int32_t *>(c->q), done, s);
        if (rc) return rc;
        rc = run_select_ops(c->L, c->P, p, 0, p.island, c->order, c->sel, c->keys_in, c->keys_out,
                            c->idx_in, c->rank, c->q, c->keys_in /* free after the sort: block sums */,
                            done, s, genp, true, nullptr);
        if (rc) return rc;
    }
    return PGA_OK;
}

// Crossover, mutation, canonicalisation, replacement (Alg. 1) from
// the selection launch_select left in order / sel / sigma; the last CTA
// advances the generation.
int launch_breed(pga_ctx *c, cudaStream_t s, bool late_masks) {
    const pga_params &p = c->p;
    const int32_t *done = &c->st->done;
    const int32_t *genp = &c->st->gen;
    BreedArgs a{};
    fill_breed(a, p, c->P, c->N);
    a.cm_in0 = c->pop[0];
    a.cm_in1 = c->pop[1];
    a.cm_out0 = c->pop[0];
    a.cm_out1 = c->pop[1];
    a.gm_out0 = c->popT[0];
    a.gm_out1 = c->popT[1];
    a.top16 = c->top;
    a.order = c->order;
    a.sel = c->sel;
    a.sigma = c->sigma;
    a.Pcap = c->Pcap;
    a.p_off = (int64_t)p.island * c->P;
    a.ldn = c->ldn;
    a.done = done;
    a.gen_ptr = genp;
    // the gene-major copy is produced by the label-sparse pass while its
    // checks are live (it transposes exactly the blocks the dense sweep needs)
    a.gm_skip = (sparse_theta_eff(c) > 0.0 && c->N <= SPARSE_MAX_N) ? c->sp_live : nullptr;
    a.adv_st = c->st;           // the breed's last CTA advances the generation (no k_advance)
    if (!(c->P <= SMALL_GA_P) && c->mmask && (mutmask_use(c->P) || (late_masks && mutmask_late(c)))) {
        // masks from the side stream
        a.mmask = c->mmask;
        a.mw = (c->N + 31) / 32;
    }
    a.adv_ctr = c->breed_ctr;
    count_launch();
    if (c->N <= BREED2_MAXN)
        PGA_CUDA(launch_breed2<false>(a, c->P, c->N, s));
    else
        PGA_CUDA(launch_pdl(k_breed<false>, dim3((unsigned)((c->P + BS - 1) / BS)), dim3(BW * 32),
                            breed_smem(c->N), s, a));
    PGA_MARK(c, 7, s);
    return PGA_OK;
}

// Mate slots (Q10) depend only on (seed, generation, island): for P >
// SMALL_GA_P they are computed on a side stream forked at the start of a
// generation's evaluation and joined at its end, so the Feistel permutation
// runs beside the fitness pass instead of on the selection's critical path.
// (P <= SMALL_GA_P: k_select_small computes them itself.)
// the generation's mutation masks (the breed's per-gene MUT draws) on s
int launch_mutmask(pga_ctx *c, cudaStream_t s) {
    BreedArgs t{};
    fill_breed(t, c->p, c->P, c->N);
    const int mw = (c->N + 31) / 32;
    const int64_t nth = c->P * (int64_t)mw;
    k_mutmask<<<(unsigned)((nth + 255) / 256), 256, 0, s>>>(t.rk, (uint32_t)c->p.island, &c->st->gen, &c->st->done,
                                                            c->P, c->N, c->p.elite, (int64_t)c->p.island * c->P,
                                                            t.thr_m, mw, c->mmask);
    PGA_LAUNCHED();
    return PGA_OK;
}

// For P > MUTMASK_MAXP the masks are computed beside the statistics and the
// selection of a non-migration generation (latency-bound sort / scan launches
// that leave most SMs idle), and the breed of that generation reads them.
bool mutmask_late(const pga_ctx *c) {
    return c->mmask && c->P > MUTMASK_MAXP && c->P > SMALL_GA_P && !getenv_flag("PGA_NO_MUTMASK_LATE", false);
}

int launch_mates_fork(pga_ctx *c, cudaStream_t s) {
    if (c->P <= SMALL_GA_P) return PGA_OK;
    const int64_t M = 2 * ((c->P - c->p.elite + 1) / 2);
    PGA_CUDA(cudaEventRecord(c->fork_ev, s));
    PGA_CUDA(cudaStreamWaitEvent(c->side, c->fork_ev, 0));
    k_mates<<<(unsigned)((M + 255) / 256), 256, 0, c->side>>>(M, c->p.seed, 0u, (uint32_t)c->p.island, c->sigma,
                                                               &c->st->done, &c->st->gen);
    PGA_LAUNCHED();
    if (c->mmask && mutmask_use(c->P)) {
        const int rc = launch_mutmask(c, c->side);
        if (rc) return rc;
    }
    PGA_CUDA(cudaEventRecord(c->join_side_ev, c->side));
    return PGA_OK;
}

int launch_mates_join(pga_ctx *c, cudaStream_t s) {
    if (c->P <= SMALL_GA_P) return PGA_OK;
    PGA_CUDA(cudaStreamWaitEvent(s, c->join_side_ev, 0));
    return PGA_OK;
}

int launch_export(pga_ctx *c, void *dev_send, cudaStream_t s) {
    PGA_LAUNCH_PDL(k_export, dim3(c->p.migrants), dim3(128), 0, s, (const double *)c->L, (const uint16_t *)c->top,
                   (const int32_t *)c->order, (const uint16_t *)c->pop[0], (const uint16_t *)c->pop[1],
                   (const pga::DevState *)c->st, (int)c->ldn, (int)c->N, (int)c->p.migrants,
                   (int64_t)(c->mig_bytes / c->p.migrants), (unsigned char *)dev_send);
    return PGA_OK;
}

int launch_import(pga_ctx *c, const void *dev_recv, int32_t G, cudaStream_t s) {
    PGA_LAUNCH_PDL(k_import, dim3(1), dim3(256), 0, s, (const unsigned char *)dev_recv, (int)G, (int)c->p.migrants,
                   (int64_t)(c->mig_bytes / c->p.migrants), (const int32_t *)c->order, c->P, c->L, c->top,
                   c->pop[0], c->pop[1], c->popT[0], c->popT[1], (const pga::DevState *)c->st, (int)c->ldn,
                   (int)c->N, c->Pcap);
    return PGA_OK;
}

}  // namespace pga
