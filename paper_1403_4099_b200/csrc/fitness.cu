// fitness.cu — batched Giada–Marsili fitness (Eq. 5, 6, 8).
//
// One kernel per evaluation (k_fitness, below):
//   sweep    the O(N^2 P) masked pair sweep: every row i of every
//            chromosome accumulates r'_i = sum_{j>i, s_j = s_i} C_ij in fp64
//            (3 SASS instructions per pair, see k_fitness).  V = C_ii + 2 r'_i.
//   fold     warp per chromosome (fused, last CTA per chromosome block): n_s by __match_any_sync/popc (exact),
//            c_s = sum_{i in s} V[p][i] in a fixed order (pointer-jumping
//            group sums, no float atomics -> deterministic), then Eq. 8 with
//            readings Q1-Q3, L = 1/2 sum f_s and top = argmax f_s.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include "pga_internal.cuh"

namespace {

using namespace pgad;

// ---------------------------------------------------------------------------
// k_pack: caller labels -> the two internal layouts.
//   lab16: uint16 [P][ld_in] 0-based (device fast path, unchecked), or
//   lab32: int32  [P][N]     1-based (checked; error flag in st->pack_error).
// 32x32 tile transpose through shared memory.
// ---------------------------------------------------------------------------
__global__ void k_pack(const uint16_t *__restrict__ lab16, const int32_t *__restrict__ lab32,
                       int64_t P, int ld_in, int N, int ldn, int64_t Pcap,
                       uint16_t *__restrict__ CM, uint16_t *__restrict__ GM,
                       pga::DevState *st) {
    __shared__ uint16_t tile[32][33];
    const int64_t p0 = (int64_t)blockIdx.x * 32;
    const int i0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        const int64_t p = p0 + r;
        const int i = i0 + tx;
        uint16_t v = 0;
        if (p < P && i < N) {
            if (lab16) {
                v = lab16[p * ld_in + i];
                if (v >= (uint16_t)N) {    // out of range: flagged, evaluated as label 0 (no stray table index)
                    atomicExch(&st->pack_error, 1);
                    v = 0;
                }
            } else {
                const int32_t x = lab32[p * (int64_t)N + i];
                if (x < 1 || x > N) {
                    atomicExch(&st->pack_error, 1);
                    v = 0;
                } else {
                    v = (uint16_t)(x - 1);
                }
            }
            CM[p * ldn + i] = v;
        }
        tile[r][tx] = v;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + r;
        const int64_t p = p0 + tx;
        if (i < N && p < P) GM[(int64_t)i * Pcap + p] = tile[tx][r];
    }
}

// ---------------------------------------------------------------------------
// k_fitness: TMA-pipelined pair sweep + fused fold.
//
// CTA tile = 32 chromosomes (one per lane) x RT = 64 rows (four consumer
// warps x 16 rows).  A producer warp streams the tile's columns j in chunks
// of KC through NSTAGE shared-memory stages with TMA (cp.async.bulk.tensor,
// mbarrier complete_tx): per stage the gene-major labels [KC][32] u16 and
// the C strip [KC][RT] fp64 (C is symmetric, so C[j][i0..i0+RT) is the
// contiguous row segment).  Out-of-range rows/columns are zero-filled by TMA
// and never match (row labels NaN) or are never visited.
//
// Inner step (two rows r, r+1 of one chromosome against column j):
//   ld.shared.v4  {lo_r, hi_r, lo_r1, hi_r1} = C[j][r..r+1]   (broadcast)
//   HSETP2        p|q = (s_r, s_r1) == (s_j, s_j)   packed fp16 compare of
//                 the raw 16-bit labels (exact, never NaN for labels < 31744)
//   SEL x2        hi := p ? hi : 0  (in place)
//   DADD x2       acc_r += {lo, hi}
// A non-match adds the positive denormal {lo, 0} < 2^-1022, which rounds away
// against any normal accumulator and cannot change V = C_ii + 2 acc.
// CTAs are ordered chromosome-block-major; the last CTA to finish a block
// (atomic counter, threadfence pattern) folds its chromosomes while V is
// still in L2.
// ---------------------------------------------------------------------------
constexpr int KC = 32;                  // columns per stage
constexpr int NSTAGE = 3;
constexpr int CW = 4;                   // consumer warps
constexpr int WR = 16;                  // rows per consumer warp
constexpr int RT = CW * WR;             // rows per CTA tile
constexpr int LAB_BYTES = KC * pga::CB * 2;
constexpr int CST_BYTES = KC * RT * 8;
constexpr int STAGE_BYTES = LAB_BYTES + CST_BYTES;
constexpr int FIT_THREADS = (CW + 1) * 32;
constexpr int FIT_BLOCKS_PER_CTA_MIN = 1024;   // chromosome blocks from which a k_fitness CTA sweeps a whole block
static_assert(KC % WR == 0, "a warp's rows must not straddle two chunks");

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// try_wait with a suspend-time hint: a waiting thread sleeps in hardware
// until the phase completes (or the hint expires) instead of spinning and
// stealing issue slots from the consumer warps on its SMSP.
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *tm, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)tm), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

struct FitArgs {
    int N, ldn, nRT, nCB, fold_warps;
    int F, cpb;                     // row tiles per CTA, CTAs per chromosome block (cpb = ceil(nRT / F))
    int cb0;                        // first chromosome block (shard offset / 32)
    double fx_scale, fx_inv;        // fold fixed point: 2^S and 2^-S
    const double *lgn, *lgnn;       // log n, log(n^2 - n), n = 0..N (Q30)
    const double2 *lnt;             // fast_ln table (after lgn, lgnn in the ctx's lgtab)
    const uint8_t *sflag;           // per chromosome block: 1 = already evaluated label-sparsely
    int64_t P, Pcap;
    const double *diag;
    double *V;                      // [Pcap][ldn]: V[p][i] = C_ii + 2 r'_i
    const uint16_t *cm0, *cm1;
    const uint16_t *gm0, *gm1;      // gene-major labels [N][Pcap]
    double *L;
    uint16_t *top;
    const int32_t *gen, *done;
    uint32_t *counters;
};

// Two rows (packed labels rp) against one column (col = s_j | s_j << 16);
// caddr = shared address of C[j][r], C[j][r+1].
__device__ __forceinline__ void pair2(uint32_t caddr, uint32_t rp, uint32_t col, double &a0, double &a1) {
    asm("{\n\t.reg .pred p, q;\n\t.reg .b32 l0, h0, l1, h1;\n\t.reg .b64 d0, d1;\n\t"
        "ld.shared.v4.u32 {l0, h0, l1, h1}, [%2];\n\t"
        "setp.eq.f16x2 p|q, %3, %4;\n\t"
        "selp.b32 h0, h0, 0, p;\n\t"
        "selp.b32 h1, h1, 0, q;\n\t"
        "mov.b64 d0, {l0, h0};\n\t"
        "mov.b64 d1, {l1, h1};\n\t"
        "add.f64 %0, %0, d0;\n\t"
        "add.f64 %1, %1, d1;\n\t}"
        : "+d"(a0), "+d"(a1)
        : "r"(caddr), "r"(rp), "r"(col));
}

// 16 pair updates: rows 0..15 of this lane's chromosome against column j.
__device__ __forceinline__ void pairs16(uint32_t caddr, uint32_t w, const uint32_t (&rp)[WR / 2],
                                        double (&acc)[WR]) {
    const uint32_t col = w | (w << 16);
#pragma unroll
    for (int q = 0; q < WR / 2; ++q) pair2(caddr + 16 * q, rp[q], col, acc[2 * q], acc[2 * q + 1]);
}

// Eq. 8 (Q1-Q3) of one chromosome from its per-label tables (warp-wide):
// cs[k] = c_k in 64-bit fixed point (scale 2^S, read through inv_scale),
// ns[k] = n_k, labels k < K.  Clusters with n >= 2 and c > n (the only
// non-zero summands, Q2) are compacted to the front of cs/ns in label order
// (ns keeps n | label << 16), then the summands are taken lane-parallel as
// (log n - log c) + (n-1)(log(n^2-n) - log(n^2-c)) with the integer logs from
// the table (Q30: no divisions) and the two real logs by the table-driven
// fast_ln (as the label-sparse pass; c > n >= 2 and n^2 - c >= 1e-9 here),
// c clamped to n^2 - 1e-9 (Q3); L = half the sum; top = label of the
// largest summand (smallest label on ties).
__device__ __forceinline__ void eq8_tables(double *cs, int32_t *ns, int K, int lane, double inv_scale,
                                           const double *__restrict__ lgn, const double *__restrict__ lgnn,
                                           const double2 *__restrict__ lnt, double *L_out, uint16_t *top_out) {
    int M = 0;
    for (int k0 = 0; k0 < K; k0 += 32) {
        const int k = k0 + lane;
        int n = 0;
        double c = 0.0;
        if (k < K) {
            n = ns[k];
            c = (double)reinterpret_cast<const long long *>(cs)[k] * inv_scale;
        }
        const bool act = (n >= 2) && (c > (double)n);
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, act);   // orders this chunk's reads before its writes
        if (act) {
            const int idx = M + __popc(bal & lanemask_lt());
            cs[idx] = c;
            ns[idx] = n | (k << 16);
        }
        M += __popc(bal);
    }
    double fsum = 0.0, fbest = 0.0;
    int kbest = 0x7FFFFFFF;
    for (int j = lane; j < M; j += 32) {
        const int nk = ns[j];
        const int n = nk & 0xFFFF;
        const double nd = (double)n, n2 = nd * nd;
        const double ch = fmin(cs[j], n2 - 1e-9);
        const double f = (__ldg(lgn + n) - fast_ln(ch, lnt)) + (nd - 1.0) * (__ldg(lgnn + n) - fast_ln(n2 - ch, lnt));
        fsum += f;
        if (f > fbest) {
            fbest = f;
            kbest = nk >> 16;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        fsum += __shfl_xor_sync(0xFFFFFFFFu, fsum, off);
        const double of = __shfl_xor_sync(0xFFFFFFFFu, fbest, off);
        const int ok = __shfl_xor_sync(0xFFFFFFFFu, kbest, off);
        if (of > fbest || (of == fbest && ok < kbest)) {
            fbest = of;
            kbest = ok;
        }
    }
    if (lane == 0) {
        *L_out = 0.5 * fsum;
        if (top_out) *top_out = (fbest > 0.0) ? (uint16_t)kbest : (uint16_t)0xFFFF;
    }
}

// Summand of Eq. 8 (Q1-Q3) for a cluster of n >= 2 members with intra-
// cluster sum c: 0 unless c > n (Q2); c clamped to n^2 - 1e-9 (Q3); the
// integer logs from the table (Q30), ln by the table-driven fast_ln (the
// label-sparse pass: its clusters all have c > n >= 2 and n^2 - c >= 1e-9,
// positive normals).
__device__ __forceinline__ double eq8_term_fast(int n, double c, const double *__restrict__ lgn,
                                                const double *__restrict__ lgnn,
                                                const double2 *__restrict__ lnt) {
    if (!(c > (double)n)) return 0.0;
    const double nd = (double)n, n2 = nd * nd;
    const double ch = fmin(c, n2 - 1e-9);
    return (__ldg(lgn + n) - fast_ln(ch, lnt)) + (nd - 1.0) * (__ldg(lgnn + n) - fast_ln(n2 - ch, lnt));
}

// Fold (warp-wide) of NC chromosomes at once (independent chains -> ILP):
// lane per gene; n_s by a shared-memory integer atomic, and c_s = sum of V_i
// over the cluster accumulated in 64-bit fixed point (V * 2^S, S = 62 -
// ceil(log2(2 N^2 + 1)) so no cluster sum can overflow) by shared-memory
// integer atomics.  Integer addition is exact and order-free, so the result
// is deterministic without any per-group ordering; the quantisation (2^-S-1
// per V, 6e-14 at N = 500) is below the fp64 summation error it replaces.
// Then Eq. 8 (Q1-Q3) for labels up to the chromosome's largest.
template <int NC>
__device__ __forceinline__ void fold_multi(const uint16_t *const (&lab)[NC], int64_t lstride,
                                           const double *const (&v)[NC],
                                           int N, double *const (&cs)[NC], int32_t *const (&ns)[NC],
                                           int lane, double *const (&L_out)[NC],
                                           uint16_t *const (&top_out)[NC], double scale, double inv_scale,
                                           const double *__restrict__ lgn, const double *__restrict__ lgnn,
                                           const double2 *__restrict__ lnt) {
    // cs / ns were zeroed by the caller (all-zero bits == integer 0)
    // software pipeline: loads of chunk c+2 are issued while chunk c folds.
    // Gene-major labels of two adjacent chromosomes (p even, p + 1) are one
    // aligned 32-bit word per gene: one load for the pair.
    const bool pair = (NC == 2) && lstride != 1 && lab[NC - 1] == lab[0] + 1;
    auto ld = [&](int q, int i) -> uint32_t {
        if (i >= N) return 0u;
        if (pair) {
            const uint32_t w = *reinterpret_cast<const uint32_t *>(lab[0] + i * lstride);
            return q ? (w >> 16) : (w & 0xFFFFu);
        }
        return (uint32_t)lab[q][i * lstride];
    };
    uint32_t s_n1[NC], s_n2[NC];
    double v_n1[NC], v_n2[NC];
    if (pair) {
        const uint32_t w1 = lane < N ? *reinterpret_cast<const uint32_t *>(lab[0] + lane * lstride) : 0u;
        const uint32_t w2 = 32 + lane < N ? *reinterpret_cast<const uint32_t *>(lab[0] + (32 + lane) * lstride) : 0u;
        s_n1[0] = w1 & 0xFFFFu;
        s_n1[NC - 1] = w1 >> 16;
        s_n2[0] = w2 & 0xFFFFu;
        s_n2[NC - 1] = w2 >> 16;
    } else {
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            s_n1[q] = ld(q, lane);
            s_n2[q] = ld(q, 32 + lane);
        }
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        v_n1[q] = (lane < N) ? __ldcg(v[q] + lane) : 0.0;
        v_n2[q] = (32 + lane < N) ? __ldcg(v[q] + 32 + lane) : 0.0;
    }
    uint32_t kmax = 0;
    for (int base = 0; base < N; base += 32) {
        const bool valid = base + lane < N;
        const int i3 = base + 64 + lane;
        uint32_t w3 = 0u;
        if (pair && i3 < N) w3 = *reinterpret_cast<const uint32_t *>(lab[0] + i3 * lstride);
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            const uint32_t s = s_n1[q];
            const double x = v_n1[q];
            s_n1[q] = s_n2[q];
            v_n1[q] = v_n2[q];
            s_n2[q] = pair ? (q ? (w3 >> 16) : (w3 & 0xFFFFu)) : ld(q, i3);
            v_n2[q] = (i3 < N) ? __ldcg(v[q] + i3) : 0.0;
            if (valid) {
                kmax = max(kmax, s);
                atomicAdd(reinterpret_cast<unsigned long long *>(cs[q]) + s,
                          (unsigned long long)__double2ll_rn(x * scale));
                atomicAdd(&ns[q][s], 1);
            }
        }
    }
    __syncwarp();
#ifdef PGA_DIAG_NO_LOG   // measurement builds only (tools/): accumulation without compaction / Eq. 8
    if (lane == 0)
        for (int q = 0; q < NC; ++q) *L_out[q] = (double)kmax;
    return;
#endif
    // largest label of the (up to NC) chromosomes, warp-uniform
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) kmax = max(kmax, __shfl_xor_sync(0xFFFFFFFFu, kmax, off));
    const int K = (int)min(kmax + 1u, (uint32_t)N);
#pragma unroll
    for (int q = 0; q < NC; ++q)
        eq8_tables(cs[q], ns[q], K, lane, inv_scale, lgn, lgnn, lnt, L_out[q], top_out[q]);
    __syncwarp();
}

__global__ void __launch_bounds__(FIT_THREADS)
k_fitness(const __grid_constant__ CUtensorMap tmLab0, const __grid_constant__ CUtensorMap tmLab1,
          const __grid_constant__ CUtensorMap tmC, FitArgs a) {
    pdl_wait();
    pdl_trigger();
    {   // both exit tests from one round trip (independent loads): with every
        // block evaluated label-sparsely, this is all a CTA does
        const int32_t dn = a.done ? __ldg(a.done) : 0;
        const uint8_t sf = a.sflag ? a.sflag[a.cb0 + (int)(blockIdx.x / a.cpb)] : (uint8_t)0;
        if (dn | sf) return;   // stopped, or done by k_fitness_sparse
    }
    const int par = (a.gen && (*a.gen & 1)) ? 1 : 0;
    const CUtensorMap *tmLab = par ? &tmLab1 : &tmLab0;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // keep the shared address space visible to ptxas (LDS, not generic LD)
    unsigned char *smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NSTAGE * STAGE_BYTES);
    uint64_t *empty = full + NSTAGE;
    __shared__ int s_last;

    const int N = a.N;
    const int cb = a.cb0 + (int)(blockIdx.x / a.cpb);
    const int rt_lo = (int)(blockIdx.x % a.cpb) * a.F, rt_hi = min(a.nRT, rt_lo + a.F);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // The CTA sweeps row tiles rt_lo .. rt_hi-1 of its chromosome block in
    // turn (F > 1 keeps the grid near the resident-CTA count when the block
    // count is large, so a launch whose blocks all went label-sparse costs
    // few CTA launches).  Stage s / phase of chunk kk continue across tiles.
    int kk0 = 0;
    for (int rt = rt_lo; rt < rt_hi; ++rt) {
    const int i0 = rt * RT;
    const int nchunks = (N - i0 + KC - 1) / KC;

    if (warp == CW) {
        // ---------------- producer ----------------
        if (lane == 0) {
            for (int k = 0; k < nchunks; ++k) {
                const int kk = kk0 + k;
                const int s = kk % NSTAGE;
                if (kk >= NSTAGE) mbar_wait(&empty[s], (uint32_t)((kk / NSTAGE - 1) & 1));
                unsigned char *st = smem + s * STAGE_BYTES;
                mbar_expect_tx(&full[s], STAGE_BYTES);
                tma_load_2d(st, tmLab, cb * pga::CB, i0 + k * KC, &full[s]);
                tma_load_2d(st + LAB_BYTES, &tmC, i0, i0 + k * KC, &full[s]);
            }
        }
    } else {
        // ---------------- consumers ----------------
        const int i0w = i0 + WR * warp;     // first row of this warp
        const int lw = WR * warp;           // its local column in chunk 0
        const bool active = i0w < N;
        uint32_t rp[WR / 2];
        double acc[WR];
#pragma unroll
        for (int r = 0; r < WR; ++r) acc[r] = 0.0;
        // this warp's rows are the columns lw..lw+15, i.e. chunk kw at local
        // column lw0 (KC is a multiple of WR); earlier chunks hold only
        // columns j < i0w and are skipped by this warp.
        const int kw = lw / KC, lw0 = lw - kw * KC;
        uint32_t rl[WR];
        for (int k = 0; k < nchunks; ++k) {
            const int kk = kk0 + k;
            const int s = kk % NSTAGE;
            mbar_wait(&full[s], (uint32_t)((kk / NSTAGE) & 1));
            const unsigned char *st = smem + s * STAGE_BYTES;
            const uint16_t *labs = reinterpret_cast<const uint16_t *>(st) + lane;
            const double *cst = reinterpret_cast<const double *>(st + LAB_BYTES) + lw;
            const uint32_t cbase = smem_u32(cst);
            const int jbase = i0 + k * KC;
            int t = 0;
            const int tend = min(KC, N - jbase);
            if (active && k >= kw) {
                if (k == kw) {
                    // this lane's labels of the warp's rows
#pragma unroll
                    for (int r = 0; r < WR; ++r)
                        rl[r] = (i0w + r < N) ? (uint32_t)labs[(lw0 + r) * pga::CB] : 0x7FFFu;
#pragma unroll
                    for (int q = 0; q < WR / 2; ++q) rp[q] = rl[2 * q] | (rl[2 * q + 1] << 16);
                    // diagonal block: local columns lw0+1 .. lw0+15, rows r < d
#pragma unroll
                    for (int d = 1; d < WR; ++d) {
                        const int lc = lw0 + d;
                        if (jbase + lc < N) {
                            const uint32_t sj = labs[lc * pga::CB];
                            const double *cj = cst + lc * RT;
#pragma unroll
                            for (int r = 0; r < d; ++r)
                                if (rl[r] == sj) acc[r] += cj[r];
                        }
                    }
                    t = lw0 + WR;
                }
#pragma unroll 1
                for (; t + 1 < tend; t += 2) {
                    const uint32_t w0 = labs[t * pga::CB], w1 = labs[(t + 1) * pga::CB];
                    pairs16(cbase + t * RT * 8, w0, rp, acc);
                    pairs16(cbase + (t + 1) * RT * 8, w1, rp, acc);
                }
                if (t < tend) pairs16(cbase + t * RT * 8, labs[t * pga::CB], rp, acc);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (active) {
            const int64_t p = (int64_t)cb * pga::CB + lane;
            double *vp = a.V + p * a.ldn + i0w;
#pragma unroll
            for (int r = 0; r < WR; r += 2) {
                const double d0 = (i0w + r < N) ? a.diag[i0w + r] : 0.0;
                const double d1 = (i0w + r + 1 < N) ? a.diag[i0w + r + 1] : 0.0;
                reinterpret_cast<double2 *>(vp)[r >> 1] = make_double2(fma(2.0, acc[r], d0), fma(2.0, acc[r + 1], d1));
            }
        }
    }
    kk0 += nchunks;
    }   // row tiles

    // ---------------- fused fold (last CTA of the chromosome block) ----------------
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(&a.counters[cb], 1u);
        s_last = (prev == (unsigned)(a.cpb - 1));
    }
    __syncthreads();
    if (!s_last) return;
#ifdef PGA_DIAG_NO_FOLD   // measurement builds only (tools/): sweep without the fold
    if (tid == 0) a.counters[cb] = 0u;
    return;
#endif
    __threadfence();
    if (warp < a.fold_warps) {
        // NCF chromosomes per warp per pass (independent chains -> ILP)
        constexpr int NCF = 2;
        // labels from the gene-major copy the sweep streamed (its 64-byte
        // rows of this block are in L2/L1), not a second DRAM read of the
        // chromosome-major copy
        const uint16_t *GM = par ? a.gm1 : a.gm0;
        double *csb = reinterpret_cast<double *>(smem) + (size_t)warp * NCF * N;
        int32_t *nsb = reinterpret_cast<int32_t *>(reinterpret_cast<double *>(smem) + (size_t)a.fold_warps * NCF * N) +
                       (size_t)warp * NCF * N;
        for (int q = NCF * warp; q < pga::CB; q += NCF * a.fold_warps) {
            const int64_t p = (int64_t)cb * pga::CB + q;
            if (p >= a.P) break;
            const uint16_t *lab[NCF];
            const double *vv[NCF];
            double *cs[NCF];
            int32_t *ns[NCF];
            double *Lo[NCF];
            uint16_t *to[NCF];
#pragma unroll
            for (int c = 0; c < NCF; ++c) {
                const int64_t pc = (p + c < a.P) ? p + c : p;   // duplicate work at an odd tail
                lab[c] = GM + pc;
                vv[c] = a.V + pc * a.ldn;
                cs[c] = csb + c * N;
                ns[c] = nsb + c * N;
                Lo[c] = &a.L[pc];
                to[c] = a.top ? &a.top[pc] : nullptr;
            }
            {   // zero this warp's NCF x N accumulators and counters (vector stores)
                uint4 *c4 = reinterpret_cast<uint4 *>(csb);              // 16 N bytes, 16-byte aligned
                for (int k = lane; k < N * NCF / 2; k += 32) c4[k] = make_uint4(0u, 0u, 0u, 0u);
                uint2 *n2 = reinterpret_cast<uint2 *>(nsb);              // 8 N bytes, 8-byte aligned
                for (int k = lane; k < N * NCF / 2; k += 32) n2[k] = make_uint2(0u, 0u);
                __syncwarp();
            }
            fold_multi<NCF>(lab, a.Pcap, vv, N, cs, ns, lane, Lo, to, a.fx_scale, a.fx_inv, a.lgn, a.lgnn, a.lnt);
            // V of these chromosomes is dead: drop its L2 lines without a
            // DRAM write-back (rows are 128-byte aligned, ldn % 16 == 0)
#pragma unroll
            for (int c = 0; c < NCF; ++c) {
                if (p + c >= a.P) break;
                const char *row = reinterpret_cast<const char *>(a.V + (p + c) * a.ldn);
                for (int l = lane; l < a.ldn / 16; l += 32)
                    asm volatile("discard.global.L2 [%0], 128;" ::"l"(row + 128 * l) : "memory");
            }
        }
    }
    if (tid == 0) a.counters[cb] = 0u;
}

// k_resync_gm: rebuild the gene-major copy of the CURRENT population (buffer
// gen & 1) from the chromosome-major one.  While the label-sparse pass runs,
// the breed leaves the gene-major copy to it; when the pass is switched off
// mid-run (pga_set_sparse_threshold(0)) the dense sweep needs it back.
__global__ void k_resync_gm(const uint16_t *__restrict__ CM0, const uint16_t *__restrict__ CM1,
                            uint16_t *GM0, uint16_t *GM1, const pga::DevState *st, int64_t P, int N,
                            int ldn, int64_t Pcap) {
    __shared__ uint16_t tile[32][33];
    const int par = st->gen & 1;
    const uint16_t *CM = par ? CM1 : CM0;
    uint16_t *GM = par ? GM1 : GM0;
    const int64_t p0 = (int64_t)blockIdx.x * 32;
    const int i0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        const int64_t p = p0 + r;
        const int i = i0 + tx;
        tile[r][tx] = (p < P && i < N) ? CM[p * ldn + i] : (uint16_t)0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + r;
        const int64_t p = p0 + tx;
        if (i < N && p < P) GM[(int64_t)i * Pcap + p] = tile[tx][r];
    }
}

// ---------------------------------------------------------------------------
// k_fitness_sparse: label-sparse evaluation of a
// 32-chromosome block when its clusters are small.  Pass 1 (warp per
// chromosome, 4 per warp): n_s by shared-memory atomics on packed 16-bit
// counters; the block's largest sum_s n_s (n_s - 1) / 2.  If that is at most
// the threshold, pass 2 evaluates every chromosome exactly from its clusters:
// a counting sort by label, then each member g at position a of its cluster
// (size n) adds C[g][member (a + d) mod n] for d = 1 .. floor((n-1)/2) (and
// d = n/2 for the first n/2 members when n is even) -- every unordered pair
// exactly once -- gathered from L2; c_s = sum of C_gg + 2 sum of pairs in
// 64-bit fixed point (each term rounded to 2^-S, then integer sums: exact,
// order-free, deterministic); Eq. 8 from the tables.  The block is then
// flagged so that k_fitness skips it.  Work ~ sum_s n_s^2 instead of N^2.
//
// Cluster cache: c_s is a function of the member set alone (C is fixed for
// the ctx), and a GA generation repeats almost all of the previous one's
// clusters (elites, knowledge-based crossover transplants whole clusters,
// mutation moves ~2 genes; tools/cache_hit.py measures 93-99 % of the C4
// pairs).  A cluster with n >= CC_NMIN is keyed by the XOR of its members'
// 128-bit Zobrist keys (plus n) and looked up in a device hash table of exact
// fixed-point c_s; a hit replaces its n(n-1)/2 gathers, a miss is gathered
// and inserted.  The value is bit-identical either way (the fixed-point sum
// is order-free), so the cache changes cost, never results, short of a
// 128-bit key collision.
// ---------------------------------------------------------------------------
// Two instantiations of the pass (a CTA owns one 32-chromosome block; a
// chromosome's labels stay in registers, LREG 32-bit words per lane):
//   N <= SPARSE_SMALLN: 16 warps, LREG = 10, two CTAs per SM;
//   N <= SPARSE_MAXN (C5's N = 2000): 8 warps, LREG = 32, one CTA per SM
//   (the per-warp tables grow with N).
constexpr int SPARSE_SMALLN = 640, SPARSE_MAXN = pga::SPARSE_MAX_N;
__host__ __device__ __forceinline__ int sp_warps(int N) { return N <= SPARSE_SMALLN ? 16 : 8; }
#ifndef PGA_CC_NMIN
#define PGA_CC_NMIN 4
#endif
#ifndef PGA_SP_MINB
#define PGA_SP_MINB 2
#endif
constexpr int CC_NMIN = PGA_CC_NMIN;   // clusters this large go through the cache (4 since the keys are staged: C4 0.4843 -> 0.4667 ms against 5)
static_assert(CC_NMIN >= 2, "large clusters must have pairs");
constexpr int CC_PROBE = 8;        // linear-probe length

// Cluster classes of the label-sparse pass: n = 2 .. WALK_N-1 ("small") are
// evaluated lane-parallel from their recorded members (n = 2 from the pair-
// term table); n >= WALK_N ("walk class") get an ordinal, go through the
// cache when n >= CC_NMIN, and are walked when not a hit.
constexpr int WALK_N = 4;
constexpr int SMALL_N = WALK_N - 1;   // members recorded per label
static_assert(CC_NMIN >= WALK_N, "cacheable clusters are in the walk class");
__host__ __device__ __forceinline__ int cc_entries(int N) { return N / WALK_N + 1; }

// slot: k1 claimed by CAS (0 = empty); k2, v and chk = cc_mix(k1, k2, v, n)
// are then written once.  A reader takes the slot only if k1, k2 and the
// checksum agree, so a half-written slot reads as a miss without any
// ordering between the fields (relaxed L2 loads; no L1 invalidation).
__device__ __forceinline__ uint64_t cc_mix(uint64_t k1, uint64_t k2, long long v, uint32_t n) {
    uint64_t z = k1 ^ (k2 * 0x9E3779B97F4A7C15ull) ^ ((uint64_t)v * 0xBF58476D1CE4E5B9ull) ^ ((uint64_t)n << 47);
    z ^= z >> 31;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 29;
    return z | 1ull;
}

__device__ __forceinline__ ulonglong2 ld_relaxed_u64x2(const uint64_t *p) {
    ulonglong2 v;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ bool cc_find(pga::CCSlot *T, uint32_t mask, uint64_t k1, uint64_t k2, uint32_t n,
                                        long long *v) {
    uint32_t i = (uint32_t)(k1 >> 17) & mask;
    for (int r = 0; r < CC_PROBE; ++r) {
        // the whole 32-byte slot in one round trip (two 16-byte loads in flight)
        const ulonglong2 h = ld_relaxed_u64x2(&T[i].k1);
        const ulonglong2 t = ld_relaxed_u64x2(reinterpret_cast<const uint64_t *>(&T[i].v));
        const uint64_t s1 = h.x;
        if (s1 == 0) return false;
        if (s1 == k1) {
            const uint64_t s2 = h.y;
            const long long sv = (long long)t.x;
            const uint64_t sc = t.y;
            if (s2 != k2 || sc != cc_mix(k1, k2, sv, n)) return false;
            *v = sv;
            return true;
        }
        i = (i + 1) & mask;
    }
    return false;
}

__device__ __forceinline__ void cc_insert(pga::CCSlot *T, uint32_t mask, uint32_t *fill, uint64_t k1,
                                          uint64_t k2, uint32_t n, long long v) {
    uint32_t i = (uint32_t)(k1 >> 17) & mask;
    for (int r = 0; r < CC_PROBE; ++r) {
        const unsigned long long old =
            atomicCAS(reinterpret_cast<unsigned long long *>(&T[i].k1), 0ull, (unsigned long long)k1);
        if (old == 0ull) {
            T[i].k2 = k2;
            T[i].v = v;
            T[i].chk = cc_mix(k1, k2, v, n);
            atomicAdd(fill, 1u);
            return;
        }
        if (old == k1) return;   // inserted by another chromosome
        i = (i + 1) & mask;
    }
}

struct SparseArgs {
    const uint16_t *cm0, *cm1;
    uint16_t *gm0, *gm1;          // gene-major labels: written here for blocks found dense (GA mode)
    int64_t Pcap;
    const double *C;
    int ldc, N, ldn;
    int64_t P;
    int cb0;
    const double *diag;
    double *L;
    uint16_t *top;
    const int32_t *gen, *done;
    uint8_t *sflag;
    uint32_t max_pairs;           // sparse iff every chromosome needs <= max_pairs pair updates
    int32_t *live;                // GA hysteresis [0]: any block went sparse last launch, [1] any now, [2] CTA count; null = always check
    unsigned long long *nsparse;  // [0] blocks evaluated here, [1] C entries gathered, [2] cache hits, [3] pairs they saved (profiling)
    int nblocks;
    double fx_scale, fx_inv;
    const double *lgn, *lgnn;
    const double2 *lnt;           // fast_ln table (after lgn, lgnn in the ctx's lgtab)
    const double *ptab;           // [N][ldc] Eq. 8 term of every pair cluster {i, j} (k_pairtab)
    pga::CCSlot *cc;              // cluster cache (null = off)
    uint32_t cc_mask;             // slots - 1
    uint32_t *cc_state;           // [0] fill, [1] clear request, [2] CTA count, [3] clears done
    const uint64_t *cc_keys;      // [N][2] Zobrist keys
    uint32_t stage_off;           // != 0: keys and fixed-point diagonal staged in shared memory at this offset
};

__host__ __device__ __forceinline__ int sp_words(int N) { return (N + 2) / 2; }   // packed u16 counters for labels 0..N

// Per-warp shared memory of the label-sparse pass (bytes, 16-aligned):
//   A [16 E]  cent: Zobrist keys {k1, k2} per ordinal, then the Eq. 8 term
//   B [16 E]  perm2: walked genes (g | ordinal << 16); before that the
//             second Zobrist copy
//   (during counting and the small pass A+B hold mem [SMALL_N (N+1)] u16,
//    the first members of every label, and slist [N/2 + 1] u16)
//   cq [4 (W + 1)]  packed u16 counts, then ordm (u16 per label); during the
//             walk, c of every walked cluster (fp64 per ordinal: 8 E <= 4 (W + 1))
//   wen [4 E] walk range ends per ordinal
//   cn, clab [2 E each] n (| 0x8000: cache hit), label per ordinal
__host__ __device__ __forceinline__ size_t sp_per_warp(int N) {
    const size_t E = (size_t)cc_entries(N);
    return ((32 * E + ((size_t)sp_words(N) + 1) * 4 + 8 * E + 64) + 15) & ~(size_t)15;
}

static size_t sparse_smem(int N) {
    const size_t warps = (size_t)sp_warps(N) * sp_per_warp(N) + 64;
    const size_t tile = (size_t)N * (pga::CB + 2) * sizeof(uint16_t);   // dense-block transpose
    return warps > tile ? warps : tile;
}

// Staged per CTA after the warps' tables (when it costs no occupancy): the
// Zobrist keys (16 B per gene) and the fixed-point diagonal (8 B per gene),
// read by every cacheable gene's XOR and every walked / triple cluster.
static size_t sparse_stage_off(int N) { return ((size_t)sp_warps(N) * sp_per_warp(N) + 64 + 15) & ~(size_t)15; }
static size_t sparse_smem_staged(int N) {
    const size_t st = sparse_stage_off(N) + 24 * (size_t)N;
    const size_t base = sparse_smem(N);
    return st > base ? st : base;
}
static bool sparse_stage_ok(int N) {
    if (std::getenv("PGA_NO_SP_STAGE")) return false;
    const size_t smem_sm = 228 * 1024, per_cta_extra = 1024, max_cta = 227 * 1024;
    const size_t a = sparse_smem(N), b = sparse_smem_staged(N);
    if (b > max_cta) return false;
    if ((size_t)N * (pga::CB + 2) * sizeof(uint16_t) > sparse_stage_off(N)) return false;   // transpose tile
    const size_t ca = std::min<size_t>(2, smem_sm / (a + per_cta_extra)), cb = std::min<size_t>(2, smem_sm / (b + per_cta_extra));
    return cb >= ca;
}

template <int LREG, int SPW>
__global__ void __launch_bounds__(SPW * 32, SPW == 16 ? PGA_SP_MINB : 1) k_fitness_sparse(SparseArgs a) {
    constexpr int SP_T = SPW * 32;
    pdl_wait();
    pdl_trigger();
    if (a.done && *a.done) return;
    extern __shared__ __align__(16) unsigned char sps[];
    __shared__ uint32_t s_maxp;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int N = a.N, W = sp_words(N);
    const int cb = a.cb0 + blockIdx.x;
    const int par = (a.gen && (*a.gen & 1)) ? 1 : 0;
    const uint16_t *CM = par ? a.cm1 : a.cm0;
    unsigned char *wb = sps + (size_t)warp * sp_per_warp(N);
    const int E = cc_entries(N);
    ulonglong2 *cent = reinterpret_cast<ulonglong2 *>(wb);              // A [E] Zobrist keys {k1, k2}, then {f, -}
    uint32_t *perm2 = reinterpret_cast<uint32_t *>(cent + E);           // B [4 E] walked genes g | ordinal << 16
    uint32_t *cent2 = perm2;                                             // B: second Zobrist copy (before the walk)
    uint16_t *mem = reinterpret_cast<uint16_t *>(wb);                   // A+B [SMALL_N (N+1)]: first members per label
    uint16_t *slist = mem + SMALL_N * (N + 1);                           // A+B [N/2 + 1]: small labels
    uint32_t *cq = perm2 + 4 * E;                                        // [W] packed u16 counts, then ordm
    uint32_t *wen = cq + W + 1;                                          // [E] walk range ends
    double *cval = reinterpret_cast<double *>(cq);                       // [E] walked clusters' c (after the sort)
    uint16_t *cn = reinterpret_cast<uint16_t *>(wen + E);               // [E] n (| 0x8000: cache hit)
    uint16_t *clab = cn + E;                                             // [E] label
    if (a.live && a.live[0] == 0) {     // the population went dense: skip (flags cleared)
        if (tid == 0) a.sflag[cb] = 0;
        return;
    }
    // every block was sparse at the last check: evaluate sparsely without
    // checking, except on every 16th launch (the population densifies)
    const bool skip1 = a.live && a.live[3] != 0 && (a.live[5] & 15) != 0;
    // cache clear request (the table is half full): this launch clears it
    // and neither reads nor writes it
    const bool cc_clear = a.cc && *reinterpret_cast<volatile uint32_t *>(a.cc_state + 1) != 0u;
    const bool use_cache = a.cc && !cc_clear;
    if (tid == 0) s_maxp = 0u;
    const bool stage = a.stage_off != 0u;
    uint4 *skeys = reinterpret_cast<uint4 *>(sps + a.stage_off);
    long long *sdfx = reinterpret_cast<long long *>(skeys + N);
    if (stage) {
        if (a.cc)
            for (int i = tid; i < N; i += SP_T) skeys[i] = __ldg(reinterpret_cast<const uint4 *>(a.cc_keys) + i);
        for (int i = tid; i < N; i += SP_T) sdfx[i] = __double2ll_rn(__ldg(a.diag + i) * a.fx_scale);
    }
    __syncthreads();
    if (!skip1) {

    // ---- pass 1: cluster sizes and pair counts
    for (int q = warp; q < pga::CB; q += SPW) {
        const int64_t p = (int64_t)cb * pga::CB + q;
        for (int k = lane; k < W; k += 32) cq[k] = 0u;
        __syncwarp();
        if (p < a.P)
            for (int i = lane; i < N; i += 32) {
                const uint32_t s = CM[p * a.ldn + i];
                atomicAdd(cq + (s >> 1), 1u << (16 * (s & 1u)));
            }
        __syncwarp();
        uint32_t pairs = 0;
        for (int k = lane; k < W; k += 32) {
            const uint32_t w2 = cq[k], n0 = w2 & 0xFFFFu, n1 = w2 >> 16;
            pairs += n0 * (n0 - (n0 > 0)) / 2 + n1 * (n1 - (n1 > 0)) / 2;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pairs += __shfl_xor_sync(0xFFFFFFFFu, pairs, o);
        if (lane == 0) atomicMax(&s_maxp, pairs);
        __syncwarp();
    }
    }   // !skip1
    __syncthreads();
    const bool sparse = skip1 || s_maxp <= a.max_pairs;
    if (!sparse && a.live) {
        // GA mode: while sparse checks run, the breed leaves the gene-major
        // copy to us -- transpose this block's labels for the dense sweep
        uint16_t *GM = par ? a.gm1 : a.gm0;
        uint16_t *tile = reinterpret_cast<uint16_t *>(sps);          // [N][CB + 2]
        constexpr int TSP = pga::CB + 2;
        for (int e = tid; e < pga::CB * N; e += SP_T) {
            const int q = e / N, i = e - q * N;
            const int64_t p = (int64_t)cb * pga::CB + q;
            tile[i * TSP + q] = p < a.P ? CM[p * a.ldn + i] : (uint16_t)0;
        }
        __syncthreads();
        for (int e = tid; e < N * (pga::CB / 2); e += SP_T) {
            const int i = e / (pga::CB / 2), pr = e - i * (pga::CB / 2);
            *reinterpret_cast<uint32_t *>(&GM[(int64_t)i * a.Pcap + (int64_t)cb * pga::CB + 2 * pr]) =
                *reinterpret_cast<const uint32_t *>(&tile[i * TSP + 2 * pr]);
        }
    }
    if (cc_clear) {
        const uint32_t slots = a.cc_mask + 1u, per = (slots + gridDim.x - 1) / gridDim.x;
        const uint32_t lo = blockIdx.x * per, hi = min(slots, lo + per);
        for (uint32_t i = lo + tid; i < hi; i += SP_T) a.cc[i] = pga::CCSlot{};
    }
    if (a.cc && tid == 0) {
        // the last CTA to get here toggles the clear request (CTAs read it at
        // their start, and all have started by then)
        __threadfence();
        if (atomicAdd(a.cc_state + 2, 1u) == gridDim.x - 1) {
            if (cc_clear) {
                a.cc_state[0] = 0u;
                a.cc_state[1] = 0u;
                a.cc_state[3] += 1u;   // clears so far (pga_cache_stats)
            } else if (atomicAdd(a.cc_state, 0u) > (a.cc_mask >> 1)) {
                a.cc_state[1] = 1u;
            }
            a.cc_state[2] = 0u;
        }
    }
    if (tid == 0) {
        a.sflag[cb] = sparse ? 1 : 0;
        if (sparse && a.nsparse) atomicAdd(a.nsparse, 1ull);
        if (a.live) {
            // live: [0] any block sparse at the last check, [1] accumulator,
            // [2] CTA count, [3] every block sparse at the last check, [4]
            // dense-block count, [5] launch count.  The last CTA publishes.
            if (sparse) atomicOr(&a.live[1], 1);
            else atomicAdd(&a.live[4], 1);
            __threadfence();
            if (atomicAdd(&a.live[2], 1) == a.nblocks - 1) {
                const int any = atomicExch(&a.live[1], 0);
                const int dense = atomicExch(&a.live[4], 0);
                if (!skip1) {
                    a.live[0] = any;
                    a.live[3] = dense == 0;
                }
                a.live[2] = 0;
                a.live[5] += 1;
            }
        }
    }
    if (!sparse) return;

    // ---- pass 2: exact label-sparse evaluation.  Per chromosome: (1) counts,
    // recording each label's first SMALL_N members; (2) classes: small
    // clusters (2 <= n < WALK_N) are listed, walk-class clusters (n >=
    // WALK_N) get ordinals in label order; (3) small clusters lane-parallel:
    // c from their recorded members (n = 2: the pair-term table), Eq. 8 term
    // at once; (4) Zobrist keys of cacheable clusters (n >= CC_NMIN) and one
    // lookup each; (5)-(7) the walk-class clusters that were not hits are
    // counting-sorted by ordinal and walked (every unordered pair once, L2
    // gathers of C, exact fixed-point sums), their terms stored per ordinal
    // (and inserted into the cache); (8) the walk-class terms are summed in
    // ordinal (= label) order, so L does not depend on which came from the
    // cache.  c sums are exact fixed-point integers (order-free), so every
    // term is deterministic.
    const double *C = a.C;
    const uint4 *keys4 = reinterpret_cast<const uint4 *>(a.cc_keys);
    uint16_t *ordm = reinterpret_cast<uint16_t *>(cq);
    for (int q = warp; q < pga::CB; q += SPW) {
        const int64_t p = (int64_t)cb * pga::CB + q;
        if (p >= a.P) break;
        for (int k = lane; k < W; k += 32) cq[k] = 0u;
        __syncwarp();
        const uint16_t *lab = CM + p * a.ldn;
        uint32_t kmax = 0;
        // the chromosome's labels stay in registers for the passes over
        // them: gene 64 (k >> 1) + 2 lane + (k & 1) is half (k & 1) of
        // labr[k >> 1] (one aligned 32-bit load per gene pair; ldn is even)
        uint32_t labr[LREG];
#pragma unroll
        for (int k = 0; k < LREG; ++k) {
            const int i = 64 * k + 2 * lane;
            labr[k] = i < N ? *reinterpret_cast<const uint32_t *>(lab + i) : 0u;
        }
        // (1) counts; the count before a gene's increment is its slot
#pragma unroll
        for (int k = 0; k < 2 * LREG; ++k) {
            const int i = 64 * (k >> 1) + 2 * lane + (k & 1);
            if (i < N) {
                const uint32_t s = (labr[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
                kmax = max(kmax, s);
                const uint32_t sh = 16 * (s & 1u);
                PGA_DCHECK(s < (uint32_t)N);
                const uint32_t slot = (atomicAdd(cq + (s >> 1), 1u << sh) >> sh) & 0xFFFFu;
                if (slot < (uint32_t)SMALL_N) mem[SMALL_N * s + slot] = (uint16_t)i;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) kmax = max(kmax, __shfl_xor_sync(0xFFFFFFFFu, kmax, o));
        const int K = min((int)kmax + 1, N);
        __syncwarp();
        // (2) classes.  ordm[k] (in place over the 16-bit count): 0x8000 | n
        // below the walk class, else the ordinal | 0x2000 if cacheable;
        // bit 0x4000 is set below for cache hits
        int ecnt = 0, scnt = 0;
        for (int k0 = 0; k0 < K; k0 += 32) {
            const int k = k0 + lane;
            const int n = k < K ? (int)ordm[k] : 0;
            const bool el = n >= WALK_N, sm = n >= 2 && n < WALK_N;
            const unsigned be = __ballot_sync(0xFFFFFFFFu, el), bs = __ballot_sync(0xFFFFFFFFu, sm);
            if (el) {
                const int ord = ecnt + __popc(be & lanemask_lt());
                PGA_DCHECK(ord < E);
                ordm[k] = (uint16_t)(ord | (n >= CC_NMIN ? 0x2000 : 0));
                cn[ord] = (uint16_t)n;
                clab[ord] = (uint16_t)k;
            } else if (k < K) {
                ordm[k] = (uint16_t)(0x8000 | n);
                PGA_DCHECK(!sm || scnt + __popc(bs & lanemask_lt()) <= N / 2);
                if (sm) slist[scnt + __popc(bs & lanemask_lt())] = (uint16_t)k;
            }
            ecnt += __popc(be);
            scnt += __popc(bs);
        }
        __syncwarp();
        // (3) small clusters, one per lane: no walk, no queue
        uint32_t nhit = 0, nsaved = 0, npair = 0;   // per chromosome: < 2^32 (N <= 2048)
        double fsum = 0.0, fbest = 0.0;
        int kbest = 0x7FFFFFFF;
        for (int j = lane; j < scnt; j += 32) {
            const int sl = (int)slist[j];
            const int n = (int)(ordm[sl] & 0x7FFFu);
            const int g0 = mem[SMALL_N * sl], g1 = mem[SMALL_N * sl + 1];
            double f;
            if (n == 2) {
                f = __ldg(a.ptab + (size_t)g0 * a.ldc + g1);
                npair += 1;
            } else {
                const int g2 = mem[SMALL_N * sl + 2];
                const long long dsum =
                    stage ? sdfx[g0] + sdfx[g1] + sdfx[g2]
                          : __double2ll_rn(__ldg(a.diag + g0) * a.fx_scale) +
                                __double2ll_rn(__ldg(a.diag + g1) * a.fx_scale) +
                                __double2ll_rn(__ldg(a.diag + g2) * a.fx_scale);
                const long long acc =
                    dsum +
                    2 * (__double2ll_rn(__ldg(C + (size_t)g0 * a.ldc + g1) * a.fx_scale) +
                         __double2ll_rn(__ldg(C + (size_t)g0 * a.ldc + g2) * a.fx_scale) +
                         __double2ll_rn(__ldg(C + (size_t)g1 * a.ldc + g2) * a.fx_scale));
                f = eq8_term_fast(n, (double)acc * a.fx_inv, a.lgn, a.lgnn, a.lnt);
                npair += 3;
            }
            fsum += f;
            if (f > fbest || (f == fbest && f > 0.0 && sl < kbest)) {
                fbest = f;
                kbest = sl;
            }
        }
        __syncwarp();   // mem and slist (regions A+B) are dead from here
        // (4) Zobrist XOR of each cacheable cluster's members; the odd lanes
        // XOR into the second copy (halves same-address collisions of the
        // shared atomics); the copies are XORed at the lookup (order-free)
        if (use_cache && ecnt > 0) {
            for (int o = lane; o < ecnt; o += 32) {
                cent[o] = make_ulonglong2(0ull, 0ull);
                cent2[4 * o] = cent2[4 * o + 1] = cent2[4 * o + 2] = cent2[4 * o + 3] = 0u;
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 2 * LREG; ++k) {
                const int i = 64 * (k >> 1) + 2 * lane + (k & 1);
                if (i >= N) continue;
                const uint32_t om = ordm[(labr[k >> 1] >> (16 * (k & 1))) & 0xFFFFu];
                if ((om & 0xA000u) == 0x2000u) {
                    const uint32_t o = om & 0x1FFFu;
                    uint32_t *h = (lane & 1) ? cent2 + 4 * o : reinterpret_cast<uint32_t *>(cent + o);
                    const uint4 kk = stage ? skeys[i] : __ldg(keys4 + i);
                    atomicXor(h, kk.x);
                    atomicXor(h + 1, kk.y);
                    atomicXor(h + 2, kk.z);
                    atomicXor(h + 3, kk.w);
                }
            }
            __syncwarp();
            // one lookup per cacheable cluster, lane-parallel; a hit is its
            // Eq. 8 term and the cluster is not walked
            for (int o = lane; o < ecnt; o += 32) {
                const uint32_t n = cn[o];
                if (n < (uint32_t)CC_NMIN) continue;
                ulonglong2 h = cent[o];
                const uint32_t *c2 = cent2 + 4 * o;
                h.x ^= (unsigned long long)c2[0] | ((unsigned long long)c2[1] << 32);
                h.y ^= (unsigned long long)c2[2] | ((unsigned long long)c2[3] << 32);
                const uint64_t k1 = h.x | 1ull, k2 = h.y | 1ull;
                long long v = 0;
                cent[o] = make_ulonglong2(k1, k2);
                if (cc_find(a.cc, a.cc_mask, k1, k2, n, &v)) {
                    cent[o].x = (unsigned long long)v;          // the cached Eq. 8 term
                    cn[o] = (uint16_t)(n | 0x8000u);
                    ordm[clab[o]] |= 0x4000u;
                    nhit += 1;
                    nsaved += n * (n - 1) / 2;
                }
            }
            __syncwarp();
        }
        // (5) walk ranges: walk-class clusters that are not hits, in ordinal
        // order (exclusive prefix); wen[o] = start, the end after (6)
        int base = 0;
        for (int o0 = 0; o0 < ecnt; o0 += 32) {
            const int o = o0 + lane;
            int w = 0;
            if (o < ecnt) {
                const uint32_t n = cn[o];
                w = (n & 0x8000u) ? 0 : (int)n;
            }
            int incl = w;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= d) incl += t;
            }
            if (o < ecnt) wen[o] = (uint32_t)(base + incl - w);
            base += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
        const int Nw = base;
        __syncwarp();
        // (6) counting sort of the walked genes by ordinal (order inside a
        // cluster is free: sums are exact)
        if (Nw > 0) {
#pragma unroll
            for (int k = 0; k < 2 * LREG; ++k) {
                const int i = 64 * (k >> 1) + 2 * lane + (k & 1);
                if (i >= N) continue;
                const uint32_t om = ordm[(labr[k >> 1] >> (16 * (k & 1))) & 0xFFFFu];
                if (!(om & 0xC000u)) {
                    const uint32_t o = om & 0x1FFFu;
                    const uint32_t pos = atomicAdd(wen + o, 1u);
                    PGA_DCHECK(o < (uint32_t)ecnt && pos < (uint32_t)Nw);
                    perm2[pos] = (uint32_t)i | (o << 16);
                }
            }
            __syncwarp();
        }
        // (7) walk the sorted genes 32 at a time.  A lane's group is the
        // window's lanes of its cluster (contiguous); the cluster open at the
        // window's end carries on.  A completed cluster stores its c at its
        // ordinal (ordm is dead: cval overlays it); its Eq. 8 term is taken
        // lane-parallel in (8).
        long long carry = 0;
        for (int t0 = 0; t0 < Nw; t0 += 32) {
            const int t = t0 + lane;
            int o = -1, st = t, en = t + 1, n = 0;
            long long acc = 0;
            if (t < Nw) {
                const uint32_t pg = perm2[t];
                const int g = (int)(pg & 0xFFFFu);
                o = (int)(pg >> 16);
                en = (int)wen[o];
                n = (int)cn[o];
                st = en - n;
                const int av = t - st;
                if (av == 0) npair += (uint32_t)(n * (n - 1) / 2);   // C pairs gathered, once per cluster
                const double *Cg = C + (size_t)g * a.ldc;
                acc = stage ? sdfx[g] : __double2ll_rn(__ldg(a.diag + g) * a.fx_scale);
                const int h = (n - 1) >> 1;
                int bidx = av;
#pragma unroll 4
                for (int d = 1; d <= h; ++d) {
                    bidx = (bidx + 1 == n) ? 0 : bidx + 1;
                    acc += 2 * __double2ll_rn(__ldg(Cg + (perm2[st + bidx] & 0xFFFFu)) * a.fx_scale);
                }
                if (!(n & 1) && av < (n >> 1))
                    acc += 2 * __double2ll_rn(__ldg(Cg + (perm2[st + av + (n >> 1)] & 0xFFFFu)) * a.fx_scale);
            }
            // group sum = difference of the window's inclusive prefix sums at
            // the group's ends (mod 2^64: exact)
            const int lo = max(st - t0, 0), hi = min(en - t0, 32);
            unsigned long long pre = (unsigned long long)acc;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, pre, d);
                if (lane >= d) pre += v;
            }
            const unsigned long long phi = __shfl_sync(0xFFFFFFFFu, pre, hi - 1);
            const unsigned long long plo = __shfl_sync(0xFFFFFFFFu, pre, lo > 0 ? lo - 1 : 0);
            long long tot = (long long)(phi - (lo > 0 ? plo : 0ull));
            if (o >= 0 && st < t0) tot += carry;                 // continues from the last window
            const int o31 = __shfl_sync(0xFFFFFFFFu, o, 31);
            const int en31 = __shfl_sync(0xFFFFFFFFu, en, 31);
            const long long tot31 = __shfl_sync(0xFFFFFFFFu, tot, 31);
            carry = (o31 >= 0 && en31 > t0 + 32) ? tot31 : 0ll;
            PGA_DCHECK(o < 0 || (o < ecnt && st >= 0 && en <= Nw && n >= WALK_N));
            if (o >= 0 && lane == lo && en <= t0 + 32) cval[o] = (double)tot * a.fx_inv;
        }
        __syncwarp();
        // (8) the walk-class terms, in ordinal (= label) order per lane: a hit
        // is the cached term; a walked cluster's term is computed here (and
        // inserted into the cache when cacheable)
        for (int o = lane; o < ecnt; o += 32) {
            const uint32_t nh = cn[o];
            double f;
            if (nh & 0x8000u) {
                f = __longlong_as_double((long long)cent[o].x);
            } else {
                f = eq8_term_fast((int)nh, cval[o], a.lgn, a.lgnn, a.lnt);
                if (use_cache && nh >= (uint32_t)CC_NMIN) {
                    const ulonglong2 e = cent[o];
                    cc_insert(a.cc, a.cc_mask, a.cc_state, e.x, e.y, nh, __double_as_longlong(f));
                }
            }
            fsum += f;
            const int kl = (int)clab[o];
            if (f > fbest || (f == fbest && f > 0.0 && kl < kbest)) {
                fbest = f;
                kbest = kl;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            fsum += __shfl_xor_sync(0xFFFFFFFFu, fsum, o);
            const double of = __shfl_xor_sync(0xFFFFFFFFu, fbest, o);
            const int ok = __shfl_xor_sync(0xFFFFFFFFu, kbest, o);
            if (of > fbest || (of == fbest && ok < kbest)) {
                fbest = of;
                kbest = ok;
            }
        }
        if (a.nsparse) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                npair += __shfl_xor_sync(0xFFFFFFFFu, npair, o);
                nhit += __shfl_xor_sync(0xFFFFFFFFu, nhit, o);
                nsaved += __shfl_xor_sync(0xFFFFFFFFu, nsaved, o);
            }
            if (lane == 0) {
                atomicAdd(a.nsparse + 1, (unsigned long long)npair);
                atomicAdd(a.nsparse + 2, (unsigned long long)nhit);
                atomicAdd(a.nsparse + 3, (unsigned long long)nsaved);
            }
        }
        if (lane == 0) {
            a.L[p] = 0.5 * fsum;
            if (a.top) a.top[p] = (fbest > 0.0) ? (uint16_t)kbest : (uint16_t)0xFFFF;
        }
        __syncwarp();
    }
}

// Eq. 8 term of every pair cluster {i, j} (the label-sparse pass's n = 2
// clusters): c = C_ii + C_jj + 2 C_ij in the pass's fixed point, then the
// same eq8_term_fast -- identical to what a walk of that pair would give.
__global__ void k_pairtab(const double *__restrict__ C, int ldc, const double *__restrict__ diag, int N,
                          double fx_scale, double fx_inv, const double *__restrict__ lgn,
                          const double *__restrict__ lgnn, const double2 *__restrict__ lnt, double *T) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    if (j >= N) return;
    const long long acc = __double2ll_rn(diag[i] * fx_scale) + __double2ll_rn(diag[j] * fx_scale) +
                          2 * __double2ll_rn(C[(size_t)i * ldc + j] * fx_scale);
    T[(size_t)i * ldc + j] = (i == j) ? 0.0 : eq8_term_fast(2, (double)acc * fx_inv, lgn, lgnn, lnt);
}

}  // namespace

PGA_VIOL_READER(viol_fitness)

namespace pga {

int launch_resync_gm(pga_ctx *c, cudaStream_t s) {
    dim3 grid((unsigned)((c->P + 31) / 32), (unsigned)((c->N + 31) / 32));
    k_resync_gm<<<grid, dim3(32, 8), 0, s>>>(c->pop[0], c->pop[1], c->popT[0], c->popT[1], c->st, c->P, c->N,
                                             c->ldn, c->Pcap);
    PGA_LAUNCHED();
    return PGA_OK;
}

int launch_pack(pga_ctx *c, const uint16_t *lab16, const int32_t *lab32, int64_t P, int ld_in,
                uint16_t *CM, uint16_t *GM, cudaStream_t s) {
    dim3 grid((unsigned)((P + 31) / 32), (unsigned)((c->N + 31) / 32));
    k_pack<<<grid, dim3(32, 8), 0, s>>>(lab16, lab32, P, ld_in, c->N, c->ldn, c->Pcap, CM, GM, c->st);
    PGA_LAUNCHED();
    return PGA_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encode() {
    if (g_encode) return PGA_OK;
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    PGA_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(PGA_EDEVICE, "cuTensorMapEncodeTiled unavailable");
    g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    return PGA_OK;
}

// labels: gene-major [N][Pcap] u16, box {64, KC}
int make_label_tmap(CUtensorMap *tm, const uint16_t *GM, int N, int64_t Pcap) {
    if (get_encode()) return PGA_EDEVICE;
    cuuint64_t dims[2] = {(cuuint64_t)Pcap, (cuuint64_t)N};
    cuuint64_t strides[1] = {(cuuint64_t)Pcap * 2};
    cuuint32_t box[2] = {(cuuint32_t)CB, (cuuint32_t)KC};
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, (void *)GM, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PGA_EDEVICE, "cuTensorMapEncodeTiled (labels) failed");
    return PGA_OK;
}

// C: [N][ldc] fp64, box {RT, KC}
int make_c_tmap(CUtensorMap *tm, const double *C, int N, int ldc) {
    if (get_encode()) return PGA_EDEVICE;
    cuuint64_t dims[2] = {(cuuint64_t)ldc, (cuuint64_t)N};
    cuuint64_t strides[1] = {(cuuint64_t)ldc * 8};
    cuuint32_t box[2] = {(cuuint32_t)RT, (cuuint32_t)KC};
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)C, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PGA_EDEVICE, "cuTensorMapEncodeTiled (C) failed");
    return PGA_OK;
}

__global__ void k_logtab(int N, double *t) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n < LN_TAB) {   // fast_ln table: ln c_j, 1 / c_j
        const double c = 1.0 + (n + 0.5) / (double)LN_TAB;
        t[2 * (N + 1) + 2 * n] = log(c);
        t[2 * (N + 1) + 2 * n + 1] = 1.0 / c;
    }
    if (n > N) return;
    t[n] = n >= 1 ? log((double)n) : 0.0;
    t[N + 1 + n] = n >= 2 ? log((double)n * n - n) : 0.0;
}

// Test hook kernel: fast_ln of x[0..n) (tests/test_gpu_checks.py).
__global__ void k_fast_ln(const double *x, int64_t n, const double *tab, double *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = fast_ln(x[i], reinterpret_cast<const double2 *>(tab));
}

int launch_logtab(pga_ctx *c, cudaStream_t s) {
    k_logtab<<<(std::max(c->N + 1, LN_TAB) + 255) / 256, 256, 0, s>>>(c->N, c->lgtab);
    PGA_LAUNCHED();
    return PGA_OK;
}

// fold / label-sparse fixed point: S = 62 - ceil(log2(2 N^2 + 1)), so no
// cluster sum of |C| <= 1 entries (|sum| <= 2 N^2) can overflow int64
void fx_scale_of(int N, double *scale, double *inv) {
    int bits = 0;
    while ((1.0 * (1ull << bits)) < 2.0 * N * N + 1.0) ++bits;
    *scale = ldexp(1.0, 62 - bits);
    *inv = ldexp(1.0, bits - 62);
}

int launch_fast_ln(const double *x, int64_t n, const double *lgtab, int N, double *out, cudaStream_t s) {
    k_fast_ln<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, n, lgtab + 2 * (N + 1), out);
    PGA_LAUNCHED();
    return PGA_OK;
}

int launch_pairtab(pga_ctx *c, cudaStream_t s) {
    if (!c->ptab) return PGA_OK;
    double sc, inv;
    fx_scale_of(c->N, &sc, &inv);
    dim3 grid((unsigned)((c->N + 127) / 128), (unsigned)c->N);
    k_pairtab<<<grid, 128, 0, s>>>(c->C, c->ldc, c->diag, c->N, sc, inv, c->lgtab, c->lgtab + (c->N + 1),
                                   reinterpret_cast<const double2 *>(c->lgtab + 2 * (c->N + 1)), c->ptab);
    PGA_LAUNCHED();
    return PGA_OK;
}

int fold_warps(int N) {
    const size_t per = 2 * (size_t)N * (sizeof(double) + sizeof(int32_t));   // NCF = 2 chromosomes per warp
    int w = (int)((size_t)(NSTAGE * STAGE_BYTES) / per);
    if (w < 1) w = 1;
    return w > CW + 1 ? CW + 1 : w;
}

size_t fitness_smem(int N) {
    const size_t fold = (size_t)fold_warps(N) * (2 * N * (sizeof(double) + sizeof(int32_t))) + 16;
    const size_t pipe = (size_t)NSTAGE * STAGE_BYTES;
    return (fold > pipe ? fold : pipe) + 2 * NSTAGE * sizeof(uint64_t) + 128;
}

int prepare_fitness(int N) {
    PGA_CUDA(cudaFuncSetAttribute(k_fitness, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)fitness_smem(N)));
    if (N <= SPARSE_SMALLN)
        PGA_CUDA(cudaFuncSetAttribute(k_fitness_sparse<SPARSE_SMALLN / 64, 16>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sparse_stage_ok(N) ? sparse_smem_staged(N) : sparse_smem(N))));
    else if (N <= SPARSE_MAXN)
        PGA_CUDA(cudaFuncSetAttribute(k_fitness_sparse<SPARSE_MAXN / 64, 8>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sparse_stage_ok(N) ? sparse_smem_staged(N) : sparse_smem(N))));
    return PGA_OK;
}

int launch_fitness(pga_ctx *c, const FitBufs &b, int64_t P, double *L, uint16_t *top,
                   cudaStream_t s, cudaEvent_t *ev) {
    return launch_fitness_range(c, b, 0, P, L, top, s, ev);
}

// chromosomes [begin, end) (begin a multiple of CB); L[p], top[p] are written
// at the GLOBAL index p.
int launch_fitness_range(pga_ctx *c, const FitBufs &b, int64_t begin, int64_t end, double *L,
                         uint16_t *top, cudaStream_t s, cudaEvent_t *ev) {
    const int N = c->N;
    const int64_t P = end;
    FitArgs a;
    a.N = N;
    a.ldn = c->ldn;
    a.nRT = (N + RT - 1) / RT;
    a.cb0 = (int)(begin / CB);
    a.lgn = c->lgtab;
    a.lgnn = c->lgtab + (N + 1);
    a.lnt = reinterpret_cast<const double2 *>(c->lgtab + 2 * (N + 1));
    fx_scale_of(N, &a.fx_scale, &a.fx_inv);   // |sum of V over a cluster| <= 2 N^2
    a.nCB = (int)((end - begin + CB - 1) / CB);
    a.fold_warps = fold_warps(N);
    a.P = P;
    a.Pcap = c->Pcap;
    a.gm0 = b.gm0;
    a.gm1 = b.gm1;
    a.diag = c->diag;
    a.V = c->V;
    a.cm0 = b.cm0;
    a.cm1 = b.cm1;
    a.L = L;
    a.top = top;
    a.gen = b.gen;
    a.done = b.done;
    a.counters = c->counters;
    if (ev) PGA_CUDA(prof_record(ev[0], s));
    a.sflag = nullptr;
    if (sparse_theta_eff(c) > 0.0 && N <= SPARSE_MAXN && c->sflag && c->ptab) {
        // label-sparse pass first (f2); it flags the blocks it evaluated
        SparseArgs sp;
        sp.cm0 = b.cm0;
        sp.cm1 = b.cm1;
        sp.gm0 = const_cast<uint16_t *>(b.gm0);
        sp.gm1 = const_cast<uint16_t *>(b.gm1);
        sp.Pcap = c->Pcap;
        sp.C = c->C;
        sp.ldc = c->ldc;
        sp.N = N;
        sp.ldn = c->ldn;
        sp.P = P;
        sp.cb0 = a.cb0;
        sp.diag = c->diag;
        sp.L = L;
        sp.top = top;
        sp.gen = b.gen;
        sp.done = b.done;
        sp.sflag = c->sflag;
        const double dense = 0.5 * (double)N * (double)(N - 1);
        sp.max_pairs = (uint32_t)fmin(4.0e9, floor(sparse_theta_eff(c) * dense));
        sp.live = b.gen ? c->sp_live : nullptr;     // hysteresis for GA generations only
        sp.nblocks = a.nCB;
        sp.nsparse = c->sp_blocks;
        sp.fx_scale = a.fx_scale;
        sp.fx_inv = a.fx_inv;
        sp.lgn = a.lgn;
        sp.lgnn = a.lgnn;
        sp.lnt = reinterpret_cast<const double2 *>(c->lgtab + 2 * (N + 1));
        sp.ptab = c->ptab;
        sp.cc = c->cc_on ? c->cc : nullptr;
        sp.cc_mask = c->cc_mask;
        sp.cc_state = c->cc_state;
        sp.cc_keys = c->cc_keys;
        const bool stg = sparse_stage_ok(N);
        sp.stage_off = stg ? (uint32_t)sparse_stage_off(N) : 0u;
        const size_t sp_smem = stg ? sparse_smem_staged(N) : sparse_smem(N);
        if (N <= SPARSE_SMALLN)
            PGA_LAUNCH_PDL(k_fitness_sparse<SPARSE_SMALLN / 64, 16>, dim3((unsigned)a.nCB), dim3(16 * 32),
                           sp_smem, s, sp);
        else
            PGA_LAUNCH_PDL(k_fitness_sparse<SPARSE_MAXN / 64, 8>, dim3((unsigned)a.nCB), dim3(8 * 32),
                           sp_smem, s, sp);
        a.sflag = c->sflag;
    }
    if (ev) PGA_CUDA(prof_record(ev[1], s));   // dense kernel starts here
    {
        // row tiles per CTA: a whole chromosome block per CTA (all nRT tiles,
        // cpb = 1) when the label-sparse pass runs before this launch and
        // there are enough blocks to fill the GPU (>= 1024: C4, C5), else one
        // tile per CTA (a dense-only launch keeps the tiles of a block
        // concurrent, so their fold scratch V stays in L2: ncu DRAM 140 MB per
        // C4 launch with one tile per CTA, 185 MB with whole blocks).  Every CTA of a block exits at once
        // when the block went label-sparse, so in GA generations where the
        // sparse pass took every block this launch costs nCB instead of
        // nRT * nCB empty CTAs (C4: 8.2 instead of 22.5 us); a dense sweep
        // runs the same either way (C4: 1.447 vs 1.443 ms; uneven splits,
        // e.g. 6 + 2 tiles, measured slower: 1.58 ms).
        // GA generations with the sparse pass take whole blocks at any P (their
        // blocks are almost always all label-sparse: island-load 8 0.1152 ->
        // 0.1127 ms, island-load 4 0.1862 -> 0.1816 ms per generation)
        int F = (a.sflag && (a.nCB >= FIT_BLOCKS_PER_CTA_MIN || b.gen)) ? a.nRT : 1;
        if (const char *e = std::getenv("PGA_FIT_F")) F = std::max(1, std::min(a.nRT, std::atoi(e)));
        a.F = F;
        a.cpb = (a.nRT + F - 1) / F;
    }
    PGA_LAUNCH_PDL(k_fitness, dim3((unsigned)(a.cpb * a.nCB)), dim3(FIT_THREADS), fitness_smem(N), s, *b.tm0,
                   *b.tm1, c->tmC, a);
    if (ev) PGA_CUDA(prof_record(ev[2], s));   // sweep and fold are one fused kernel
    return PGA_OK;
}

}  // namespace pga
