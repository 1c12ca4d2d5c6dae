// fitness.cu — batched Giada–Marsili fitness (Eq. 5, 6, 8).
//
// Two kernels per evaluation:
//   k_sweep  the O(N^2 P) masked pair sweep.  One warp = 64 chromosomes
//            (two per lane) x TI = 8 rows i0..i0+7; it walks the columns j > i
//            of its rows and accumulates r'_i = sum_{j>i, s_j = s_i} C_ij in
//            fp64.  The label test is a packed fp16 compare (labels are stored
//            as raw 16-bit patterns, exact and never NaN for N < 31744) whose
//            1.0h/0.0h result, placed in the high word of a double, is exactly
//            2^-63 or 0; one DFMA then adds C_ij * 2^-63 or 0.  Per pair: one
//            HSET2 + one DFMA.  Output V[p][i] = C_ii + 2 r'_i.
//   k_fold   warp per chromosome: n_s by __match_any_sync/popc (exact),
//            c_s = sum_{i in s} V[p][i] in a fixed order (pointer-jumping
//            group sums, no float atomics -> deterministic), then Eq. 8 with
//            readings Q1-Q3, L = 1/2 sum f_s and top = argmax f_s.
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include "pga_internal.cuh"

namespace {

using namespace pgad;

__device__ __forceinline__ uint32_t heq(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("set.eq.f16x2.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// high word = 0x3C00xxxx pattern from heq (low half is always 0 by
// construction) -> the double 2^-63 or +0.
__device__ __forceinline__ double mask_d(uint32_t h) { return __hiloint2double((int)h, 0); }

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
// k_sweep
// grid.x = nRB (row blocks, ascending = longest first) * nQ; block = 4 warps,
// warp w handles chromosome block cb = q*4 + w of row block rb.
// ---------------------------------------------------------------------------
constexpr int SWEEP_WARPS = 4;

__global__ void __launch_bounds__(SWEEP_WARPS * 32)
k_sweep(const double *__restrict__ C, int ldc, const double *__restrict__ diag,
        const uint32_t *__restrict__ GM0, const uint32_t *__restrict__ GM1,
        const int32_t *__restrict__ gen_ptr,  // gene-major labels as u32 pairs [N][Pcap/2]
        int N, int64_t Pcap, int nCB, int nQ, double *__restrict__ V, int ldn,
        const int32_t *__restrict__ done_flag) {
    if (done_flag && *done_flag) return;
    const uint32_t *GM32 = (gen_ptr && (*gen_ptr & 1)) ? GM1 : GM0;
    const int rb = blockIdx.x / nQ;
    const int q = blockIdx.x - rb * nQ;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cb = q * SWEEP_WARPS + warp;
    if (cb >= nCB) return;
    const int i0 = rb * pga::TI;
    const int64_t half = Pcap >> 1;
    const uint32_t *lab = GM32 + (int64_t)cb * 32 + lane;   // + j * half

    // row labels, in the compare layout: (s_i << 16) | NaN
    uint32_t rowA[pga::TI], rowB[pga::TI];
#pragma unroll
    for (int r = 0; r < pga::TI; ++r) {
        const int i = i0 + r;
        uint32_t w = 0xFFFFFFFFu;
        if (i < N) w = __ldg(lab + (int64_t)i * half);
        rowA[r] = (w << 16) | 0x7FFFu;
        rowB[r] = (w & 0xFFFF0000u) | 0x7FFFu;
        if (i >= N) rowA[r] = rowB[r] = 0xFFFF7FFFu;   // NaN halves never match
    }
    double accA[pga::TI], accB[pga::TI];
#pragma unroll
    for (int r = 0; r < pga::TI; ++r) accA[r] = accB[r] = 0.0;

    // diagonal block: columns i0+1 .. i0+7, rows r < t only (pairs j > i)
#pragma unroll
    for (int t = 1; t < pga::TI; ++t) {
        const int j = i0 + t;
        if (j < N) {
            const uint32_t w = __ldg(lab + (int64_t)j * half);
            const uint32_t a = w << 16;
            const double *cj = C + (int64_t)j * ldc + i0;
#pragma unroll
            for (int r = 0; r < t; ++r) {
                const double c = __ldg(cj + r);
                accA[r] = fma(c, mask_d(heq(a, rowA[r])), accA[r]);
                accB[r] = fma(c, mask_d(heq(w, rowB[r])), accB[r]);
            }
        }
    }

    // main loop over full columns j >= i0 + TI
    int j = i0 + pga::TI;
#pragma unroll 1
    for (; j + 1 < N; j += 2) {
        const uint32_t w0 = __ldg(lab + (int64_t)j * half);
        const uint32_t w1 = __ldg(lab + (int64_t)(j + 1) * half);
        const double2 *c0p = reinterpret_cast<const double2 *>(C + (int64_t)j * ldc + i0);
        const double2 *c1p = reinterpret_cast<const double2 *>(C + (int64_t)(j + 1) * ldc + i0);
        double2 c0[4], c1[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            c0[k] = __ldg(c0p + k);
            c1[k] = __ldg(c1p + k);
        }
        const uint32_t a0 = w0 << 16, a1 = w1 << 16;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            accA[2 * k] = fma(c0[k].x, mask_d(heq(a0, rowA[2 * k])), accA[2 * k]);
            accB[2 * k] = fma(c0[k].x, mask_d(heq(w0, rowB[2 * k])), accB[2 * k]);
            accA[2 * k + 1] = fma(c0[k].y, mask_d(heq(a0, rowA[2 * k + 1])), accA[2 * k + 1]);
            accB[2 * k + 1] = fma(c0[k].y, mask_d(heq(w0, rowB[2 * k + 1])), accB[2 * k + 1]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            accA[2 * k] = fma(c1[k].x, mask_d(heq(a1, rowA[2 * k])), accA[2 * k]);
            accB[2 * k] = fma(c1[k].x, mask_d(heq(w1, rowB[2 * k])), accB[2 * k]);
            accA[2 * k + 1] = fma(c1[k].y, mask_d(heq(a1, rowA[2 * k + 1])), accA[2 * k + 1]);
            accB[2 * k + 1] = fma(c1[k].y, mask_d(heq(w1, rowB[2 * k + 1])), accB[2 * k + 1]);
        }
    }
    if (j < N) {
        const uint32_t w0 = __ldg(lab + (int64_t)j * half);
        const double2 *c0p = reinterpret_cast<const double2 *>(C + (int64_t)j * ldc + i0);
        const uint32_t a0 = w0 << 16;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 c = __ldg(c0p + k);
            accA[2 * k] = fma(c.x, mask_d(heq(a0, rowA[2 * k])), accA[2 * k]);
            accB[2 * k] = fma(c.x, mask_d(heq(w0, rowB[2 * k])), accB[2 * k]);
            accA[2 * k + 1] = fma(c.y, mask_d(heq(a0, rowA[2 * k + 1])), accA[2 * k + 1]);
            accB[2 * k + 1] = fma(c.y, mask_d(heq(w0, rowB[2 * k + 1])), accB[2 * k + 1]);
        }
    }

    // epilogue: V[p][i] = C_ii + 2 * 2^63 * acc   (exact rescale)
    const double two64 = 18446744073709551616.0;  // 2 * 2^63
    const int64_t pA = (int64_t)cb * pga::CB + 2 * lane;
    double *vA = V + pA * ldn + i0;
    double *vB = vA + ldn;
#pragma unroll
    for (int r = 0; r < pga::TI; r += 2) {
        double d0 = 0.0, d1 = 0.0;
        if (i0 + r < N) d0 = __ldg(diag + i0 + r);
        if (i0 + r + 1 < N) d1 = __ldg(diag + i0 + r + 1);
        reinterpret_cast<double2 *>(vA)[r >> 1] = make_double2(fma(two64, accA[r], d0), fma(two64, accA[r + 1], d1));
        reinterpret_cast<double2 *>(vB)[r >> 1] = make_double2(fma(two64, accB[r], d0), fma(two64, accB[r + 1], d1));
    }
}

// ---------------------------------------------------------------------------
// k_fold: one warp per chromosome.  smem per warp: cs[N] fp64, ns[N] int32.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128)
k_fold(const uint16_t *__restrict__ CM0, const uint16_t *__restrict__ CM1,
       const int32_t *__restrict__ gen_ptr, int ldn, const double *__restrict__ V, int N, int64_t P,
       double *__restrict__ Lout, uint16_t *__restrict__ topout,
       const int32_t *__restrict__ done_flag) {
    if (done_flag && *done_flag) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nw = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint16_t *CM = (gen_ptr && (*gen_ptr & 1)) ? CM1 : CM0;
    double *cs = reinterpret_cast<double *>(smem_raw) + (size_t)warp * N;
    int32_t *ns = reinterpret_cast<int32_t *>(reinterpret_cast<double *>(smem_raw) + (size_t)nw * N) +
                  (size_t)warp * N;
    const int64_t p = (int64_t)blockIdx.x * nw + warp;
    if (p >= P) return;
    for (int k = lane; k < N; k += 32) {
        cs[k] = 0.0;
        ns[k] = 0;
    }
    __syncwarp();
    const uint16_t *lab = CM + p * ldn;
    const double *v = V + p * ldn;
    for (int base = 0; base < N; base += 32) {
        const int i = base + lane;
        const bool valid = i < N;
        const uint32_t s = valid ? (uint32_t)lab[i] : (0x10000u + (uint32_t)lane);
        double sum = valid ? v[i] : 0.0;
        const unsigned m = __match_any_sync(0xFFFFFFFFu, s);
        // next member of my group after me (32 = none)
        const unsigned after = (lane == 31) ? 0u : (m & ~((2u << lane) - 1u));
        int nxt = after ? (__ffs(after) - 1) : 32;
#pragma unroll
        for (int step = 0; step < 5; ++step) {
            const double o = __shfl_sync(0xFFFFFFFFu, sum, nxt & 31);
            const int on = __shfl_sync(0xFFFFFFFFu, nxt, nxt & 31);
            if (nxt < 32) {
                sum += o;
                nxt = on;
            }
        }
        const int leader = __ffs(m) - 1;
        if (valid && lane == leader) {
            cs[s] += sum;
            ns[s] += __popc(m);
        }
        __syncwarp();
    }
    // Eq. 8 over clusters k = lane, lane+32, ...
    double fsum = 0.0, fbest = 0.0;
    int kbest = 0x7FFFFFFF;
    for (int k = lane; k < N; k += 32) {
        const int n = ns[k];
        if (n >= 2) {
            const double f = cluster_term(n, cs[k]);
            fsum += f;
            if (f > fbest) {
                fbest = f;
                kbest = k;
            }
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
        Lout[p] = 0.5 * fsum;
        if (topout) topout[p] = (fbest > 0.0) ? (uint16_t)kbest : (uint16_t)0xFFFF;
    }
}

}  // namespace

namespace pga {

int launch_pack(pga_ctx *c, const uint16_t *lab16, const int32_t *lab32, int64_t P, int ld_in,
                uint16_t *CM, uint16_t *GM, cudaStream_t s) {
    dim3 grid((unsigned)((P + 31) / 32), (unsigned)((c->N + 31) / 32));
    k_pack<<<grid, dim3(32, 8), 0, s>>>(lab16, lab32, P, ld_in, c->N, c->ldn, c->Pcap, CM, GM, c->st);
    PGA_LAUNCHED();
    return PGA_OK;
}

int fold_warps(int N) {
    const size_t per = (size_t)N * (sizeof(double) + sizeof(int32_t));
    int w = (int)((200 * 1024) / per);
    return w < 1 ? 1 : (w > 4 ? 4 : w);
}

size_t fold_smem(int N) { return (size_t)fold_warps(N) * N * (sizeof(double) + sizeof(int32_t)); }

int prepare_fitness(int N) {
    PGA_CUDA(cudaFuncSetAttribute(k_fold, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)fold_smem(N)));
    return PGA_OK;
}

int launch_fitness(pga_ctx *c, const FitBufs &b, int64_t P, double *L, uint16_t *top,
                   cudaStream_t s, cudaEvent_t *ev) {
    const int N = c->N;
    const int nRB = (N + TI - 1) / TI;
    const int nCB = (int)((P + CB - 1) / CB);
    const int nQ = (nCB + SWEEP_WARPS - 1) / SWEEP_WARPS;
    if (ev) PGA_CUDA(cudaEventRecord(ev[0], s));
    k_sweep<<<(unsigned)(nRB * nQ), SWEEP_WARPS * 32, 0, s>>>(
        c->C, c->ldc, c->diag, reinterpret_cast<const uint32_t *>(b.gm0),
        reinterpret_cast<const uint32_t *>(b.gm1), b.gen, N, c->Pcap, nCB, nQ, c->V, c->ldn, b.done);
    PGA_LAUNCHED();
    if (ev) PGA_CUDA(cudaEventRecord(ev[1], s));
    const int fw = fold_warps(N);
    k_fold<<<(unsigned)((P + fw - 1) / fw), fw * 32, fold_smem(N), s>>>(
        b.cm0, b.cm1, b.gen, c->ldn, c->V, N, P, L, top, b.done);
    PGA_LAUNCHED();
    if (ev) PGA_CUDA(cudaEventRecord(ev[2], s));
    return PGA_OK;
}

}  // namespace pga
