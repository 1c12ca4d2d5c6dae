// corr.cu — Eq. 7: Pearson correlation of T observations of N
// assets, with per-column centring (reading Q5).
//   k_colstats : two-pass column mean and centred l2 norm (fp64)
//   k_normalize: Z[t][i] = (X[t][i] - mean_i) / norm_i
//   k_gram     : C = Z^T Z on the fp64 tensor path (mma.sync m8n8k4 f64 ->
//                SASS DMMA; tcgen05 has no f64 kind), upper-triangle tiles
//                only, mirrored on store so C is exactly symmetric, C_ii := 1.
#include <cuda_runtime.h>

#include "pga_internal.cuh"

namespace {

__global__ void k_colstats(const double *__restrict__ X, int T, int N, double *mean, double *inv_norm,
                           int32_t *status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    double s = 0.0;
    bool finite = true;
    for (int t = 0; t < T; ++t) {
        const double v = X[(int64_t)t * N + i];
        finite &= isfinite(v);
        s += v;
    }
    const double m = s / (double)T;
    double ss = 0.0;
    for (int t = 0; t < T; ++t) {
        const double d = X[(int64_t)t * N + i] - m;
        ss += d * d;
    }
    const double nrm = sqrt(ss);
    if (!finite || !(nrm > 0.0)) {
        atomicExch(status, 1);
        inv_norm[i] = 0.0;
    } else {
        inv_norm[i] = 1.0 / nrm;
    }
    mean[i] = m;
}

// Z is [Tpad][Npad] (zero padded)
__global__ void k_normalize(const double *__restrict__ X, int T, int N, const double *mean,
                            const double *inv_norm, double *Z, int Npad) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t t = idx / Npad;
    const int i = (int)(idx - t * Npad);
    if (t >= T) return;
    Z[idx] = (i < N) ? (X[t * N + i] - mean[i]) * inv_norm[i] : 0.0;
}

// 64x64 output tile per block (4 warps, each 32x32 = 4x4 DMMA 8x8 tiles),
// K staged 32 at a time through shared memory.
constexpr int GT = 64, GK = 32;

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) k_gram(const double *__restrict__ Z, int Tpad, int Npad, int N,
                                              double *C, int ldc) {
    const int bi = blockIdx.y, bj = blockIdx.x;
    if (bj < bi) return;  // upper-triangle tiles only
    __shared__ double As[GK][GT + 1];  // As[k][i] = Z[t0+k][i0+i]
    __shared__ double Bs[GK][GT + 1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wi = (warp >> 1) * 32, wj = (warp & 1) * 32;
    const int i0 = bi * GT, j0 = bj * GT;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int t0 = 0; t0 < Tpad; t0 += GK) {
        for (int e = tid; e < GK * GT; e += 128) {
            const int k = e / GT, c = e - k * GT;
            As[k][c] = Z[(int64_t)(t0 + k) * Npad + i0 + c];
            Bs[k][c] = Z[(int64_t)(t0 + k) * Npad + j0 + c];
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GK; kk += 4) {
            // A fragment (8x4 row-major): row = lane>>2, col = lane&3
            // B fragment (4x8 col-major): row = lane&3, col = lane>>2
            double af[4], bf[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) af[a] = As[kk + (lane & 3)][wi + a * 8 + (lane >> 2)];
#pragma unroll
            for (int b = 0; b < 4; ++b) bf[b] = Bs[kk + (lane & 3)][wj + b * 8 + (lane >> 2)];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
        __syncthreads();
    }
    // C fragment: row = lane>>2, cols 2*(lane&3) + {0,1}
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = i0 + wi + a * 8 + (lane >> 2);
                const int j = j0 + wj + b * 8 + 2 * (lane & 3) + h;
                if (i < N && j < N && j >= i) {
                    const double v = (i == j) ? 1.0 : acc[a][b][h];
                    C[(int64_t)i * ldc + j] = v;
                    C[(int64_t)j * ldc + i] = v;
                }
            }
}

}  // namespace

namespace pga {

int launch_corr(const double *X, int32_t T, int32_t N, double *C, int32_t *status, cudaStream_t s) {
    const int Npad = (N + GT - 1) / GT * GT;
    const int Tpad = (T + GK - 1) / GK * GK;
    double *mean = nullptr, *inv = nullptr, *Z = nullptr;
    PGA_CUDA(pga::pool_malloc_async((void **)&mean, sizeof(double) * N, s));
    PGA_CUDA(pga::pool_malloc_async((void **)&inv, sizeof(double) * N, s));
    PGA_CUDA(pga::pool_malloc_async((void **)&Z, sizeof(double) * (size_t)Npad * Tpad, s));
    k_colstats<<<(N + 127) / 128, 128, 0, s>>>(X, T, N, mean, inv, status);
    PGA_LAUNCHED();
    PGA_CUDA(cudaMemsetAsync(Z, 0, sizeof(double) * (size_t)Npad * Tpad, s));
    const int64_t tot = (int64_t)T * Npad;
    k_normalize<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(X, T, N, mean, inv, Z, Npad);
    PGA_LAUNCHED();
    dim3 grid(Npad / GT, Npad / GT);
    k_gram<<<grid, 128, 0, s>>>(Z, Tpad, Npad, N, C, N);
    PGA_LAUNCHED();
    PGA_CUDA(cudaFreeAsync(mean, s));
    PGA_CUDA(cudaFreeAsync(inv, s));
    PGA_CUDA(cudaFreeAsync(Z, s));
    return PGA_OK;
}

}  // namespace pga
