// stream.cu — on-device correlation stream, feeding
// the batched GA (batch.cu).  The paper's pre-processing (§4.2.5):
// "a covariance matrix was then computed using an iterative online
// exponentially-weighted moving average (EWMA) filter with a default
// forgetting factor of lambda = 0.98.  The correlation matrix was computed
// from the covariance matrix and was cleaned using random matrix theory
// methods ... eliminating eigenvalues in the Wishart range in a
// trace-preserving manner."  Operation order and readings: DESIGN.md Q31-Q33
// (SPEC S:279-301).
//
//   k_ewma        observations staged in shared memory 64 at a time; threads
//                 0..N-1: d_t = x_t - m_{t-1}, m_t = lam m + (1-lam) x_t; thread per
//                 upper entry (i <= j): cov = lam cov + (1-lam) d_i d_j, snapshot
//                 after observation t = warm-1 + b*stride
//   k_clean       CTA per snapshot: correlation, two-sided Jacobi eigensolver
//                 (parallel round-robin ordering, shared memory), in-band
//                 eigenvalues -> their mean, reconstruction, unit diagonal
//
// The recurrences use explicitly rounded multiplies and adds (no FMA
// contraction) in the SPEC's operation order, so the EWMA state and the
// uncleaned correlation are bit-identical to a plain fp64 evaluation.
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "pga_internal.cuh"

namespace {

constexpr int SMAX_N = 64;   // k_clean keeps A and V (N x (N+1) fp64 each) in shared memory
constexpr int JT = 256;

// EWMA mean and covariance in one pass over the stream.  Observations are
// staged TC at a time in shared memory; threads 0..N-1 advance the means
// (every CTA redundantly, identically), then each thread advances its
// covariance entries (i <= j) through the chunk and snapshots them after
// observation t = warm-1 + b*stride.
constexpr int TC = 64, ET = 256;

__global__ void __launch_bounds__(ET) k_ewma(const double *__restrict__ X, int T, int N, double lam, int warm,
                                             int stride, int B, double *__restrict__ R) {
    extern __shared__ double sx[];            // [TC][N] observations, then [TC][N] deviations
    double *sd = sx + TC * N;
    __shared__ double s_m[SMAX_N];
    const int tid = threadIdx.x;
    const int E = N * (N + 1) / 2;
    const int e = blockIdx.x * ET + tid;
    int i = 0, j = 0;
    if (e < E) {                              // e -> (i, j), i <= j, row-major upper triangle
        int rem = e;
        while (rem >= N - i) {
            rem -= N - i;
            ++i;
        }
        j = i + rem;
    }
    const double oml = 1.0 - lam;
    if (tid < N) s_m[tid] = 0.0;
    double cov = 0.0;
    int b = 0, next = warm - 1;
    for (int t0 = 0; t0 < T && b < B; t0 += TC) {
        const int tc = min(TC, T - t0);
        __syncthreads();
        for (int k = tid; k < tc * N; k += ET) sx[k] = X[(size_t)t0 * N + k];
        __syncthreads();
        if (tid < N) {                        // d = x - m_prev; m <- lam m + (1 - lam) x
            double m = s_m[tid];
            for (int t = 0; t < tc; ++t) {
                const double x = sx[t * N + tid];
                sd[t * N + tid] = __dsub_rn(x, m);
                m = __dadd_rn(__dmul_rn(lam, m), __dmul_rn(oml, x));
            }
            s_m[tid] = m;
        }
        __syncthreads();
        if (e < E) {                          // cov <- lam cov + (1 - lam) d_i d_j
            for (int t = 0; t < tc; ++t) {
                cov = __dadd_rn(__dmul_rn(lam, cov), __dmul_rn(oml, __dmul_rn(sd[t * N + i], sd[t * N + j])));
                if (t0 + t == next) {
                    R[((size_t)b * N + i) * N + j] = cov;
                    ++b;
                    next += stride;
                }
            }
        } else {
            for (int t = 0; t < tc; ++t)      // keep b in step (uniform loop exit)
                if (t0 + t == next) {
                    ++b;
                    next += stride;
                }
        }
    }
}

__device__ __forceinline__ double block_sum(double v, double *red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int k = 0; k < JT / 32; ++k) s += red[k];   // same order in every thread
    return s;
}

// pair k of round r of the circle schedule on n2 (even) indices
__device__ __forceinline__ void rr_pair(int r, int k, int n2, int &p, int &q) {
    if (k == 0) {
        p = r;
        q = n2 - 1;
    } else {
        p = (r + k) % (n2 - 1);
        q = (r - k + n2 - 1) % (n2 - 1);
    }
    if (p > q) {
        const int t = p;
        p = q;
        q = t;
    }
}

__global__ void __launch_bounds__(JT) k_clean(const double *__restrict__ R, int N, double q, int clean,
                                              double *__restrict__ Cout, int32_t *status) {
    extern __shared__ double sm[];
    __shared__ double red[JT / 32];
    __shared__ double s_c[SMAX_N / 2], s_s[SMAX_N / 2];
    __shared__ int s_p[SMAX_N / 2], s_q[SMAX_N / 2];
    __shared__ double s_w[SMAX_N];
    const int ld = N + 1;
    double *A = sm, *V = sm + (size_t)N * ld;
    const int b = blockIdx.x, tid = threadIdx.x;
    const double *Rb = R + (size_t)b * N * N;
    double *Cb = Cout + (size_t)b * N * N;

    // correlation from covariance: C_ij = cov_ij / sqrt(cov_ii cov_jj), unit diagonal
    for (int e = tid; e < N * N; e += JT) {
        const int i = e / N, j = e - (e / N) * N;
        const int a = min(i, j), c = max(i, j);
        const double vi = Rb[(size_t)a * N + a], vj = Rb[(size_t)c * N + c];
        if (i == j) {
            if (!(vi > 0.0)) atomicExch(status, 1);
            A[i * ld + j] = 1.0;
        } else {
            A[i * ld + j] = Rb[(size_t)a * N + c] / sqrt(vi * vj);
        }
        V[i * ld + j] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (!clean) {
        for (int e = tid; e < N * N; e += JT) Cb[e] = A[(e / N) * ld + (e - (e / N) * N)];
        return;
    }

    // two-sided Jacobi: A <- J^T A J, V <- V J, parallel round-robin pairs
    const int n2 = N + (N & 1), np = n2 / 2;
    for (int sweep = 0; sweep < 40; ++sweep) {
        double off = 0.0, dn = 0.0;
        for (int e = tid; e < N * N; e += JT) {
            const int i = e / N, j = e - (e / N) * N;
            const double x = A[i * ld + j];
            if (i == j) dn += x * x;
            else off += x * x;
        }
        off = block_sum(off, red);
        dn = block_sum(dn, red);
        if (!(off > 1e-30 * dn)) break;   // uniform across the CTA
        for (int r = 0; r < n2 - 1; ++r) {
            if (tid < np) {
                int p, qq;
                rr_pair(r, tid, n2, p, qq);
                double c = 1.0, s = 0.0;
                if (qq < N) {
                    const double apq = A[p * ld + qq];
                    if (apq != 0.0) {
                        const double tau = (A[qq * ld + qq] - A[p * ld + p]) / (2.0 * apq);
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + t * t);
                        s = t * c;
                    }
                }
                s_p[tid] = p;
                s_q[tid] = qq < N ? qq : -1;
                s_c[tid] = c;
                s_s[tid] = s;
            }
            __syncthreads();
            for (int e = tid; e < np * N; e += JT) {       // rows p, q of J^T A
                const int k = e / N, j = e - (e / N) * N;
                const int p = s_p[k], qq = s_q[k];
                if (qq < 0) continue;
                const double c = s_c[k], s = s_s[k];
                const double apj = A[p * ld + j], aqj = A[qq * ld + j];
                A[p * ld + j] = c * apj - s * aqj;
                A[qq * ld + j] = s * apj + c * aqj;
            }
            __syncthreads();
            for (int e = tid; e < np * N; e += JT) {       // columns p, q of (J^T A) J and V J
                const int k = e / N, i = e - (e / N) * N;
                const int p = s_p[k], qq = s_q[k];
                if (qq < 0) continue;
                const double c = s_c[k], s = s_s[k];
                const double aip = A[i * ld + p], aiq = A[i * ld + qq];
                A[i * ld + p] = c * aip - s * aiq;
                A[i * ld + qq] = s * aip + c * aiq;
                const double vip = V[i * ld + p], viq = V[i * ld + qq];
                V[i * ld + p] = c * vip - s * viq;
                V[i * ld + qq] = s * vip + c * viq;
            }
            __syncthreads();
        }
    }
    // Marchenko-Pastur band [(1 - sqrt q)^2, (1 + sqrt q)^2]: in-band
    // eigenvalues -> their mean (trace preserving)
    if (tid == 0) {
        const double rq = sqrt(q), lo = (1.0 - rq) * (1.0 - rq), hi = (1.0 + rq) * (1.0 + rq);
        double sum = 0.0;
        int cnt = 0;
        for (int k = 0; k < N; ++k) {
            const double w = A[k * ld + k];
            if (w >= lo && w <= hi) {
                sum += w;
                ++cnt;
            }
        }
        const double mean = cnt ? sum / cnt : 0.0;
        for (int k = 0; k < N; ++k) {
            const double w = A[k * ld + k];
            s_w[k] = (w >= lo && w <= hi) ? mean : w;
        }
    }
    __syncthreads();
    // C' = V diag(w') V^T (upper triangle and diagonal, into A)
    for (int e = tid; e < N * N; e += JT) {
        const int i = e / N, j = e - (e / N) * N;
        if (j < i) continue;
        double acc = 0.0;
        for (int k = 0; k < N; ++k) acc += V[i * ld + k] * s_w[k] * V[j * ld + k];
        A[i * ld + j] = acc;
    }
    __syncthreads();
    // unit diagonal: C''_ij = C'_ij / sqrt(C'_ii C'_jj) from the upper triangle, mirrored
    for (int e = tid; e < N * N; e += JT) {
        const int i = e / N, j = e - (e / N) * N;
        const int a = min(i, j), c = max(i, j);
        Cb[e] = (i == j) ? 1.0 : A[a * ld + c] / sqrt(A[a * ld + a] * A[c * ld + c]);
    }
}

int stream_count(int T, int warm, int stride) { return T < warm ? 0 : (T - warm) / stride + 1; }

#define STRY(x)              \
    do {                     \
        int _rc = (x);       \
        if (_rc) return _rc; \
    } while (0)

int launch_stream(const double *X, int T, int N, double lam, int warm, int stride, double q, int clean,
                  double *C, int32_t *status, double *R, cudaStream_t s) {
    const int B = stream_count(T, warm, stride);
    const int E = N * (N + 1) / 2;
    const size_t esm = (size_t)2 * TC * N * sizeof(double);
    PGA_CUDA(cudaFuncSetAttribute(k_ewma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esm));
    k_ewma<<<(E + ET - 1) / ET, ET, esm, s>>>(X, T, N, lam, warm, stride, B, R);
    PGA_LAUNCHED();
    const size_t smem = (size_t)2 * N * (N + 1) * sizeof(double);
    PGA_CUDA(cudaFuncSetAttribute(k_clean, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_clean<<<B, JT, smem, s>>>(R, N, q, clean, C, status);
    PGA_LAUNCHED();
    return PGA_OK;
}

}  // namespace

extern "C" {

int pga_stream_count(int32_t T, int32_t warm, int32_t stride) {
    if (T < 0 || warm < 1 || stride < 1) return pga::fail(PGA_EINVAL, "need T >= 0, warm >= 1, stride >= 1");
    return stream_count(T, warm, stride);
}

int pga_corr_stream(const double *X, int32_t T, int32_t N, double lambda, int32_t warm, int32_t stride,
                    double q, int32_t on_device, double *C_out, int32_t *status, int32_t device, void *stream) {
    if (!X || !C_out) return pga::fail(PGA_EINVAL, "NULL argument");
    if (N < 1 || N > SMAX_N) return pga::fail(PGA_EINVAL, "correlation stream needs 1 <= N <= 64");
    if (!(lambda > 0.0 && lambda < 1.0)) return pga::fail(PGA_EINVAL, "lambda must lie in (0, 1)");
    if (warm < 1 || stride < 1 || T < warm) return pga::fail(PGA_EINVAL, "need warm >= 1, stride >= 1, T >= warm");
    if (!std::isfinite(q)) return pga::fail(PGA_EINVAL, "q must be finite");
    if (on_device && !status) return pga::fail(PGA_EINVAL, "device path needs a status flag");
    const int clean = q >= 0.0;
    const double qq = q == 0.0 ? (double)N * (1.0 - lambda) : q;
    const int B = stream_count(T, warm, stride);
    if (!on_device)
        for (size_t k = 0; k < (size_t)T * N; ++k)
            if (!std::isfinite(X[k])) return pga::fail(PGA_EINVAL, "X has a non-finite entry");
    STRY(pga::ensure_device(device));
    if (on_device) {
        // stream-ordered scratch: no device-wide synchronisation
        cudaStream_t st = (cudaStream_t)stream;
        double *R = nullptr;
        PGA_CUDA(pga::pool_malloc_async((void **)&R, sizeof(double) * ((size_t)B * N * N + 1), st));
        int rc = launch_stream(X, T, N, lambda, warm, stride, qq, clean, C_out, status, R, st);
        cudaFreeAsync(R, st);
        return rc;
    }
    // host path: one stream, stream-ordered scratch
    cudaStream_t st;
    PGA_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    } guard{st};
    const size_t nX = (size_t)T * N, nR = (size_t)B * N * N;
    unsigned char *blob = nullptr;
    PGA_CUDA(pga::pool_malloc_async((void **)&blob, sizeof(double) * (nX + 2 * nR) + 64, st));
    struct BlobGuard {
        void *p;
        cudaStream_t s;
        ~BlobGuard() { cudaFreeAsync(p, s); }
    } bg{blob, st};
    double *dX = reinterpret_cast<double *>(blob), *R = dX + nX, *dC = R + nR;
    int32_t *dst = reinterpret_cast<int32_t *>(dC + nR);
    PGA_CUDA(cudaMemsetAsync(dst, 0, sizeof(int32_t), st));
    PGA_CUDA(cudaMemcpyAsync(dX, X, sizeof(double) * nX, cudaMemcpyHostToDevice, st));
    STRY(launch_stream(dX, T, N, lambda, warm, stride, qq, clean, dC, dst, R, st));
    int32_t h = 0;
    PGA_CUDA(cudaMemcpyAsync(&h, dst, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    PGA_CUDA(cudaStreamSynchronize(st));
    if (status) *status = h;
    if (h) return pga::fail(PGA_ENUMERIC, "non-positive EWMA variance at an emission");
    PGA_CUDA(cudaMemcpyAsync(C_out, dC, sizeof(double) * nR, cudaMemcpyDeviceToHost, st));
    PGA_CUDA(cudaStreamSynchronize(st));
    return PGA_OK;
}

}  // extern "C"
