// Microbenchmark (measurement tool, not product): random 8-byte gathers from
// an L2-resident fp64 array the size of C at N = 500 (2 MB), as the
// label-sparse pass issues them.  Reports gathers/s and 32-byte sectors/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k(const double *__restrict__ c, int n, int iters, double *out) {
    uint32_t x = 2654435761u * (blockIdx.x * blockDim.x + threadIdx.x) + 12345u;
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        uint32_t idx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x = x * 1664525u + 1013904223u;
            idx[u] = x % n;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += __ldg(c + idx[u]);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    const int n = 500 * 504;                 // C at N = 500, ldc = 504
    double *c, *out;
    cudaMalloc(&c, sizeof(double) * n);
    cudaMemset(c, 0, sizeof(double) * n);
    const int threads = 256, blocks = 148 * 8, iters = 2000;
    cudaMalloc(&out, sizeof(double) * threads * blocks);
    k<<<blocks, threads>>>(c, n, 10, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(c, n, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double g = (double)blocks * threads * iters * 8;
    printf("random 8-byte gathers from a 2 MB array: %.3e gathers/s = %.1f GB/s of 32-byte sectors "
           "(%.0f B/clk at 1965 MHz)\n", g / (ms * 1e-3), g * 32 / (ms * 1e-3) / 1e9,
           g * 32 / (ms * 1e-3) / 1.965e9);
    return 0;
}
