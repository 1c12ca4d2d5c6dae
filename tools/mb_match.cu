// MATCH.ANY throughput per SM (measurement tool): independent match_any
// streams in many warps; keys with few / many distinct values.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(uint32_t seed, int reps, int distinct, uint32_t *out, long long *clk) {
  const int lane = threadIdx.x & 31;
  uint32_t x = seed * (threadIdx.x + 1) + blockIdx.x, acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint32_t k0 = ((x + r * 2654435761u) >> 7) % distinct;
    uint32_t k1 = ((x + r * 40503u) >> 5) % distinct;
    acc += __match_any_sync(0xFFFFFFFFu, k0) ^ __match_any_sync(0xFFFFFFFFu, k1 + 7);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  uint32_t *out; long long *clk;
  cudaMalloc(&out, 4 * 148 * 1024); cudaMalloc(&clk, 8 * 148);
  for (int distinct : {2, 8, 32, 1000}) for (int bs : {128, 1024}) {
    int reps = 2000;
    k<<<148, bs>>>(3, 10, distinct, out, clk);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, bs>>>(3, reps, distinct, out, clk);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h; cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    double matches_per_sm = 2.0 * reps * (bs / 32);
    printf("distinct=%4d warps/SM=%2d: %.1f SM-cycles per warp-MATCH (clock64), %.3f ms\n", distinct, bs / 32,
           h / matches_per_sm, ms);
  }
  return 0;
}
