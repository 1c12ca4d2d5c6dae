// Does redux.sync with per-group membermasks (from match.any) run in one pass?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(const uint32_t* lab, const uint32_t* val, uint32_t* out, long long* clk, int reps, int mode) {
  const int lane = threadIdx.x & 31;
  uint32_t s = lab[threadIdx.x], v = val[threadIdx.x], acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    unsigned m = (mode == 0) ? 0xFFFFFFFFu : __match_any_sync(0xFFFFFFFFu, s);
    acc += __reduce_add_sync(m, v + r);
    s ^= (acc & 1) << 20;  // keep a dependency, labels stay grouped per bit 20
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  const int n = 32 * 8;
  uint32_t hl[n], hv[n];
  for (int i = 0; i < n; ++i) { hl[i] = (i * 2654435761u >> 9) % 20; hv[i] = i * 7 + 1; }
  uint32_t *dl, *dv, *dout; long long* dclk;
  cudaMalloc(&dl, sizeof(hl)); cudaMalloc(&dv, sizeof(hv)); cudaMalloc(&dout, 4 * n * 148); cudaMalloc(&dclk, 8 * 148);
  cudaMemcpy(dl, hl, sizeof(hl), cudaMemcpyHostToDevice); cudaMemcpy(dv, hv, sizeof(hv), cudaMemcpyHostToDevice);
  // correctness (1 rep, mode 1)
  k<<<1, 32>>>(dl, dv, dout, dclk, 1, 1);
  uint32_t ho[32]; cudaMemcpy(ho, dout, 128, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 32; ++i) { uint32_t e = 0; for (int j = 0; j < 32; ++j) if (hl[j] == hl[i]) e += hv[j]; if (e != ho[i]) bad++; }
  printf("partitioned redux correct lanes: %d/32\n", 32 - bad);
  for (int mode = 0; mode < 2; ++mode) {
    k<<<1, 32>>>(dl, dv, dout, dclk, 1000, mode);
    long long c; cudaMemcpy(&c, dclk, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %.1f cycles per iteration (1 warp)\n", mode, mode ? "match+partitioned redux" : "full-mask redux", c / 1000.0);
  }
  return 0;
}
