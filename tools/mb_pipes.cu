// Pipe-throughput microbenchmark (measurement tool): ops per SM per clock
// for DFMA, DADD, HSET2, IMAD, LOP3, FFMA, IADD3, ISETP+SEL, measured with
// clock64 inside the kernel (so independent of the SM clock value).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 8;  // independent chains per thread
constexpr int IT = 2048;

template <int OP>
__global__ void __launch_bounds__(256) k(double *outd, uint32_t *outu, float *outf, long long *clk, uint32_t seed) {
    double d[CH];
    uint32_t u[CH];
    float f[CH];
    for (int c = 0; c < CH; ++c) {
        d[c] = 1.0 + 1e-9 * (threadIdx.x + c);
        u[c] = seed * (threadIdx.x + 7 * c + 1);
        f[c] = 1.0f + 1e-6f * (threadIdx.x + c);
    }
    const double dm = 0.999999999, da = 1e-12;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < IT; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (OP == 0) d[c] = fma(d[c], dm, da);
            if (OP == 1) d[c] = d[c] + da;
            if (OP == 2) asm volatile("set.eq.f16x2.f16x2 %0, %0, %1;" : "+r"(u[c]) : "r"(seed));
            if (OP == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(u[c]) : "r"(seed), "r"(c));
            if (OP == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[c]) : "r"(seed), "r"(c));
            if (OP == 5) f[c] = fmaf(f[c], 0.9999f, 1e-7f);
            if (OP == 6) asm volatile("add.u32 %0, %0, %1;" : "+r"(u[c]) : "r"(seed));
            if (OP == 7) asm volatile("{.reg .pred p; setp.eq.u32 p, %0, %1; selp.b32 %0, %1, %2, p;}" : "+r"(u[c]) : "r"(seed), "r"(c));
            if (OP == 8) { unsigned long long m; asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(m) : "r"(u[c]), "r"(seed)); u[c] = (uint32_t)(m >> 32) ^ u[c]; }
        }
    }
    long long t1 = clock64();
    double sd = 0; uint32_t su = 0; float sf = 0;
    for (int c = 0; c < CH; ++c) { sd += d[c]; su ^= u[c]; sf += f[c]; }
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    outd[g] = sd; outu[g] = su; outf[g] = sf;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char *name, int blocks_per_sm, double *od, uint32_t *ou, float *of, long long *dclk) {
    const int sms = 148, grid = sms * blocks_per_sm, bs = 256;
    k<OP><<<grid, bs>>>(od, ou, of, dclk, 3);
    cudaDeviceSynchronize();
    long long h[148 * 8];
    cudaMemcpy(h, dclk, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    // all blocks of an SM run concurrently (grid == resident capacity)
    double ops_per_sm = (double)blocks_per_sm * bs * CH * IT;
    printf("%-10s warps/SM=%2d  %.1f ops/clk/SM\n", name, blocks_per_sm * bs / 32, ops_per_sm / mx);
}

int main() {
    double *od; uint32_t *ou; float *of; long long *dclk;
    cudaMalloc(&od, sizeof(double) * 148 * 8 * 256);
    cudaMalloc(&ou, sizeof(uint32_t) * 148 * 8 * 256);
    cudaMalloc(&of, sizeof(float) * 148 * 8 * 256);
    cudaMalloc(&dclk, sizeof(long long) * 148 * 8);
    for (int b : {1, 2, 4}) {
        run<0>("DFMA", b, od, ou, of, dclk);
        run<1>("DADD", b, od, ou, of, dclk);
        run<2>("HSET2", b, od, ou, of, dclk);
        run<3>("IMAD", b, od, ou, of, dclk);
        run<4>("LOP3", b, od, ou, of, dclk);
        run<5>("FFMA", b, od, ou, of, dclk);
        run<6>("IADD", b, od, ou, of, dclk);
        run<7>("ISETP+SEL", b, od, ou, of, dclk);
        run<8>("IMADWIDE+", b, od, ou, of, dclk);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
