// Microbenchmark of the fitness inner loop (measurement tool, not product).
// Each warp: 64 chromosomes (2/lane) x 8 rows; columns streamed from shared
// memory; variants of the masked fp64 accumulate.  Reports executed
// pair-updates per SM-clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int KC = 64;

__device__ __forceinline__ uint32_t heq(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("set.eq.f16x2.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

template <int V>
__device__ __forceinline__ double acc1(double acc, double c, uint32_t col, uint32_t row) {
    if (V == 0) {  // MOV: {0, h}
        return fma(c, __hiloint2double((int)heq(col, row), 0), acc);
    } else if (V == 1) {  // WIDE
        unsigned long long m;
        asm("mul.wide.u32 %0, %1, 0x80000000;" : "=l"(m) : "r"(heq(col, row)));
        return fma(c, __longlong_as_double((long long)m), acc);
    } else if (V == 2) {  // hi-word select of C (denormal residue on mismatch)
        uint32_t h = heq(col, row);
        int hi = __double2hiint(c), lo = __double2loint(c);
        return acc + __hiloint2double(h ? hi : 0, lo);
    } else {  // predicated add (ptxas if-converts)
        return (heq(col, row) != 0) ? acc + c : acc;
    }
}

template <int V>
__global__ void __launch_bounds__(128) k(const uint32_t *labs_g, const double *c_g, int reps, double *out,
                                         long long *clk) {
    __shared__ uint32_t labs[KC][32];
    __shared__ double cs[KC][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < KC * 32; i += blockDim.x) {
        (&labs[0][0])[i] = labs_g[i];
        (&cs[0][0])[i] = c_g[i];
    }
    __syncthreads();
    uint32_t rowA[8], rowB[8];
    double a[8], b[8];
    for (int r = 0; r < 8; ++r) {
        uint32_t w = labs[r][lane];
        rowA[r] = (w << 16) | 0x7FFF;
        rowB[r] = (w & 0xFFFF0000u) | 0x7FFF;
        a[r] = b[r] = 0;
    }
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 4
        for (int t = 0; t < KC; ++t) {
            const uint32_t w = labs[t][lane];
            const uint32_t wa = w << 16;
            const double2 *c2 = reinterpret_cast<const double2 *>(&cs[t][8 * warp]);
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) {
                const double2 c = c2[k2];
                a[2 * k2] = acc1<V>(a[2 * k2], c.x, wa, rowA[2 * k2]);
                b[2 * k2] = acc1<V>(b[2 * k2], c.x, w, rowB[2 * k2]);
                a[2 * k2 + 1] = acc1<V>(a[2 * k2 + 1], c.y, wa, rowA[2 * k2 + 1]);
                b[2 * k2 + 1] = acc1<V>(b[2 * k2 + 1], c.y, w, rowB[2 * k2 + 1]);
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int r = 0; r < 8; ++r) s += a[r] + b[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// V4: one chromosome per lane, 16 rows, HSETP2 dual predicate + in-place
// hi-word SEL + DADD (non-match adds the positive denormal {C_lo, 0}).
__global__ void __launch_bounds__(128) k4(const uint32_t *labs_g, const double *c_g, int reps, double *out,
                                          long long *clk) {
    __shared__ uint32_t labs[KC][32];
    __shared__ double cs[KC][64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < KC * 32; i += blockDim.x) (&labs[0][0])[i] = labs_g[i];
    for (int i = threadIdx.x; i < KC * 64; i += blockDim.x) (&cs[0][0])[i] = c_g[i % (KC * 32)];
    __syncthreads();
    uint32_t rowpk[8];
    double a[16];
    for (int r = 0; r < 8; ++r) {
        uint32_t w0 = labs[2 * r][lane] & 0xFFFF, w1 = labs[2 * r + 1][lane] & 0xFFFF;
        rowpk[r] = (w1 << 16) | w0;
    }
    for (int r = 0; r < 16; ++r) a[r] = 0;
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 2
        for (int t = 0; t < KC; ++t) {
            const uint32_t w = labs[t][lane] & 0xFFFF;
            const uint32_t col = (w << 16) | w;
            const double2 *c2 = reinterpret_cast<const double2 *>(&cs[t][16 * (warp & 3)]);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                double2 c = c2[r];
                int lo0 = __double2loint(c.x), hi0 = __double2hiint(c.x);
                int lo1 = __double2loint(c.y), hi1 = __double2hiint(c.y);
                int s0, s1;
                asm("{.reg .pred p, q;\n\tsetp.eq.f16x2 p|q, %2, %3;\n\tselp.b32 %0, %4, 0, p;\n\tselp.b32 %1, %5, 0, q;}"
                    : "=r"(s0), "=r"(s1) : "r"(rowpk[r]), "r"(col), "r"(hi0), "r"(hi1));
                a[2 * r] += __hiloint2double(s0, lo0);
                a[2 * r + 1] += __hiloint2double(s1, lo1);
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int r = 0; r < 16; ++r) s += a[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// V5: as V4, the whole 2-pair step in one PTX block so the select can be
// done in place on the loaded hi words.
__global__ void __launch_bounds__(128) k5(const uint32_t *labs_g, const double *c_g, int reps, double *out,
                                          long long *clk) {
    __shared__ uint32_t labs[KC][32];
    __shared__ __align__(16) double cs[KC][64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < KC * 32; i += blockDim.x) (&labs[0][0])[i] = labs_g[i];
    for (int i = threadIdx.x; i < KC * 64; i += blockDim.x) (&cs[0][0])[i] = c_g[i % (KC * 32)];
    __syncthreads();
    uint32_t rowpk[8];
    double a[16];
    for (int r = 0; r < 8; ++r) {
        uint32_t w0 = labs[2 * r][lane] & 0xFFFF, w1 = labs[2 * r + 1][lane] & 0xFFFF;
        rowpk[r] = (w1 << 16) | w0;
    }
    for (int r = 0; r < 16; ++r) a[r] = 0;
    const uint32_t cbase = (uint32_t)__cvta_generic_to_shared(&cs[0][16 * (warp & 3)]);
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 2
        for (int t = 0; t < KC; ++t) {
            const uint32_t w = labs[t][lane] & 0xFFFF;
            const uint32_t col = (w << 16) | w;
            const uint32_t addr = cbase + t * 64 * 8;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                asm("{\n\t.reg .pred p, q;\n\t.reg .b32 l0, h0, l1, h1;\n\t.reg .b64 d0, d1;\n\t"
                    "ld.shared.v4.u32 {l0, h0, l1, h1}, [%2];\n\t"
                    "setp.eq.f16x2 p|q, %3, %4;\n\t"
                    "selp.b32 h0, h0, 0, p;\n\t"
                    "selp.b32 h1, h1, 0, q;\n\t"
                    "mov.b64 d0, {l0, h0};\n\t"
                    "mov.b64 d1, {l1, h1};\n\t"
                    "add.f64 %0, %0, d0;\n\t"
                    "add.f64 %1, %1, d1;\n\t}"
                    : "+d"(a[2 * r]), "+d"(a[2 * r + 1])
                    : "r"(addr + r * 16), "r"(rowpk[r]), "r"(col));
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int r = 0; r < 16; ++r) s += a[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// V6: split C = Chi + Clo in fp32 (Chi exact on a 2^-19 grid), HSETP2 dual
// predicate, predicated FADDs, flush to fp64 every KC columns.
__global__ void __launch_bounds__(128) k6(const uint32_t *labs_g, const double *c_g, int reps, double *out,
                                          long long *clk) {
    __shared__ uint32_t labs[KC][32];
    __shared__ __align__(16) float2 cs[KC][64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < KC * 32; i += blockDim.x) (&labs[0][0])[i] = labs_g[i];
    for (int i = threadIdx.x; i < KC * 64; i += blockDim.x) {
        double c = c_g[i % (KC * 32)];
        float hi = (float)(rint(c * 524288.0) / 524288.0);
        (&cs[0][0])[i] = make_float2(hi, (float)(c - (double)hi));
    }
    __syncthreads();
    uint32_t rowpk[8];
    double a[16];
    for (int r = 0; r < 8; ++r) {
        uint32_t w0 = labs[2 * r][lane] & 0xFFFF, w1 = labs[2 * r + 1][lane] & 0xFFFF;
        rowpk[r] = (w1 << 16) | w0;
    }
    for (int r = 0; r < 16; ++r) a[r] = 0;
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        float h[16], l[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) h[r] = l[r] = 0.f;
#pragma unroll 4
        for (int t = 0; t < KC / 2; ++t) {
            const uint32_t w = labs[t][lane] & 0xFFFF;
            const uint32_t col = (w << 16) | w;
            const float4 *c4 = reinterpret_cast<const float4 *>(&cs[t][16 * (warp & 3)]);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const float4 c = c4[r];
                asm("{\n\t.reg .pred p, q;\n\t"
                    "setp.eq.f16x2 p|q, %8, %9;\n\t"
                    "@p add.f32 %0, %0, %4;\n\t"
                    "@p add.f32 %1, %1, %5;\n\t"
                    "@q add.f32 %2, %2, %6;\n\t"
                    "@q add.f32 %3, %3, %7;\n\t}"
                    : "+f"(h[2 * r]), "+f"(l[2 * r]), "+f"(h[2 * r + 1]), "+f"(l[2 * r + 1])
                    : "f"(c.x), "f"(c.y), "f"(c.z), "f"(c.w), "r"(rowpk[r]), "r"(col));
            }
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) a[r] += (double)h[r] + (double)l[r];
    }
    long long t1 = clock64();
    double s = 0;
    for (int r = 0; r < 16; ++r) s += a[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

void run6(int ctas_per_sm, uint32_t *dl, double *dc, double *dout, long long *dclk) {
    int sms = 148, grid = sms * ctas_per_sm, reps = 800;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k6<<<grid, 128>>>(dl, dc, 10, dout, dclk);
    cudaEventRecord(e0);
    k6<<<grid, 128>>>(dl, dc, reps, dout, dclk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double pairs = (double)grid * 4 * 32 * 16 * (KC / 2) * reps;
    printf("%-10s ctas/sm=%d  %.3f ms  %.3e pairs/s  %.1f pairs/clk/SM@1965\n", "F32SPLIT", ctas_per_sm, ms,
           pairs / (ms * 1e-3), pairs / (ms * 1e-3) / (sms * 1965e6));
}

void run5(int ctas_per_sm, uint32_t *dl, double *dc, double *dout, long long *dclk) {
    int sms = 148, grid = sms * ctas_per_sm, reps = 400;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k5<<<grid, 128>>>(dl, dc, 10, dout, dclk);
    cudaEventRecord(e0);
    k5<<<grid, 128>>>(dl, dc, reps, dout, dclk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double pairs = (double)grid * 4 * 32 * 16 * KC * reps;
    printf("%-10s ctas/sm=%d  %.3f ms  %.3e pairs/s  %.1f pairs/clk/SM@1965\n", "PTXSEL", ctas_per_sm, ms,
           pairs / (ms * 1e-3), pairs / (ms * 1e-3) / (sms * 1965e6));
}

void run4(int ctas_per_sm, uint32_t *dl, double *dc, double *dout, long long *dclk) {
    int sms = 148, grid = sms * ctas_per_sm, reps = 400;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k4<<<grid, 128>>>(dl, dc, 10, dout, dclk);
    cudaEventRecord(e0);
    k4<<<grid, 128>>>(dl, dc, reps, dout, dclk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double pairs = (double)grid * 4 * 32 * 16 * KC * reps;
    printf("%-10s ctas/sm=%d  %.3f ms  %.3e pairs/s  %.1f pairs/clk/SM@1965\n", "HSETP2SEL", ctas_per_sm, ms,
           pairs / (ms * 1e-3), pairs / (ms * 1e-3) / (sms * 1965e6));
}

template <int V>
void run(const char *name, int ctas_per_sm, uint32_t *dl, double *dc, double *dout, long long *dclk) {
    int sms = 148;
    int grid = sms * ctas_per_sm;
    int reps = 400;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<V><<<grid, 128>>>(dl, dc, 10, dout, dclk);
    cudaEventRecord(e0);
    k<V><<<grid, 128>>>(dl, dc, reps, dout, dclk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double pairs = (double)grid * 4 * 32 * 16 * KC * reps;
    int mhz = 0;
    cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
    double per_clk_sm = pairs / (ms * 1e-3) / (sms * 1965e6);
    printf("%-10s ctas/sm=%d  %.3f ms  %.3e pairs/s  %.1f pairs/clk/SM@1965\n", name, ctas_per_sm, ms,
           pairs / (ms * 1e-3), per_clk_sm);
}


// V7: as V5 with TWO chromosomes per lane sharing each broadcast C load:
// one ld.shared.v4 (C[j][r], C[j][r+1]) feeds 2 rows x 2 chromosomes x 32
// lanes = 128 pair updates (V5: 64), halving shared-memory wavefronts per pair.
__global__ void __launch_bounds__(128) k7(const uint32_t *labs_g, const double *c_g, int reps, double *out,
                                          long long *clk) {
    __shared__ uint32_t labs[KC][32];
    __shared__ __align__(16) double cs[KC][64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < KC * 32; i += blockDim.x) (&labs[0][0])[i] = labs_g[i];
    for (int i = threadIdx.x; i < KC * 64; i += blockDim.x) (&cs[0][0])[i] = c_g[i % (KC * 32)];
    __syncthreads();
    uint32_t rowA[4], rowB[4];
    double a[8], b[8];
    for (int r = 0; r < 4; ++r) {
        const uint32_t x0 = labs[2 * r][lane], x1 = labs[2 * r + 1][lane];
        rowA[r] = ((x1 & 0xFFFF) << 16) | (x0 & 0xFFFF);
        rowB[r] = (x1 & 0xFFFF0000u) | (x0 >> 16);
    }
    for (int r = 0; r < 8; ++r) a[r] = b[r] = 0;
    const uint32_t cbase = (uint32_t)__cvta_generic_to_shared(&cs[0][8 * (warp & 7)]);
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 2
        for (int t = 0; t < KC; ++t) {
            const uint32_t w = labs[t][lane];
            const uint32_t colA = (w << 16) | (w & 0xFFFF), colB = (w & 0xFFFF0000u) | (w >> 16);
            const uint32_t addr = cbase + t * 64 * 8;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                asm("{\n\t.reg .pred p, q, u, v;\n\t.reg .b32 l0, h0, l1, h1, g0, g1;\n\t.reg .b64 d0, d1, d2, d3;\n\t"
                    "ld.shared.v4.u32 {l0, h0, l1, h1}, [%4];\n\t"
                    "setp.eq.f16x2 p|q, %5, %6;\n\t"
                    "setp.eq.f16x2 u|v, %7, %8;\n\t"
                    "selp.b32 g0, h0, 0, p;\n\t"
                    "selp.b32 g1, h1, 0, q;\n\t"
                    "selp.b32 h0, h0, 0, u;\n\t"
                    "selp.b32 h1, h1, 0, v;\n\t"
                    "mov.b64 d0, {l0, g0};\n\t"
                    "mov.b64 d1, {l1, g1};\n\t"
                    "mov.b64 d2, {l0, h0};\n\t"
                    "mov.b64 d3, {l1, h1};\n\t"
                    "add.f64 %0, %0, d0;\n\t"
                    "add.f64 %1, %1, d1;\n\t"
                    "add.f64 %2, %2, d2;\n\t"
                    "add.f64 %3, %3, d3;\n\t}"
                    : "+d"(a[2 * r]), "+d"(a[2 * r + 1]), "+d"(b[2 * r]), "+d"(b[2 * r + 1])
                    : "r"(addr + r * 16), "r"(rowA[r]), "r"(colA), "r"(rowB[r]), "r"(colB));
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int r = 0; r < 8; ++r) s += a[r] + b[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

void run7(int ctas_per_sm, uint32_t *dl, double *dc, double *dout, long long *dclk) {
    int sms = 148, grid = sms * ctas_per_sm, reps = 400;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k7<<<grid, 128>>>(dl, dc, 10, dout, dclk);
    cudaEventRecord(e0);
    k7<<<grid, 128>>>(dl, dc, reps, dout, dclk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double pairs = (double)grid * 4 * 32 * 16 * KC * reps;
    printf("%-10s ctas/sm=%d  %.3f ms  %.3e pairs/s  %.1f pairs/clk/SM@1965\n", "PTXSEL2CH", ctas_per_sm, ms,
           pairs / (ms * 1e-3), pairs / (ms * 1e-3) / (sms * 1965e6));
}

int main() {
    uint32_t hl[KC * 32];
    double hc[KC * 32];
    for (int i = 0; i < KC * 32; ++i) {
        hl[i] = ((i * 2654435761u) >> 7) % 20 | ((((i * 40503u) >> 5) % 20) << 16);
        hc[i] = 0.001 * (i % 97);
    }
    uint32_t *dl;
    double *dc, *dout;
    long long *dclk;
    cudaMalloc(&dl, sizeof(hl));
    cudaMalloc(&dc, sizeof(hc));
    cudaMalloc(&dout, sizeof(double) * 148 * 16 * 128);
    cudaMalloc(&dclk, sizeof(long long) * 148 * 16);
    cudaMemcpy(dl, hl, sizeof(hl), cudaMemcpyHostToDevice);
    cudaMemcpy(dc, hc, sizeof(hc), cudaMemcpyHostToDevice);
    for (int occ : {2, 4, 6, 8}) {
        run5(occ, dl, dc, dout, dclk);
        run7(occ, dl, dc, dout, dclk);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
