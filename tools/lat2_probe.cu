// Latency probe (tooling only): per-op dependent latency in cycles on one warp.
#include <cstdio>
#include "../paper_1810_07323_b200/csrc/common.cuh"
using namespace coru_gpu;
__device__ __forceinline__ double rsq64(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double h = 0.5 * x;
    r = r * fma(-h * r, r, 1.5);
    r = r * fma(-h * r, r, 1.5);
    return r;
}
__device__ __forceinline__ double rcp64(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}
__global__ void k(double* out, long long* cyc, double a, double b, int nw) {
    __shared__ double sm[1024];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    double x = a + threadIdx.x * 1e-9;
    long long t[16]; int n = 0;
    t[n++] = clock64();
    for (int i = 0; i < 256; ++i) x = fma(x, b, a);
    t[n++] = clock64();
    double s = x;
    for (int i = 0; i < 32; ++i) s = warp_sum(s);            // 5-level double butterfly
    t[n++] = clock64();
    double r = x + 1.5;
    for (int i = 0; i < 32; ++i) r = fast_rsqrt(r + 1.0);     // F2F + MUFU + 4 DFMA
    t[n++] = clock64();
    double q = x + 1.5;
    for (int i = 0; i < 32; ++i) q = fast_rcp(q + 1.0);
    t[n++] = clock64();
    double f = x;
    for (int i = 0; i < 32; ++i) f = double(float(f)) + 1.0;   // F2F pair
    t[n++] = clock64();
    int idx = threadIdx.x;
    double l = 0;
    for (int i = 0; i < 64; ++i) { l += sm[idx]; idx = (int(l) & 1) + threadIdx.x; }   // dependent LDS
    t[n++] = clock64();
    for (int i = 0; i < 64; ++i) __syncthreads();
    t[n++] = clock64();
    double r2 = x + 1.5;
    for (int i = 0; i < 32; ++i) r2 = rsq64(r2 + 1.0);
    t[n++] = clock64();
    double q2 = x + 1.5;
    for (int i = 0; i < 32; ++i) q2 = rcp64(q2 + 1.0);
    t[n++] = clock64();
    double e1 = 0, e2 = 0;
    for (int i = 0; i < 1000; ++i) { double y = 1.0 + i * 0.37 + threadIdx.x; double a1 = rsq64(y), a2 = 1.0 / sqrt(y); e1 = fmax(e1, fabs(a1 - a2) / a2); double b1 = rcp64(y), b2 = 1.0 / y; e2 = fmax(e2, fabs(b1 - b2) / b2); }
    float fs = float(x);
    for (int i = 0; i < 32; ++i) for (int o = 16; o > 0; o >>= 1) fs += __shfl_xor_sync(0xffffffffu, fs, o);
    t[n++] = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = (t[1] - t[0]) / 256; cyc[1] = (t[2] - t[1]) / 32; cyc[2] = (t[3] - t[2]) / 32;
        cyc[3] = (t[4] - t[3]) / 32; cyc[4] = (t[5] - t[4]) / 32; cyc[5] = (t[6] - t[5]) / 64;
        cyc[6] = (t[7] - t[6]) / 64; cyc[7] = (t[10] - t[9]) / 32; cyc[8] = (t[8] - t[7]) / 32; cyc[9] = (t[9] - t[8]) / 32;
        cyc[10] = (long long)(e1 * 1e18); cyc[11] = (long long)(e2 * 1e18);
    }
    out[threadIdx.x] = x + s + r + q + f + l + fs + r2 + q2;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 256);
    const char* names[] = {"DFMA dep", "warp_sum<double> 5 lvl", "fast_rsqrt", "fast_rcp", "F2F d->f->d +DADD",
                           "LDS.64 dep", "__syncthreads", "warp_sum<float> 5 lvl", "rsq64(MUFU f64)", "rcp64(MUFU f64)", "rsq64 relerr e-18", "rcp64 relerr e-18"};
    for (int nw : {1, 2, 8, 32}) {
        for (int rep = 0; rep < 2; ++rep) { k<<<1, 32 * nw>>>(o, c, 0.5, 0.999, nw); cudaDeviceSynchronize(); }
        printf("warps=%d:", nw);
        for (int i = 0; i < 12; ++i) printf("  %s=%lld", names[i], c[i]);
        printf("\n");
    }
    return 0;
}
