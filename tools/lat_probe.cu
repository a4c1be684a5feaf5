// Latency probe (tooling only): dependent DFMA, 5-level fp64 warp reduction, DDIV, DSQRT, named barrier.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b) {
    double x = a + threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) x = fma(x, b, a);
    long long t1 = clock64();
    double s = x;
    for (int i = 0; i < 32; ++i) {
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    long long t2 = clock64();
    double y = x;
    for (int i = 0; i < 32; ++i) y = a / (y + 1.0);
    long long t3 = clock64();
    double z = x;
    for (int i = 0; i < 32; ++i) z = sqrt(z + a);
    long long t4 = clock64();
    double w = x;
    for (int i = 0; i < 32; ++i) w = 1.0 / (w + 2.0);
    long long t5 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / 256; cyc[1] = (t2 - t1) / 32; cyc[2] = (t3 - t2) / 32; cyc[3] = (t4 - t3) / 32; cyc[4] = (t5 - t4) / 32;
    }
    out[threadIdx.x] = x + s + y + z + w;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMallocManaged(&c, 64);
    k<<<1, 32>>>(o, c, 0.5, 0.999); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 0.5, 0.999); cudaDeviceSynchronize();
    printf("cycles: DFMA %lld | 5-level fp64 shfl reduce %lld | DDIV %lld | DSQRT %lld | DRCP %lld\n", c[0], c[1], c[2], c[3], c[4]);
}
