// DMMA (mma.sync m16n8k8 f64) latency/throughput probe and LDS.64 latency (tooling only).
#include <cstdio>
#include "common.cuh"
using namespace coru_gpu;
__global__ void k(double* out, long long* cyc, int nw) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 % 1024);
    __syncthreads();
    double a[4] = {1e-3, 2e-3, 3e-3, 4e-3}, b[2] = {0.5, 0.25};
    double c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0}, c2[4] = {0, 0, 0, 0}, c3[4] = {0, 0, 0, 0};
    const int warp = threadIdx.x >> 5;
    long long t0 = clock64();
    if (warp < nw) for (int i = 0; i < 64; ++i) dmma_16x8x8(c0, a, b);
    long long t1 = clock64();
    if (warp < nw) for (int i = 0; i < 64; ++i) { dmma_16x8x8(c0, a, b); dmma_16x8x8(c1, a, b); dmma_16x8x8(c2, a, b); dmma_16x8x8(c3, a, b); }
    long long t2 = clock64();
    int idx = threadIdx.x & 31;
    for (int i = 0; i < 64; ++i) idx = int(sm[idx]) & 1023;
    long long t3 = clock64();
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / 64; cyc[1] = (t2 - t1) / 256; cyc[2] = (t3 - t2) / 64; }
    out[threadIdx.x] = c0[0] + c1[1] + c2[2] + c3[3] + idx;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64);
    for (int nw : {1, 4, 8, 16}) {
        k<<<1, 32 * nw>>>(o, c, nw); cudaDeviceSynchronize();
        k<<<1, 32 * nw>>>(o, c, nw); cudaDeviceSynchronize();
        printf("warps=%d: dependent DMMA %lld cyc | 4 independent chains %lld cyc/DMMA | LDS.64 dependent %lld cyc\n", nw, c[0], c[1], c[2]);
    }
}
