// Microbenchmark: cycles of warp_larft (16x16) alone and while other warps run DMMA GEMMs.
#include <cstdio>
#include "cta_blas.cuh"
using namespace coru_gpu;
__global__ void k(double* out, long long* cyc, int busy) {
    __shared__ double G[16 * 16], beta[16], Tm[16 * 16];
    extern __shared__ double C[];
    double* V = C + 256 * 48;
    __shared__ double Y[16 * 48], scr[512];
    for (int e = threadIdx.x; e < 256; e += blockDim.x) G[e] = 1.0 / (1 + e % 17);
    for (int e = threadIdx.x; e < 16; e += blockDim.x) beta[e] = 1.5;
    for (int e = threadIdx.x; e < 256 * 24; e += blockDim.x) V[e] = 0.001 * (e % 13);
    for (int e = threadIdx.x; e < 256 * 48; e += blockDim.x) C[e] = 0.002 * (e % 7);
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    long long t0 = clock64();
    if (warp == 0) {
        for (int it = 0; it < 4; ++it) warp_larft<double>(16, G, 16, beta, Tm, 16);
        if (threadIdx.x == 0) cyc[0] = clock64() - t0;
    } else if (busy) {
        for (int it = 0; it < 4; ++it)
            cta_mm_f64(16, 44, 250, V, 24, 1, C, 1, 256, Y, 48, 1, 1.0, false, scr, 512, 1, blockDim.x / 32 - 1, 15);
        if (threadIdx.x == 32) cyc[1] = clock64() - t0;
    }
    __syncthreads();
    if (busy == 2) {
        long long t1 = clock64();
        for (int it = 0; it < 4; ++it) {
            cta_mm(16, 16, 250, V, 24, 1, V, 1, 24, G, 16, 1, 1.0, false, scr, 512);
            __syncthreads();
        }
        if (threadIdx.x == 0) cyc[2] = clock64() - t1;
    }
    if (threadIdx.x < 256) out[threadIdx.x] = Tm[threadIdx.x] + Y[threadIdx.x];
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 72 * 8);
    for (int busy = 0; busy < 3; ++busy) for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(c, 0, 64);
        k<<<1, 512, 256 * 72 * 8>>>(o, c, busy);
        long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
        printf("busy=%d larft x4: %lld cycles, Y x4: %lld cycles G x4: %lld (%s)\n", busy, h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
    }
}
