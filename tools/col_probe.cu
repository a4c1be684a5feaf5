// Panel-chain probe (tooling only): NW warps, warp w owns one 256-row column (8 values per lane in
// registers) and, for every earlier column j < w, waits for reflector j (named barrier pair), applies
// it (8 LDS + dot + warp_sum + update), then builds its own reflector (squares + warp_sum + scalars
// + 16 STS) and hands off. Reports cycles per column on the critical path, with ablations.
#include <cstdio>
#include "../paper_1810_07323_b200/csrc/common.cuh"
using namespace coru_gpu;
__device__ __forceinline__ void bsync(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
__device__ __forceinline__ void barrive(int id, int cnt) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
template <int MODE>
__global__ void k(double* out, long long* cyc) {
    __shared__ double Vp[16 * 264];
    __shared__ double beta[16];
    __shared__ double W[4 * 264];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nbp = blockDim.x >> 5;
    double x[8];
    for (int u = 0; u < 8; ++u) x[u] = 1.0 + 0.001 * (lane + 32 * u) + warp;
    __syncthreads();
    long long t0 = clock64();
    for (int rep = 0; rep < 4; ++rep) {
        for (int jj = 0; jj <= warp; ++jj) {
            const int j = jj;
            if (jj < warp) {
                if (MODE == 1 || jj + 1 == warp) bsync(1 + jj, MODE == 1 ? 32 * (nbp - jj) : 64);
                else { if (MODE != 2) bsync(1 + jj, 32 * (nbp - jj)); }
                const double bj = beta[jj];
                const double* vj = Vp + jj * 264;
                double v[8], pr[8];
                for (int u = 0; u < 8; ++u) { v[u] = vj[lane + 32 * u]; pr[u] = v[u] * x[u]; }
                for (int h = 4; h > 0; h >>= 1) for (int u = 0; u < h; ++u) pr[u] += pr[u + h];
                const double s = warp_sum(pr[0]) * bj;
                for (int u = 0; u < 8; ++u) x[u] -= s * v[u];
            } else {
                double sq[8];
                for (int u = 0; u < 8; ++u) { const int r = lane + 32 * u; sq[u] = r > j ? x[u] * x[u] : 0.0; if (r == j) W[(warp & 3) * 264 + j] = x[u]; }
                for (int h = 4; h > 0; h >>= 1) for (int u = 0; u < h; ++u) sq[u] += sq[u + h];
                const double sig = warp_sum(sq[0]);
                __syncwarp();
                const double x0 = W[(warp & 3) * 264 + j];
                double mu, v0, bb, rv;
                reflector_scalars(x0, sig + 1e-3, mu, v0, bb, rv);
                for (int u = 0; u < 8; ++u) { const int r = lane + 32 * u; x[u] = r > j ? x[u] * rv : (r == j ? mu : x[u]); }
                double* vj = Vp + jj * 264;
                for (int u = 0; u < 8; ++u) { const int r = lane + 32 * u; W[(warp & 3) * 264 + r] = x[u]; vj[r] = r > j ? x[u] : (r == j ? 1.0 : 0.0); }
                if (lane == 0) beta[jj] = bb * 1e-6;
                if (jj + 1 < nbp) barrive(1 + jj, MODE == 1 || MODE == 0 ? (MODE == 1 ? 32 * (nbp - jj) : 64) : 64);
            }
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[MODE] = (t1 - t0) / (4 * nbp);
    for (int u = 0; u < 8; ++u) out[threadIdx.x * 8 + u] = x[u];
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 512 * 8 * 8); cudaMallocManaged(&c, 64);
    const char* nm[] = {"pair-barrier (critical warp only; others unsynchronised: wrong but timing)",
                        "convoy barrier (all later warps, as before)", "critical-only, no others barrier"};
    for (int nw : {16, 8, 2}) {
        k<1><<<1, 32 * nw>>>(o, c); k<1><<<1, 32 * nw>>>(o, c);
        k<2><<<1, 32 * nw>>>(o, c); k<2><<<1, 32 * nw>>>(o, c);
        cudaDeviceSynchronize();
        printf("warps=%d: convoy %lld cyc/col, critical-only %lld cyc/col [%s]\n", nw, c[1], c[2], cudaGetErrorString(cudaGetLastError()));
    }
}
