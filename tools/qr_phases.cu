// Per-phase cycles of block 0 of the blocked TSQR factor kernel (built with -DCORU_QR_PROFILE).
#include <cstdio>
#include <vector>
#include "../paper_1810_07323_b200/csrc/tsqr.cu"
int main(int argc, char** argv) {
    const long m = argc > 1 ? atol(argv[1]) : 4000;
    const int d = argc > 2 ? atoi(argv[2]) : 60;
    int smem; cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    auto p = coru_gpu::plan_tsqr(m, d, 8, smem);
    std::vector<double> h(size_t(m) * d);
    unsigned s = 7;
    for (auto& x : h) { s = s * 1664525u + 1013904223u; x = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
    double *B, *V, *beta, *T, *R, *r;
    cudaMalloc(&B, h.size() * 8); cudaMemcpy(B, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&V, p.v_elems * 8); cudaMalloc(&beta, p.beta_elems * 8); cudaMalloc(&T, (p.t_elems + 1) * 8);
    cudaMalloc(&R, p.r_elems * 8); cudaMalloc(&r, d * d * 8);
    for (int it = 0; it < 2; ++it) {
        long long z[12] = {0};
        cudaMemcpyToSymbol(coru_gpu::g_qr_phase, z, sizeof(z));
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        coru_gpu::tsqr_factor<double>(p, B, d, V, beta, T, R, r, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpyFromSymbol(z, coru_gpu::g_qr_phase, sizeof(z));
        printf("m=%ld d=%d levels=%zu factor %.1f us | block0 cycles (summed over levels): load %lld chain %lld Tfac %lld trailing %lld export %lld | G %lld G-nosync %lld | total %lld cyc %lld ns (%s)\n",
               m, d, p.levels.size(), ms * 1e3, z[0], z[1], z[2], z[3], z[4], z[5], z[6], z[7], z[8], cudaGetErrorString(cudaGetLastError()));
    }
    long long tl[3 * 256];
    cudaMemcpyFromSymbol(tl, coru_gpu::g_qr_tl, sizeof(tl));
    printf("col: barrier-wake apply build (cycles), last level block 0\n");
    for (int j = 1; j < d; ++j)
        if (j % 16) printf("%d: %lld %lld %lld\n", j, tl[256 + j] - tl[j - 1], tl[512 + j] - tl[256 + j], tl[j] - tl[512 + j]);
}
