// Per-phase cycles of the register TSQR factor kernel (block 0), built with -DCORU_QR_PROFILE.
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
    for (int it = 0; it < 3; ++it) {
        long long z[8] = {0};
        cudaMemcpyToSymbol(coru_gpu::g_qr_reg_ph, z, sizeof(z));
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        coru_gpu::tsqr_factor<double>(p, B, d, V, beta, T, R, r, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpyFromSymbol(z, coru_gpu::g_qr_reg_ph, sizeof(z));
        const double steps = double(d) * p.levels.size();
        printf("m=%ld d=%d levels=%zu kinds=%d factor %.1f us (%s) | per step cycles: warp0 vload %.0f apply %.0f (build %.0f) bar %.0f | builder vload %.0f apply %.0f build %.0f bar %.0f\n",
               m, d, p.levels.size(), int(p.levels[0].kind), ms * 1e3, cudaGetErrorString(cudaGetLastError()),
               z[0] / steps, z[1] / steps, z[2] / steps, z[3] / steps, z[4] / steps, z[5] / steps, z[6] / steps, z[7] / steps);
    }
}
