// Per-phase cycle counts of the QRCP kernel (built with -DCORU_QRCP_PROFILE; tooling only).
#include <cstdio>
#include <vector>
#include "../paper_1810_07323_b200/csrc/qrcp.cu"
int main(int argc, char** argv) {
    const int d = argc > 1 ? atoi(argv[1]) : 60;
    std::vector<double> h(d * d);
    unsigned s = 1;
    for (auto& x : h) { s = s * 1664525u + 1013904223u; x = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
    double *M, *Q, *T, *scr; int64_t* perm;
    cudaMalloc(&M, d * d * 8); cudaMalloc(&Q, d * d * 8); cudaMalloc(&T, d * d * 8);
    cudaMalloc(&scr, coru_gpu::qrcp_scratch_elems(d) * 8); cudaMalloc(&perm, d * 8);
    cudaMemcpy(M, h.data(), d * d * 8, cudaMemcpyHostToDevice);
    int smem; cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    for (int r = 0; r < 3; ++r) coru_gpu::qrcp<double>(M, d, d, Q, d, T, d, perm, scr, smem, 0);
    long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(coru_gpu::g_qrcp_phase, z, sizeof(z));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    coru_gpu::qrcp<double>(M, d, d, Q, d, T, d, perm, scr, smem, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpyFromSymbol(z, coru_gpu::g_qrcp_phase, sizeof(z));
    printf("d=%d: %.1f us; cycles phaseA %lld phaseB %lld Qform %lld total %lld (%s)\n", d, ms * 1e3, z[0], z[1], z[2], z[3],
           cudaGetErrorString(cudaGetLastError()));
}
