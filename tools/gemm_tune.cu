// Sweep the FP64 A-pass GEMM configurations on the BASELINE shapes (tooling only).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1810_07323_b200/csrc/gemm.cuh"
using namespace coru_gpu;
__global__ void fill(double* p, size_t n, double s) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        p[i] = double((i * 2654435761u) % 1000) * s - 0.5;
}
int main() {
    struct Shape { long m, n; int d; const char* name; };
    Shape shapes[] = {{4000, 4000, 60, "C2"}, {200000, 2000, 110, "C3"}, {32768, 32768, 220, "C4"}};
    const int only = getenv("TUNE_ONLY") ? atoi(getenv("TUNE_ONLY")) : -1;
    int si = -1;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (auto& s : shapes) {
        if (only >= 0 && ++si != only) continue;
        double *A, *X, *Y, *C, *ws;
        const int dp = (s.d + 7) / 8 * 8;
        cudaMalloc(&A, size_t(s.m) * s.n * 8);
        cudaMalloc(&X, size_t(s.n) * dp * 8); cudaMalloc(&Y, size_t(s.m) * dp * 8);
        cudaMalloc(&C, size_t(std::max(s.m, s.n)) * dp * 8);
        fill<<<1024, 256>>>(A, size_t(s.m) * s.n, 1e-3); fill<<<256, 256>>>(X, size_t(s.n) * dp, 1e-3); fill<<<256, 256>>>(Y, size_t(s.m) * dp, 1e-3);
        size_t wsz = 0;
        for (int cfg = 0; cfg < gemm_f64_num_configs(); ++cfg)
            for (int op = 0; op < 2; ++op) {
                GemmPlan p = plan_gemm_f64_cfg(op ? Op::T : Op::N, op ? s.n : s.m, op ? s.m : s.n, s.d, sms, cfg);
                wsz = std::max(wsz, size_t(p.ws_elems));
            }
        cudaMalloc(&ws, wsz * 8 + 256);
        const double flops = 2.0 * s.m * s.n * s.d;
        for (int cfg = 0; cfg < gemm_f64_num_configs(); ++cfg) {
            GemmPlan p0 = plan_gemm_f64_cfg(Op::N, s.m, s.n, s.d, sms, cfg);
            if (p0.bn >= s.d + 32) continue;  // skip tiles much wider than the sketch
            for (int op = 0; op < 2; ++op) {
                const Op o = op ? Op::T : Op::N;
                GemmPlan p = plan_gemm_f64_cfg(o, op ? s.n : s.m, op ? s.m : s.n, s.d, sms, cfg);
                auto run = [&] {
                    if (o == Op::N) gemm_f64(o, A, s.n, X, dp, C, dp, s.m, s.n, s.d, p, ws, 0);
                    else gemm_f64(o, A, s.n, Y, dp, C, dp, s.n, s.m, s.d, p, ws, 0);
                };
                for (int i = 0; i < 3; ++i) run();
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                const int reps = s.m * s.n > 1e9 ? 3 : 20;
                cudaEventRecord(e0);
                for (int i = 0; i < reps; ++i) run();
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
                printf("%s op%s cfg %2d (bm %3d bn %3d P %3d seg %2d fix %d): %8.1f us %5.1f TF  %s\n", s.name, op ? "T" : "N", cfg,
                       p.bm, p.bn, p.splits, p.max_seg, int(p.fixup), ms * 1e3, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
            }
        }
        cudaFree(A); cudaFree(X); cudaFree(Y); cudaFree(C); cudaFree(ws);
    }
}
