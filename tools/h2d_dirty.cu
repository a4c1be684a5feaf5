// Does a freshly written (dirty in CPU caches) pinned buffer copy slower than a clean one? (tooling)
#include <cstdio>
#include <thread>
#include <vector>
#include <immintrin.h>
#include <cuda_runtime.h>
static void fill(double* p, size_t n, int threads, bool nt, double v) {
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; ++t)
        ts.emplace_back([=] {
            size_t a = n * t / threads, b = n * (t + 1) / threads;
            a &= ~size_t(7);
            if (t + 1 == threads) b = n;
            for (size_t i = a; i < b; i += 2) {
                if (nt) _mm_stream_pd(p + i, _mm_set_pd(v + i + 1, v + i));
                else { p[i] = v + i; p[i + 1] = v + i + 1; }
            }
            if (nt) _mm_sfence();
        });
    for (auto& t : ts) t.join();
}
int main() {
    const size_t n = 4000 * 64;
    double *h, *d;
    cudaMallocHost(&h, n * 8);
    cudaMalloc(&d, n * 8);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 4; ++mode) for (int rep = 0; rep < 3; ++rep) {
        const int threads = mode == 3 ? 1 : 16;
        fill(h, n, threads, mode == 1, rep + mode);
        if (mode == 2) { cudaMemcpyAsync(d, h, n * 8, cudaMemcpyHostToDevice, s); cudaStreamSynchronize(s); }
        cudaEventRecord(e0, s);
        cudaMemcpyAsync(d, h, n * 8, cudaMemcpyHostToDevice, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%s: %.1f us\n", mode == 0 ? "dirty (16 thr)" : mode == 1 ? "non-temporal (16 thr)" : mode == 2 ? "second copy" : "dirty (1 thr)", ms * 1e3);
    }
}
