// How often do CUDA's log/sincos (Box-Muller on the device) differ from the host libm? (tooling)
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
static uint64_t sm(uint64_t& s) { uint64_t z = (s += 0x9E3779B97F4A7C15ULL); z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL; z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL; return z ^ (z >> 31); }
static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
__host__ __device__ inline double open01(uint64_t w) { return double((w >> 11) + 1) * 0x1.0p-53; }
__global__ void bm(const uint64_t* w, double* out, int pairs, int mode) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= pairs) return;
    double u1 = open01(w[2 * p]), u2 = open01(w[2 * p + 1]);
    double rad = sqrt(-2.0 * log(u1));
    double th = 2.0 * 3.141592653589793 * u2;
    double s, c;
    sincos(th, &s, &c);
    out[2 * p] = rad * c;
    out[2 * p + 1] = rad * s;
}
int main() {
    const int pairs = 4 << 20;
    std::vector<uint64_t> w(2 * pairs);
    uint64_t a = 42, b = 7, s[4];
    for (auto& x : s) x = sm(a) ^ sm(b);
    for (auto& x : w) {
        const uint64_t r = rotl(s[0] + s[3], 23) + s[0], t = s[1] << 17;
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
        x = r;
    }
    std::vector<double> host(2 * pairs), dev(2 * pairs);
    for (int p = 0; p < pairs; ++p) {
        double u1 = open01(w[2 * p]), u2 = open01(w[2 * p + 1]);
        double rad = std::sqrt(-2.0 * std::log(u1));
        double th = 2.0 * 3.141592653589793 * u2;
        host[2 * p] = rad * std::cos(th);
        host[2 * p + 1] = rad * std::sin(th);
    }
    uint64_t* dw; double* dout;
    cudaMalloc(&dw, w.size() * 8); cudaMalloc(&dout, dev.size() * 8);
    cudaMemcpy(dw, w.data(), w.size() * 8, cudaMemcpyHostToDevice);
    bm<<<(pairs + 255) / 256, 256>>>(dw, dout, pairs, 0);
    cudaMemcpy(dev.data(), dout, dev.size() * 8, cudaMemcpyDeviceToHost);
    long mism = 0; int64_t maxulp = 0;
    for (size_t i = 0; i < host.size(); ++i) {
        int64_t x, y; std::memcpy(&x, &host[i], 8); std::memcpy(&y, &dev[i], 8);
        if (x != y) { ++mism; int64_t d = x > y ? x - y : y - x; if (d > maxulp) maxulp = d; }
    }
    printf("values %zu mismatches %ld (%.4f%%) max ulp %lld\n", host.size(), mism, 100.0 * mism / host.size(), (long long)maxulp);
}
