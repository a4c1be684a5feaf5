// Device generation of the Gaussian test matrix Φ = gaussian(n, d, {seed, stream}) — the same
// recipe as rng_host.cpp (reference proj/include/coru/rng.hpp:13-112): SplitMix64 seeding,
// xoshiro256++ words, uniform_open01, Box–Muller r·cos θ then the spare r·sin θ, row-major fill.
//
// The word stream is bit-identical to the reference's (integer arithmetic + exact GF(2) jumps).
// The Gaussian values use the device log/sincos (≤ 1-2 ulp) instead of the host libm, so an entry
// can differ from the host generator by a few ulp (measured: ~14% of entries, max 3 ulp); the
// host generator stays available for bit-exact reproduction (coru_ctx_set_phi_mode).
//
// Layout: one warp per run of kWordsPerWarp consecutive words. The warp jumps the seed state to its
// first word with the precomputed M^(2^i) tables (lane l owns state bits 8l..8l+7, one GF(2)
// row-parity each), then kChains lanes step disjoint sub-runs of the word stream sequentially into
// shared memory, and every lane turns word pairs into Gaussians.
#include <cstdint>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "rng_dev.cuh"

namespace coru_gpu {

const uint64_t* jump_table_words(int* nbits);  // rng_host.cpp: nbits x 256 rows x 4 words

namespace {

constexpr int kWordsPerWarp = 256;  // 128 Box–Muller pairs per warp
constexpr int kChains = 8;          // sequential steppers per warp (32 words each)
constexpr int kWarps = 4;           // warps per CTA

__host__ __device__ inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

__device__ inline uint64_t xo_next(uint64_t (&s)[4]) {
    const uint64_t r = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return r;
}

// s <- M^k s for a warp-uniform k (all lanes hold the same s on entry and exit).
__device__ void warp_jump(uint64_t (&s)[4], uint64_t k, const uint64_t* __restrict__ table, int nbits,
                          unsigned char* bytes) {
    const int lane = threadIdx.x & 31;
    for (int i = 0; i < nbits && k; ++i, k >>= 1) {
        if (!(k & 1u)) continue;
        const uint64_t* m = table + size_t(i) * 256 * 4 + size_t(lane) * 8 * 4;  // rows 8·lane .. 8·lane+7
        unsigned b = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const ulonglong2 lo = __ldg(reinterpret_cast<const ulonglong2*>(m + r * 4));
            const ulonglong2 hi = __ldg(reinterpret_cast<const ulonglong2*>(m + r * 4 + 2));
            const uint64_t p = (lo.x & s[0]) ^ (lo.y & s[1]) ^ (hi.x & s[2]) ^ (hi.y & s[3]);
            b |= unsigned(__popcll(p) & 1) << r;
        }
        bytes[lane] = static_cast<unsigned char>(b);  // bit 8·lane + r of the new state
        __syncwarp();
        const uint64_t* w = reinterpret_cast<const uint64_t*>(bytes);
        s[0] = w[0];
        s[1] = w[1];
        s[2] = w[2];
        s[3] = w[3];
        __syncwarp();
    }
}

template <typename OutT>
__global__ void __launch_bounds__(kWarps * 32)
    k_gaussian(const uint64_t* __restrict__ table, int nbits, uint64_t s0, uint64_t s1, uint64_t s2, uint64_t s3,
               int64_t total, int64_t cols, int64_t ldo, OutT* __restrict__ out) {
    __shared__ __align__(16) uint64_t words[kWarps][kWordsPerWarp];
    __shared__ __align__(8) unsigned char bytes[kWarps][32];
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int64_t warp = int64_t(blockIdx.x) * kWarps + wi;
    const int64_t w0 = warp * kWordsPerWarp;   // first word of this warp (element index of the pair start)
    const int64_t nwords = ((total + 1) / 2) * 2;
    if (w0 >= nwords) return;
    uint64_t s[4] = {s0, s1, s2, s3};
    warp_jump(s, uint64_t(w0), table, nbits, bytes[wi]);
    // kChains lanes each step their own sub-run: lane c starts kWordsPerWarp/kChains·c words later.
    constexpr int kSub = kWordsPerWarp / kChains;
    if (lane < kChains) {
        uint64_t t[4] = {s[0], s[1], s[2], s[3]};
        // advance to the sub-run start by stepping (c·kSub <= 224 steps on the last chain)
        for (int j = 0; j < lane * kSub; ++j) xo_next(t);
        for (int j = 0; j < kSub; ++j) words[wi][lane * kSub + j] = xo_next(t);
    }
    __syncwarp();
    for (int p = lane; p < kWordsPerWarp / 2; p += 32) {
        const int64_t e = w0 + 2 * p;
        if (e >= total) break;
        const uint64_t a = words[wi][2 * p], b = words[wi][2 * p + 1];
        const double u1 = double((a >> 11) + 1) * 0x1.0p-53;
        const double u2 = double((b >> 11) + 1) * 0x1.0p-53;
        const double rad = sqrt(-2.0 * log(u1));
        const double theta = 2.0 * 3.141592653589793 * u2;
        double sn, cs;
        sincos(theta, &sn, &cs);
        out[(e / cols) * ldo + e % cols] = static_cast<OutT>(__dmul_rn(rad, cs));
        if (e + 1 < total) out[((e + 1) / cols) * ldo + (e + 1) % cols] = static_cast<OutT>(__dmul_rn(rad, sn));
    }
}

struct DeviceTable {
    uint64_t* ptr = nullptr;
    int nbits = 0;
};

}  // namespace

// The jump tables are uploaded once per device and stay resident (48 x 8 KB).
static cudaError_t device_table(int dev, DeviceTable* out) {
    static std::mutex mu;
    static std::vector<DeviceTable> tables;
    std::lock_guard<std::mutex> lk(mu);
    if (int(tables.size()) <= dev) tables.resize(size_t(dev) + 1);
    DeviceTable& t = tables[size_t(dev)];
    if (!t.ptr) {
        int nbits = 0;
        const uint64_t* host = jump_table_words(&nbits);
        const size_t bytes = size_t(nbits) * 256 * 4 * sizeof(uint64_t);
        cudaError_t e = cudaMalloc(&t.ptr, bytes);
        if (e != cudaSuccess) return e;
        e = cudaMemcpy(t.ptr, host, bytes, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(t.ptr);
            t.ptr = nullptr;
            return e;
        }
        t.nbits = nbits;
    }
    *out = t;
    return cudaSuccess;
}

template <typename OutT>
cudaError_t gaussian_dev(int64_t rows, int64_t cols, const uint64_t state[4], OutT* out, int64_t ldo,
                         cudaStream_t st) {
    const int64_t total = rows * cols;
    if (total <= 0) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    DeviceTable t;
    e = device_table(dev, &t);
    if (e != cudaSuccess) return e;
    if (ldo != cols) {
        e = cudaMemsetAsync(out, 0, size_t(rows) * ldo * sizeof(OutT), st);
        if (e != cudaSuccess) return e;
    }
    const int64_t warps = (total + kWordsPerWarp - 1) / kWordsPerWarp;
    const unsigned grid = unsigned((warps + kWarps - 1) / kWarps);
    k_gaussian<OutT><<<grid, kWarps * 32, 0, st>>>(t.ptr, t.nbits, state[0], state[1], state[2], state[3], total, cols,
                                                   ldo, out);
    return cudaGetLastError();
}

template cudaError_t gaussian_dev<double>(int64_t, int64_t, const uint64_t*, double*, int64_t, cudaStream_t);
template cudaError_t gaussian_dev<float>(int64_t, int64_t, const uint64_t*, float*, int64_t, cudaStream_t);

}  // namespace coru_gpu
