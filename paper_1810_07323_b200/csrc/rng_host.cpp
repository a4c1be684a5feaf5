// Host generation of the Gaussian test matrix Φ = gaussian(n, d, {seed, stream}), bit-exact with
// the reference recipe (proj/include/coru/rng.hpp):
//   SplitMix64 state expansion (rng.hpp:23-35), xoshiro256++ with state SM(seed)_i ^ SM(stream)_i and
//   the all-zero guard (rng.hpp:41-61), uniform_open01 = ((x>>11)+1)·2^-53 (rng.hpp:64), Box–Muller
//   r = sqrt(-2 ln u1), θ = 2π·u2, r·cos θ first then the spare r·sin θ (rng.hpp:86-98), row-major
//   fill (rng.hpp:107-112).
// Φ stays on the host on purpose: bit-exactness is defined by the host libm's log/sin/cos, which
// the device's math library does not reproduce. The serial part is only the xoshiro word stream
// (~1 ns/word); the transcendental Box–Muller transform is split over host threads, each pair
// being a pure function of its two words, so the output is identical for any thread count.
// Compiled with -ffp-contract=off (no FMA contraction on the host).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace coru_gpu {

namespace {

inline uint64_t splitmix_next(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

struct Xoshiro {
    uint64_t s[4];
    Xoshiro(uint64_t seed, uint64_t stream) {
        uint64_t a = seed, b = stream;
        bool zero = true;
        for (auto& w : s) {
            w = splitmix_next(a) ^ splitmix_next(b);
            zero = zero && w == 0;
        }
        if (zero) s[0] = 1;
    }
    uint64_t next() {
        const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return r;
    }
};

inline double open01(uint64_t w) { return static_cast<double>((w >> 11) + 1) * 0x1.0p-53; }

// Pair p -> (r cos θ, r sin θ) from words 2p, 2p+1.
inline void box_muller(uint64_t w1, uint64_t w2, double& c, double& s) {
    const double u1 = open01(w1), u2 = open01(w2);
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * 3.141592653589793 * u2;  // 2·std::numbers::pi·u2
    s = r * std::sin(theta);
    c = r * std::cos(theta);
}

}  // namespace

// Writes rows x cols Gaussians. Element e (row-major index) goes to out[(e / cols) * ldo + e % cols]
// converted to OutT (fp32 rounds the fp64 value). threads <= 1 runs serially.
template <typename OutT>
void gaussian_host(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, OutT* out, int64_t ldo,
                   int threads) {
    const int64_t total = rows * cols;
    const int64_t pairs = (total + 1) / 2;
    std::vector<uint64_t> words(size_t(2 * pairs));
    Xoshiro x(seed, stream);
    for (auto& w : words) w = x.next();
    // Pair p fills row-major elements 2p and 2p+1; (row, col) advance incrementally (no division
    // in the loop — an int64 divide per element cost more than the transcendental functions).
    auto work = [&](int64_t p0, int64_t p1) {
        int64_t e = 2 * p0, r = e / cols, c = e % cols;
        auto put = [&](double v) {
            out[r * ldo + c] = static_cast<OutT>(v);
            if (++c == cols) {
                c = 0;
                ++r;
            }
        };
        for (int64_t p = p0; p < p1; ++p) {
            double cv, sv;
            box_muller(words[size_t(2 * p)], words[size_t(2 * p + 1)], cv, sv);
            put(cv);
            if (2 * p + 1 < total) put(sv);
        }
    };
    if (threads <= 1 || pairs < 4096) {
        work(0, pairs);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, pairs * t / threads, pairs * (t + 1) / threads);
    for (auto& th : pool) th.join();
}

template void gaussian_host<double>(int64_t, int64_t, uint64_t, uint64_t, double*, int64_t, int);
template void gaussian_host<float>(int64_t, int64_t, uint64_t, uint64_t, float*, int64_t, int);

}  // namespace coru_gpu
