// Host generation of the Gaussian test matrix Φ = gaussian(n, d, {seed, stream}), bit-exact with
// the reference recipe (proj/include/coru/rng.hpp):
//   SplitMix64 state expansion (rng.hpp:23-35), xoshiro256++ with state SM(seed)_i ^ SM(stream)_i and
//   the all-zero guard (rng.hpp:41-61), uniform_open01 = ((x>>11)+1)·2^-53 (rng.hpp:64), Box–Muller
//   r = sqrt(-2 ln u1), θ = 2π·u2, r·cos θ first then the spare r·sin θ (rng.hpp:86-98), row-major
//   fill (rng.hpp:107-112).
//
// Φ stays on the host on purpose: bit-exactness is defined by the host libm's log/sin/cos, which
// the device math library does not reproduce. Both halves are parallel and exact:
//   * the xoshiro256++ transition is linear over GF(2)^256, so every worker jumps straight to its
//     first word with precomputed M^(2^i) (popcount(offset) 256x256 bit mat-vecs) and then runs
//     the ordinary recurrence — the word stream is identical to the serial one;
//   * each Box–Muller pair is a pure function of its two words.
// Workers come from a persistent pool (no thread creation per call). Compiled with
// -ffp-contract=off (no FMA contraction on the host).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <emmintrin.h>

namespace coru_gpu {

namespace {

inline uint64_t splitmix_next(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

struct State {
    uint64_t s[4];
};

inline State seed_state(uint64_t seed, uint64_t stream) {
    State st;
    uint64_t a = seed, b = stream;
    bool zero = true;
    for (auto& w : st.s) {
        w = splitmix_next(a) ^ splitmix_next(b);
        zero = zero && w == 0;
    }
    if (zero) st.s[0] = 1;
    return st;
}

inline uint64_t next_word(State& st) {
    uint64_t* s = st.s;
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

// 256x256 GF(2) matrix, row i = bit mask over the 256 state bits feeding output bit i.
struct Gf2 {
    uint64_t row[256][4];
};

inline int bit(const State& v, int i) { return int((v.s[i >> 6] >> (i & 63)) & 1u); }

State mul(const Gf2& m, const State& v) {
    State out{{0, 0, 0, 0}};
    for (int i = 0; i < 256; ++i) {
        const uint64_t p = (m.row[i][0] & v.s[0]) ^ (m.row[i][1] & v.s[1]) ^ (m.row[i][2] & v.s[2]) ^
                           (m.row[i][3] & v.s[3]);
        if (__builtin_parityll(p)) out.s[i >> 6] |= uint64_t(1) << (i & 63);
    }
    return out;
}

Gf2 square(const Gf2& a) {
    // (A·A) row i = XOR of rows k of A for every bit k set in A's row i.
    Gf2 c;
    std::memset(&c, 0, sizeof(c));
    for (int i = 0; i < 256; ++i)
        for (int k = 0; k < 256; ++k)
            if ((a.row[i][k >> 6] >> (k & 63)) & 1u)
                for (int w = 0; w < 4; ++w) c.row[i][w] ^= a.row[k][w];
    return c;
}

constexpr int kJumpBits = 48;  // offsets below 2^48 words

// jump[i] = M^(2^i) for the state transition M of one xoshiro256++ step.
const std::vector<Gf2>& jump_table() {
    static std::vector<Gf2> table = [] {
        std::vector<Gf2> t(kJumpBits);
        Gf2& m = t[0];
        std::memset(&m, 0, sizeof(m));
        for (int j = 0; j < 256; ++j) {  // column j = M e_j
            State e{{0, 0, 0, 0}};
            e.s[j >> 6] = uint64_t(1) << (j & 63);
            next_word(e);
            for (int i = 0; i < 256; ++i)
                if (bit(e, i)) m.row[i][j >> 6] |= uint64_t(1) << (j & 63);
        }
        for (int k = 1; k < kJumpBits; ++k) t[k] = square(t[k - 1]);
        return t;
    }();
    return table;
}

State jump(State s, uint64_t k) {
    const auto& t = jump_table();
    for (int i = 0; i < kJumpBits && k; ++i, k >>= 1)
        if (k & 1u) s = mul(t[size_t(i)], s);
    return s;
}

inline double open01(uint64_t w) { return static_cast<double>((w >> 11) + 1) * 0x1.0p-53; }

// Persistent worker pool: run(n, f) calls f(0..n-1) on n workers (the caller is worker 0).
class Pool {
public:
    void run(int n, const std::function<void(int)>& f) {
        if (n <= 1) {
            f(0);
            return;
        }
        std::unique_lock<std::mutex> call(call_mu_);  // one dispatch at a time
        ensure(n - 1);
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &f;
            active_ = n - 1;
            pending_ = n - 1;
            ++gen_;
        }
        cv_.notify_all();
        f(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }

private:
    void ensure(int workers) {
        while (int(threads_.size()) < workers) {
            const int id = int(threads_.size()) + 1;
            threads_.emplace_back([this, id] { loop(id); });
        }
    }
    void loop(int id) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)>* job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                if (id > active_) continue;
                job = job_;
            }
            (*job)(id);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<std::thread> threads_;
    const std::function<void(int)>* job_ = nullptr;
    int active_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

Pool& pool() {
    static Pool p;
    return p;
}

}  // namespace

// The same pool for other host-side bulk work (staging copies of pageable buffers, capi.cu).
void host_parallel(int n, const std::function<void(int)>& f) { pool().run(n, f); }

const uint64_t* jump_table_words(int* nbits) {
    static_assert(sizeof(Gf2) == 256 * 4 * sizeof(uint64_t), "dense table");
    *nbits = kJumpBits;
    return &jump_table()[0].row[0][0];
}

void seed_state_words(uint64_t seed, uint64_t stream, uint64_t out[4]) {
    const State s = seed_state(seed, stream);
    for (int i = 0; i < 4; ++i) out[i] = s.s[i];
}

// Non-temporal 8/4-byte store: the staging buffer is read next by a DMA engine, and a PCIe read of
// lines left dirty in the CPU caches runs ~8x slower than one from memory (measured on the B200
// box: 2 MB in ~340 us dirty vs ~43 us written with movnti).
inline void store_stream(double* p, double v) {
    long long b;
    std::memcpy(&b, &v, 8);
    _mm_stream_si64(reinterpret_cast<long long*>(p), b);
}
inline void store_stream(float* p, float v) {
    int b;
    std::memcpy(&b, &v, 4);
    _mm_stream_si32(reinterpret_cast<int*>(p), b);
}

// Writes rows x cols Gaussians; element e (row-major index) goes to out[(e / cols) * ldo + e % cols]
// converted to OutT (fp32 rounds the fp64 value). Identical output for any thread count.
// streaming != 0: non-temporal stores, and the padding columns [cols, ldo) of every row are zeroed
// (the buffer is a DMA source; see store_stream).
// Only rows [r0, r1) are produced (r0·cols must be even: a row range starts on a Box–Muller pair);
// the caller can upload finished row ranges while the next one is generated.
template <typename OutT>
void gaussian_host_rows(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, OutT* out, int64_t ldo,
                        int threads, int streaming, int64_t r0, int64_t r1) {
    const int64_t total = rows * cols;
    const int64_t e_lo = r0 * cols, e_hi = std::min(total, r1 * cols);
    if (e_hi <= e_lo) return;
    const int64_t q0 = e_lo / 2, q1 = (e_hi + 1) / 2;  // pairs of this range
    const int64_t pairs = q1 - q0;
    const State s0 = seed_state(seed, stream);
    int nt = threads < 1 ? 1 : threads;
    if (pairs < 8192) nt = 1;
    if (nt > 1 || q0 > 0) jump_table();  // build once, outside the timed fan-out
    pool().run(nt, [&](int t) {
        const int64_t p0 = q0 + pairs * t / nt, p1 = q0 + pairs * (t + 1) / nt;
        State st = p0 == 0 ? s0 : jump(s0, uint64_t(2 * p0));
        int64_t e = 2 * p0, r = e / cols, c = e % cols;
        auto put = [&](double v) {
            if (streaming) {
                store_stream(out + r * ldo + c, static_cast<OutT>(v));
            } else {
                out[r * ldo + c] = static_cast<OutT>(v);
            }
            if (++c == cols) {
                if (streaming)
                    for (int64_t z = cols; z < ldo; ++z) store_stream(out + r * ldo + z, OutT(0));
                c = 0;
                ++r;
            }
        };
        for (int64_t p = p0; p < p1; ++p) {
            const double u1 = open01(next_word(st));
            const double u2 = open01(next_word(st));
            const double rad = std::sqrt(-2.0 * std::log(u1));
            const double theta = 2.0 * 3.141592653589793 * u2;  // 2·std::numbers::pi·u2
            const double sv = rad * std::sin(theta);
            put(rad * std::cos(theta));
            if (2 * p + 1 < e_hi) put(sv);
        }
        if (streaming) _mm_sfence();
    });
}

template <typename OutT>
void gaussian_host(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, OutT* out, int64_t ldo, int threads,
                   int streaming) {
    gaussian_host_rows<OutT>(rows, cols, seed, stream, out, ldo, threads, streaming, 0, rows);
}

template void gaussian_host<double>(int64_t, int64_t, uint64_t, uint64_t, double*, int64_t, int, int);
template void gaussian_host<float>(int64_t, int64_t, uint64_t, uint64_t, float*, int64_t, int, int);
template void gaussian_host_rows<double>(int64_t, int64_t, uint64_t, uint64_t, double*, int64_t, int, int, int64_t,
                                         int64_t);
template void gaussian_host_rows<float>(int64_t, int64_t, uint64_t, uint64_t, float*, int64_t, int, int, int64_t,
                                        int64_t);

}  // namespace coru_gpu
