/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * CPU restatement (plain C) of the reference hot path coru::corutv
 * (/root/reference/proj/include/coru/corutv.hpp:79-100) and the functions it calls:
 *   - RNG: SplitMix64 / xoshiro256++ / Box–Muller Gaussian  (rng.hpp:13-112)
 *   - matmul i-k-j                                           (matrix.hpp:115-131)
 *   - householder_qr, qrcp, reflector helpers                (qr.hpp:32-143)
 *   - sketch_bases, corutv exact-D                           (corutv.hpp:49-100)
 * It is the parity checker for the CUDA path: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it (as liboracle.so via oracle/__init__.py).
 * Parity of this restatement is pinned bit-for-bit against the compiled reference
 * (oracle/_ref/libcoru_ref.so) and against the committed fixtures in tests/golden/.
 *
 * Build: oracle/Makefile (-O3 -ffp-contract=off: the reference's shipped bits need
 * uncontracted multiply-adds).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- RNG (rng.hpp) ---------------------------------------------------------------- */

/* SplitMix64::next (rng.hpp:23-35) */
static uint64_t splitmix64_next(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

typedef struct { uint64_t s[4]; } xoshiro_t;

/* Xoshiro256pp(RngSeed) (rng.hpp:41-49): state = SM(seed)_i ^ SM(stream)_i, all-zero guard */
static void xoshiro_init(xoshiro_t* r, uint64_t seed, uint64_t stream) {
    uint64_t a = seed, b = stream;
    int all_zero = 1;
    for (int i = 0; i < 4; ++i) {
        r->s[i] = splitmix64_next(&a) ^ splitmix64_next(&b);
        all_zero = all_zero && r->s[i] == 0;
    }
    if (all_zero) r->s[0] = 1;
}

/* Xoshiro256pp::next (rng.hpp:51-61) */
static uint64_t xoshiro_next(xoshiro_t* r) {
    uint64_t* s = r->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

/* uniform_open01 (rng.hpp:64): ((x >> 11) + 1)·2^-53 in (0, 1] */
static double uniform_open01(xoshiro_t* r) { return (double)((xoshiro_next(r) >> 11) + 1) * 0x1.0p-53; }

void oracle_xoshiro_words(uint64_t seed, uint64_t stream, int64_t count, uint64_t* out) {
    xoshiro_t r;
    xoshiro_init(&r, seed, stream);
    for (int64_t i = 0; i < count; ++i) out[i] = xoshiro_next(&r);
}

/* gaussian (rng.hpp:107-112) with GaussianSampler::next (rng.hpp:86-98): Box–Muller,
 * r·cos θ first, then the spare r·sin θ; row-major fill. */
void oracle_gaussian(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, double* out) {
    xoshiro_t r;
    xoshiro_init(&r, seed, stream);
    const double two_pi = 2.0 * 3.14159265358979323846; /* 2·std::numbers::pi */
    const int64_t total = rows * cols;
    int64_t i = 0;
    while (i < total) {
        const double u1 = uniform_open01(&r);
        const double u2 = uniform_open01(&r);
        const double rad = sqrt(-2.0 * log(u1));
        const double theta = two_pi * u2;
        out[i++] = rad * cos(theta);
        if (i < total) out[i++] = rad * sin(theta);
    }
}

/* ---- type-generic linear algebra ---------------------------------------------------- */

#define T double
#define SUFFIX f64
#define SQRT sqrt
#include "coru_oracle_impl.h"
#undef T
#undef SUFFIX
#undef SQRT

#define T float
#define SUFFIX f32
#define SQRT sqrtf
#include "coru_oracle_impl.h"
#undef T
#undef SUFFIX
#undef SQRT

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
