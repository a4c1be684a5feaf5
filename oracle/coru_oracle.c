/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * CPU restatement (plain C) of the reference hot path coru::corutv
 * (/root/reference/proj/include/coru/corutv.hpp:79-100) and the functions it calls:
 *   - RNG: SplitMix64 / xoshiro256++ / Box–Muller Gaussian  (rng.hpp:13-112)
 *   - matmul i-k-j                                           (matrix.hpp:115-131)
 *   - householder_qr, qrcp, reflector helpers                (qr.hpp:32-143)
 *   - sketch_bases, corutv exact-D and approx-D                (corutv.hpp:49-100)
 *   - Jacobi SVD, pinv                                        (svd.hpp:31-187)
 *   - sor_svd, tsr_svd baselines                              (baselines.hpp:43-71)
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

/* ---- SVD / pseudo-inverse of a square matrix (svd.hpp), fp64 ---------------------------- */

/* detail::jacobi_svd_square (svd.hpp:31-134). `a` (n×n) is COLUMN-major and is overwritten
 * with the rotated columns. Outputs: u, v row-major n×n, sigma[n] non-increasing.
 * One-sided cyclic Jacobi by (j,k) row order; a pair rotates when
 * |c_j·c_k| > 1e-14·sqrt(sq_j·sq_k) (:51-57); converged after a sweep with no rotation, capped at
 * 60 sweeps (:44); columns stable-sorted by descending squared norm (:79-82); zero-sigma u
 * columns completed from the canonical basis (:98-121). Returns 1 if converged. */
int oracle_jacobi_svd_square(double* a, int64_t n, double* u, double* sigma, double* v) {
    const double kTol = 1e-14;
    const int kMaxSweeps = 60;
    double* vw = (double*)calloc((size_t)(n * n), sizeof(double));
    double* sq = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) vw[j * n + j] = 1.0;
    for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        const double* c = a + j * n;
        for (int64_t i = 0; i < n; ++i) s += c[i] * c[i];
        sq[j] = s;
    }
    int converged = 0;
    for (int sweep = 0; sweep < kMaxSweeps && !converged; ++sweep) {
        int rotated = 0;
        for (int64_t j = 0; j + 1 < n; ++j) {
            for (int64_t k = j + 1; k < n; ++k) {
                double* cj = a + j * n;
                double* ck = a + k * n;
                if (sq[j] == 0.0 || sq[k] == 0.0) continue;
                double gamma = 0.0;
                for (int64_t i = 0; i < n; ++i) gamma += cj[i] * ck[i];
                if (fabs(gamma) <= kTol * sqrt(sq[j] * sq[k])) continue;
                const double zeta = (sq[k] - sq[j]) / (2.0 * gamma);
                if (!isfinite(zeta)) continue;
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double s = c * t;
                double* vj = vw + j * n;
                double* vk = vw + k * n;
                for (int64_t i = 0; i < n; ++i) {
                    const double x = cj[i], y = ck[i];
                    cj[i] = c * x - s * y;
                    ck[i] = s * x + c * y;
                }
                for (int64_t i = 0; i < n; ++i) {
                    const double x = vj[i], y = vk[i];
                    vj[i] = c * x - s * y;
                    vk[i] = s * x + c * y;
                }
                double sj = 0.0, sk = 0.0;
                for (int64_t i = 0; i < n; ++i) {
                    sj += cj[i] * cj[i];
                    sk += ck[i] * ck[i];
                }
                sq[j] = sj;
                sq[k] = sk;
                rotated = 1;
            }
        }
        if (!rotated) converged = 1;
    }
    /* stable sort by descending sq (insertion sort keeps equal keys in index order) */
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) {
        int64_t p = j;
        while (p > 0 && sq[order[p - 1]] < sq[j]) {
            order[p] = order[p - 1];
            --p;
        }
        order[p] = j;
    }
    memset(u, 0, sizeof(double) * (size_t)(n * n));
    for (int64_t j = 0; j < n; ++j) {
        const int64_t src = order[j];
        const double sg = sqrt(sq[src]);
        sigma[j] = sg;
        for (int64_t i = 0; i < n; ++i) v[i * n + j] = vw[src * n + i];
        if (sg > 0.0)
            for (int64_t i = 0; i < n; ++i) u[i * n + j] = a[src * n + i] / sg;
    }
    /* zero-sigma completion (svd.hpp:98-121) */
    double* cand = (double*)malloc(sizeof(double) * (size_t)n);
    double* best = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) {
        if (sigma[j] > 0.0) continue;
        double best_res = -1.0;
        for (int64_t e = 0; e < n; ++e) {
            memset(cand, 0, sizeof(double) * (size_t)n);
            cand[e] = 1.0;
            for (int pass = 0; pass < 2; ++pass)
                for (int64_t c = 0; c < j; ++c) {
                    double dot = 0.0;
                    for (int64_t i = 0; i < n; ++i) dot += cand[i] * u[i * n + c];
                    for (int64_t i = 0; i < n; ++i) cand[i] -= dot * u[i * n + c];
                }
            double res = 0.0;
            for (int64_t i = 0; i < n; ++i) res += cand[i] * cand[i];
            if (res > best_res) {
                best_res = res;
                memcpy(best, cand, sizeof(double) * (size_t)n);
            }
        }
        const double nrm = sqrt(best_res);
        for (int64_t i = 0; i < n; ++i) u[i * n + j] = best[i] / nrm;
    }
    free(cand); free(best); free(order); free(vw); free(sq);
    return converged;
}

/* pinv(a) (svd.hpp:167-187) for a square n×n row-major a: svd (the square branch, :150-155),
 * singular values <= n·eps·sigma_1 dropped, then matmul(v·diag(1/sigma), u^T) in i-k-j order. */
void oracle_pinv_f64(const double* a, int64_t n, double* out) {
    double* acm = (double*)malloc(sizeof(double) * (size_t)(n * n));
    double* u = (double*)malloc(sizeof(double) * (size_t)(n * n));
    double* v = (double*)malloc(sizeof(double) * (size_t)(n * n));
    double* sg = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) acm[j * n + i] = a[i * n + j];
    oracle_jacobi_svd_square(acm, n, u, sg, v);
    const double cut = (double)n * 2.220446049250313080847e-16 * sg[0];
    for (int64_t j = 0; j < n; ++j) {
        const double inv = sg[j] > cut ? 1.0 / sg[j] : 0.0;
        for (int64_t i = 0; i < n; ++i) v[i * n + j] *= inv; /* vs(i,j) = v(i,j)·inv */
    }
    memset(out, 0, sizeof(double) * (size_t)(n * n));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = 0; k < n; ++k) {
            const double vik = v[i * n + k];
            for (int64_t j = 0; j < n; ++j) out[i * n + j] += vik * u[j * n + k]; /* u^T(k,j) */
        }
    free(acm); free(u); free(v); free(sg);
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

/* Extended precision (x87 80-bit long double, 64-bit significand): the same algorithm with a
 * unit roundoff 2^11 times smaller than fp64 — a stand-in for the exact-arithmetic result the
 * fp64 executions (the reference, its FMA build, the GPU) approximate. Used only to measure
 * which fp64 execution is closer to that result (tests/parity_util.py). */
#define T long double
#define SUFFIX f80
#define SQRT sqrtl
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

/* ---- SVD-based baselines (baselines.hpp), fp64 ------------------------------------------ */

static double* transpose_copy(const double* a, int64_t m, int64_t n) {
    double* t = (double*)malloc(sizeof(double) * (size_t)(m * n));
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) t[j * m + i] = a[i * n + j];
    return t;
}

/* svd (svd.hpp:141-161) of a square n×n row-major a: u, v row-major n×n, sigma[n]. */
int oracle_svd_square_f64(const double* a, int64_t n, double* u, double* sigma, double* v) {
    double* acm = transpose_copy(a, n, n); /* a_cm[j·n + i] = a(i, j) */
    const int conv = oracle_jacobi_svd_square(acm, n, u, sigma, v);
    free(acm);
    return conv;
}

/* tsr_svd (baselines.hpp:43-56): u m×ell, sigma[ell], v n×ell; *conv = svd(b).converged.
 * Returns 1 for the reference's invalid_argument (ell < 1 or ell >= min(m, n)). */
int oracle_tsr_svd_f64(const double* a, int64_t m, int64_t n, int64_t ell, uint64_t seed, uint64_t stream,
                       int threads, double* u, double* sigma, double* v, int* conv) {
    if (ell < 1 || ell >= (m < n ? m : n)) return 1;
    double* phi1 = (double*)malloc(sizeof(double) * (size_t)(n * ell));
    double* phi2 = (double*)malloc(sizeof(double) * (size_t)(m * ell));
    oracle_gaussian(n, ell, seed, stream, phi1);      /* substream(seed, 0) */
    oracle_gaussian(m, ell, seed, stream + 1, phi2);  /* substream(seed, 1) */
    double* y1 = (double*)malloc(sizeof(double) * (size_t)(m * ell));
    double* y2 = (double*)malloc(sizeof(double) * (size_t)(n * ell));
    mm_f64(a, m, n, phi1, ell, y1, threads);          /* matmul(a, phi1) */
    mm_tn_f64(a, m, n, phi2, ell, y2, threads);       /* matmul(a.transposed(), phi2) */
    double* q1 = (double*)malloc(sizeof(double) * (size_t)(m * ell));
    double* q2 = (double*)malloc(sizeof(double) * (size_t)(n * ell));
    oracle_householder_qr_f64(y1, m, ell, q1, NULL);
    oracle_householder_qr_f64(y2, n, ell, q2, NULL);
    double* t1 = (double*)malloc(sizeof(double) * (size_t)(ell * ell));
    double* t2 = (double*)malloc(sizeof(double) * (size_t)(ell * ell));
    double* p2 = (double*)malloc(sizeof(double) * (size_t)(ell * ell));
    double* b = (double*)malloc(sizeof(double) * (size_t)(ell * ell));
    mm_tn_f64(q1, m, ell, y1, ell, t1, threads);      /* f1.q^T · y1 */
    mm_tn_f64(q2, n, ell, phi1, ell, t2, threads);    /* f2.q^T · phi1 */
    oracle_pinv_f64(t2, ell, p2);
    mm_f64(t1, ell, ell, p2, ell, b, 1);
    double* bu = (double*)malloc(sizeof(double) * (size_t)(ell * ell));
    double* bv = (double*)malloc(sizeof(double) * (size_t)(ell * ell));
    const int c = oracle_svd_square_f64(b, ell, bu, sigma, bv);
    if (conv) *conv = c;
    mm_f64(q1, m, ell, bu, ell, u, threads);          /* matmul(f1.q, bs.u) */
    mm_f64(q2, n, ell, bv, ell, v, threads);          /* matmul(f2.q, bs.v) */
    free(phi1); free(phi2); free(y1); free(y2); free(q1); free(q2);
    free(t1); free(t2); free(p2); free(b); free(bu); free(bv);
    return 0;
}

/* sor_svd (baselines.hpp:61-71): out m×n = q1 · svd_truncate(svd(q1^T a q2), k) · q2^T.
 * Returns 1 for the reference's invalid_argument cases. */
int oracle_sor_svd_f64(const double* a, int64_t m, int64_t n, int64_t k, int64_t ell, int q, uint64_t seed,
                       uint64_t stream, int threads, double* out) {
    if (m < n) { /* sor_svd(a^T)^T (baselines.hpp:63-66) */
        double* at = transpose_copy(a, m, n);
        double* ot = (double*)malloc(sizeof(double) * (size_t)(m * n));
        const int rc = oracle_sor_svd_f64(at, n, m, k, ell, q, seed, stream, threads, ot);
        if (rc == 0)
            for (int64_t i = 0; i < n; ++i)
                for (int64_t j = 0; j < m; ++j) out[j * n + i] = ot[i * m + j];
        free(at); free(ot);
        return rc;
    }
    if (ell < 1 || ell >= n || k < 1 || k > ell || q < 0) return 1; /* :67-69 */
    double* q1 = (double*)malloc(sizeof(double) * (size_t)(m * ell));
    double* q2 = (double*)malloc(sizeof(double) * (size_t)(n * ell));
    int warn = 0;
    oracle_sketch_bases_f64(a, m, n, ell, q, seed, stream, threads, q1, q2, NULL, NULL, &warn);
    /* d = matmul(matmul(q1^T, a), q2) */
    double* q1ta = (double*)calloc((size_t)(ell * n), sizeof(double));
    for (int64_t l = 0; l < ell; ++l) {
        double* row = q1ta + l * n;
        for (int64_t i = 0; i < m; ++i) {
            const double w = q1[i * ell + l];
            const double* ai = a + i * n;
            for (int64_t j = 0; j < n; ++j) row[j] += w * ai[j];
        }
    }
    double* d = (double*)malloc(sizeof(double) * (size_t)(ell * ell));
    mm_f64(q1ta, ell, n, q2, ell, d, 1);
    double* du = (double*)malloc(sizeof(double) * (size_t)(ell * ell));
    double* dv = (double*)malloc(sizeof(double) * (size_t)(ell * ell));
    double* sg = (double*)malloc(sizeof(double) * (size_t)ell);
    oracle_svd_square_f64(d, ell, du, sg, dv);
    /* svd_truncate (baselines.hpp:14-20): us(i,j) = u(i,j)·sigma_j, j < k; matmul(us, v.left_cols(k)^T) */
    double* us = (double*)malloc(sizeof(double) * (size_t)(ell * k));
    double* vkt = (double*)malloc(sizeof(double) * (size_t)(k * ell));
    for (int64_t i = 0; i < ell; ++i)
        for (int64_t j = 0; j < k; ++j) us[i * k + j] = du[i * ell + j] * sg[j];
    for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i < ell; ++i) vkt[j * ell + i] = dv[i * ell + j];
    double* core = (double*)malloc(sizeof(double) * (size_t)(ell * ell));
    mm_f64(us, ell, k, vkt, ell, core, 1);
    double* t = (double*)malloc(sizeof(double) * (size_t)(m * ell));
    mm_f64(q1, m, ell, core, ell, t, threads);        /* matmul(sb.q1, truncated) */
    double* q2t = transpose_copy(q2, n, ell);         /* sb.q2.transposed() */
    mm_f64(t, m, ell, q2t, n, out, threads);
    free(q1); free(q2); free(q1ta); free(d); free(du); free(dv); free(sg); free(us); free(vkt);
    free(core); free(t); free(q2t);
    return 0;
}
