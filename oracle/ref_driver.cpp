// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C-ABI driver around the *unmodified* reference implementation. It #includes the
// reference headers in place (-I/root/reference/proj/include; nothing is copied into
// this repo) and is built by oracle/Makefile into oracle/_ref/libcoru_ref.so, which is
// git-ignored and travels to the GPU box prebuilt. Only tests/, __graft_entry__.smoke()
// and bench.py (cpu_baseline leg and --impl reference) may load it.
//
// Every matrix crossing this boundary is dense row-major fp64, the layout of
// coru::Matrix (proj/include/coru/matrix.hpp:44-45).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

#include "coru/baselines.hpp"
#include "coru/corutv.hpp"
#include "coru/norms.hpp"
#include "coru/rpca.hpp"
#include "coru/io.hpp"
#include "coru/testgen.hpp"

using coru::Matrix;

namespace {

thread_local std::string g_err;

Matrix wrap(const double* a, int64_t m, int64_t n) {
    // The validating constructor (matrix.hpp:22-32): rejects non-finite entries like the reference.
    return Matrix(size_t(m), size_t(n), std::vector<double>(a, a + m * n));
}

void put(const Matrix& x, double* out) {
    if (out) std::memcpy(out, x.data().data(), x.size() * sizeof(double));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

// Row-parallel i-k-j product. matmul's i loop carries no dependency
// (matrix.hpp:121-129), so splitting it over threads leaves every output bit unchanged. Four rows
// share each b(k,.) load; every entry still sums over k increasing.
Matrix matmul_rows(const Matrix& a, const Matrix& b, int threads) {
    if (threads <= 1) return coru::matmul(a, b);
    Matrix c(a.rows(), b.cols());
    const size_t n = b.cols(), kk = a.cols(), m = a.rows();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
            const size_t lo = m * t / threads, hi = m * (t + 1) / threads;
            size_t i = lo;
            for (; i + 4 <= hi; i += 4) {
                double *c0 = c.row(i), *c1 = c.row(i + 1), *c2 = c.row(i + 2), *c3 = c.row(i + 3);
                const double *a0 = a.row(i), *a1 = a.row(i + 1), *a2 = a.row(i + 2), *a3 = a.row(i + 3);
                for (size_t k = 0; k < kk; ++k) {
                    const double x0 = a0[k], x1 = a1[k], x2 = a2[k], x3 = a3[k];
                    const double* bk = b.row(k);
                    for (size_t j = 0; j < n; ++j) {
                        const double bj = bk[j];
                        c0[j] += x0 * bj;
                        c1[j] += x1 * bj;
                        c2[j] += x2 * bj;
                        c3[j] += x3 * bj;
                    }
                }
            }
            for (; i < hi; ++i) {
                double* ci = c.row(i);
                const double* ai = a.row(i);
                for (size_t k = 0; k < kk; ++k) {
                    const double aik = ai[k];
                    const double* bk = b.row(k);
                    for (size_t j = 0; j < n; ++j) ci[j] += aik * bk[j];
                }
            }
        });
    }
    for (auto& th : pool) th.join();
    return c;
}

Matrix transposed_rows(const Matrix& a, int threads) {
    if (threads <= 1) return a.transposed();
    Matrix t(a.cols(), a.rows());
    std::vector<std::thread> pool;
    const size_t rows = a.cols();
    for (int th = 0; th < threads; ++th)
        pool.emplace_back([&, th] {
            for (size_t j = rows * th / threads; j < rows * (th + 1) / threads; ++j)
                for (size_t i = 0; i < a.rows(); ++i) t(j, i) = a(i, j);
        });
    for (auto& th : pool) th.join();
    return t;
}

// matmul(a.transposed(), y) without forming a^T (corutv.hpp:50,57): out row i of a^T·y sums
// a(k,i)·y(k,.) over k increasing, exactly coru::matmul's i-k-j order on the transpose. Threads
// own ranges of output rows and sweep the rows k of a together, so a and y are streamed once per
// thread instead of once per output row; every output entry keeps its summation order.
Matrix matmul_tn_cols(const Matrix& a, const Matrix& y, int threads) {
    const size_t m = a.rows(), n = a.cols(), d = y.cols();
    Matrix c(n, d);
    std::vector<std::thread> pool;
    const int nt = std::max(1, threads);
    for (int th = 0; th < nt; ++th)
        pool.emplace_back([&, th] {
            const size_t i0 = n * th / nt, i1 = n * (th + 1) / nt;
            size_t k = 0;
            for (; k + 4 <= m; k += 4) {  // four rows of a folded in sequence per accumulator load
                const double *a0 = a.row(k), *a1 = a.row(k + 1), *a2 = a.row(k + 2), *a3 = a.row(k + 3);
                const double *y0 = y.row(k), *y1 = y.row(k + 1), *y2 = y.row(k + 2), *y3 = y.row(k + 3);
                for (size_t i = i0; i < i1; ++i) {
                    const double x0 = a0[i], x1 = a1[i], x2 = a2[i], x3 = a3[i];
                    double* ci = c.row(i);
                    for (size_t j = 0; j < d; ++j) {
                        double s = ci[j];
                        s += x0 * y0[j];
                        s += x1 * y1[j];
                        s += x2 * y2[j];
                        s += x3 * y3[j];
                        ci[j] = s;
                    }
                }
            }
            for (; k < m; ++k) {
                const double* ak = a.row(k);
                const double* yk = y.row(k);
                for (size_t i = i0; i < i1; ++i) {
                    const double aki = ak[i];
                    double* ci = c.row(i);
                    for (size_t j = 0; j < d; ++j) ci[j] += aki * yk[j];
                }
            }
        });
    for (auto& t : pool) t.join();
    return c;
}

// matmul(q.transposed(), a) (corutv.hpp:90's inner product): out row l sums q(k,l)·a(k,.) over k
// increasing. Threads own column ranges of the output and sweep k, so a is read once in total.
Matrix matmul_qt_a(const Matrix& q, const Matrix& a, int threads) {
    const size_t m = a.rows(), n = a.cols(), d = q.cols();
    Matrix c(d, n);
    std::vector<std::thread> pool;
    const int nt = std::max(1, threads);
    for (int th = 0; th < nt; ++th)
        pool.emplace_back([&, th] {
            const size_t j0 = n * th / nt, j1 = n * (th + 1) / nt;
            size_t k = 0;
            for (; k + 4 <= m; k += 4) {
                const double *a0 = a.row(k), *a1 = a.row(k + 1), *a2 = a.row(k + 2), *a3 = a.row(k + 3);
                const double *q0 = q.row(k), *q1 = q.row(k + 1), *q2 = q.row(k + 2), *q3 = q.row(k + 3);
                for (size_t l = 0; l < d; ++l) {
                    const double w0 = q0[l], w1 = q1[l], w2 = q2[l], w3 = q3[l];
                    double* cl = c.row(l);
                    for (size_t j = j0; j < j1; ++j) {
                        double s = cl[j];
                        s += w0 * a0[j];
                        s += w1 * a1[j];
                        s += w2 * a2[j];
                        s += w3 * a3[j];
                        cl[j] = s;
                    }
                }
            }
            for (; k < m; ++k) {
                const double* ak = a.row(k);
                const double* qk = q.row(k);
                for (size_t l = 0; l < d; ++l) {
                    const double w = qk[l];
                    double* cl = c.row(l);
                    for (size_t j = j0; j < j1; ++j) cl[j] += w * ak[j];
                }
            }
        });
    for (auto& t : pool) t.join();
    return c;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// coru::gaussian (rng.hpp:107-112)
int ref_gaussian(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, double* out) {
    return guarded([&] { put(coru::gaussian(size_t(rows), size_t(cols), {seed, stream}), out); });
}

// Raw xoshiro256++ words (rng.hpp:39-61), for pinning the host RNG restatement.
int ref_xoshiro_words(uint64_t seed, uint64_t stream, int64_t count, uint64_t* out) {
    coru::Xoshiro256pp r({seed, stream});
    for (int64_t i = 0; i < count; ++i) out[i] = r.next();
    return 0;
}

// coru::matmul (matrix.hpp:115-131)
int ref_matmul(const double* a, int64_t m, int64_t k, const double* b, int64_t n, double* out) {
    return guarded([&] { put(coru::matmul(wrap(a, m, k), wrap(b, k, n)), out); });
}

// coru::householder_qr (qr.hpp:85-99): q m×n, r n×n
int ref_householder_qr(const double* a, int64_t m, int64_t n, double* q, double* r) {
    return guarded([&] {
        coru::QrFactors f = coru::householder_qr(wrap(a, m, n));
        put(f.q, q);
        put(f.r, r);
    });
}

// coru::qrcp (qr.hpp:106-143): q m×n, r n×n, perm n
int ref_qrcp(const double* a, int64_t m, int64_t n, double* q, double* r, int64_t* perm) {
    return guarded([&] {
        coru::QrcpFactors f = coru::qrcp(wrap(a, m, n));
        put(f.q, q);
        put(f.r, r);
        for (int64_t j = 0; j < n; ++j) perm[j] = int64_t(f.perm[size_t(j)]);
    });
}

// coru::svd (svd.hpp:141-161): u m×r, sigma[r], v n×r with r = min(m, n); returns converged in *conv.
int ref_svd(const double* a, int64_t m, int64_t n, double* u, double* sigma, double* v, int* conv) {
    return guarded([&] {
        coru::SvdFactors f = coru::svd(wrap(a, m, n));
        put(f.u, u);
        put(f.v, v);
        for (size_t j = 0; j < f.sigma.size(); ++j) sigma[j] = f.sigma[j];
        *conv = f.converged ? 1 : 0;
    });
}

// coru::pinv(a) (svd.hpp:184-187): n×m.
int ref_pinv(const double* a, int64_t m, int64_t n, double* out) {
    return guarded([&] { put(coru::pinv(wrap(a, m, n)), out); });
}

// coru::tsr_svd (baselines.hpp:43-56): u m×ell, sigma[ell], v n×ell, *conv.
int ref_tsr_svd(const double* a, int64_t m, int64_t n, int64_t ell, uint64_t seed, uint64_t stream, double* u,
                double* sigma, double* v, int* conv) {
    return guarded([&] {
        if (ell < 0) throw std::invalid_argument("tsr_svd: ell out of range");
        coru::SvdFactors f = coru::tsr_svd(wrap(a, m, n), size_t(ell), {seed, stream});
        put(f.u, u);
        put(f.v, v);
        for (size_t j = 0; j < f.sigma.size(); ++j) sigma[j] = f.sigma[j];
        *conv = f.converged ? 1 : 0;
    });
}

// coru::sor_svd (baselines.hpp:61-71): out m×n.
int ref_sor_svd(const double* a, int64_t m, int64_t n, int64_t k, int64_t ell, int q, uint64_t seed, uint64_t stream,
                double* out) {
    return guarded([&] {
        if (ell < 0 || k < 0) throw std::invalid_argument("sor_svd: bad parameters");
        put(coru::sor_svd(wrap(a, m, n), size_t(k), size_t(ell), q, {seed, stream}), out);
    });
}

// coru::corutv (corutv.hpp:79-100). u rows(a)×ell, t ell×ell, v cols(a)×ell.
// flags[0] = lower, flags[1] = conditioning_warning.
int ref_corutv(const double* a, int64_t m, int64_t n, int64_t ell, int q, int variant,
               uint64_t seed, uint64_t stream, double* u, double* t, double* v, int* flags) {
    return guarded([&] {
        if (ell < 0) throw std::invalid_argument("corutv: ell must be >= 1");
        coru::UtvApprox f = coru::corutv(wrap(a, m, n), size_t(ell), q,
                                         variant == 0 ? coru::DVariant::exact : coru::DVariant::approx,
                                         {seed, stream});
        put(f.u, u);
        put(f.t, t);
        put(f.v, v);
        flags[0] = f.lower;
        flags[1] = f.conditioning_warning;
    });
}

// Same steps as coru::corutv's exact-D, m >= n branch (corutv.hpp:49-65, 89-97), with the
// A-products spread over `threads` threads in the reference's per-entry summation order (A^T is
// never formed; the Q1^T·A product keeps matmul(q1.transposed(), a)'s order): bit-identical to
// ref_corutv. QR, QRCP and the Gaussian are the reference's own serial functions.
int ref_corutv_mt(const double* a_, int64_t m, int64_t n, int64_t ell, int q, uint64_t seed,
                  uint64_t stream, int threads, double* u, double* t, double* v, int* flags) {
    return guarded([&] {
        const Matrix a = wrap(a_, m, n);
        coru::detail::check_corutv_params(a, size_t(ell));
        if (q < 0) throw std::invalid_argument("corutv: q must be >= 0");
        if (m < n) throw std::invalid_argument("ref_corutv_mt: m >= n only");
        Matrix c2 = coru::gaussian(a.cols(), size_t(ell), {seed, stream});
        Matrix c1(a.rows(), size_t(ell));
        for (int i = 0; i <= q; ++i) {
            c1 = matmul_rows(a, c2, threads);
            c2 = matmul_tn_cols(a, c1, threads);  // = matmul(a.transposed(), c1), same bits
        }
        coru::QrFactors f1 = coru::householder_qr(c1);
        coru::QrFactors f2 = coru::householder_qr(c2);
        const bool warn = std::abs(f1.r(size_t(ell) - 1, size_t(ell) - 1)) <= 1e-14 * std::abs(f1.r(0, 0));
        // D = (Q1^T A) Q2 (corutv.hpp:90)
        const Matrix d = coru::matmul(matmul_qt_a(f1.q, a, threads), f2.q);
        coru::QrcpFactors cp = coru::qrcp(d);
        put(matmul_rows(f1.q, cp.q, threads), u);
        put(cp.r, t);
        Matrix vv(a.cols(), size_t(ell));
        for (size_t j = 0; j < size_t(ell); ++j)
            for (size_t i = 0; i < a.cols(); ++i) vv(i, j) = f2.q(i, cp.perm[j]);
        put(vv, v);
        flags[0] = 0;
        flags[1] = warn;
    });
}

// `count` independent coru::corutv calls (seeds {seed, stream0 + i}) fanned out over `threads`
// std::threads — the reference's own concurrency model, trial-level fan-out of unchanged
// decompositions (parallel.hpp:23-36, used at coru_cli.cpp:171-177). A is shared read-only
// (Matrix is safe to share, matrix.hpp:14-15). Returns sum_i sum_j |t_jj| as a checksum.
double ref_corutv_batch(const double* a_, int64_t m, int64_t n, int64_t ell, int q, uint64_t seed,
                        uint64_t stream0, int count, int threads) {
    const Matrix a = wrap(a_, m, n);
    std::vector<double> sums(size_t(count), 0.0);
    std::atomic<int> next{0};
    auto worker = [&] {
        for (int i; (i = next.fetch_add(1)) < count;) {
            coru::UtvApprox f = coru::corutv(a, size_t(ell), q, coru::DVariant::exact, {seed, stream0 + uint64_t(i)});
            double s = 0;
            for (double e : coru::singular_estimates(f)) s += e;
            sums[size_t(i)] = s;
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    double tot = 0;
    for (double s : sums) tot += s;
    return tot;
}

// coru::detail::sketch_bases (corutv.hpp:49-65)
int ref_sketch_bases(const double* a, int64_t m, int64_t n, int64_t ell, int q, uint64_t seed,
                     uint64_t stream, double* q1, double* q2, double* c1, double* c2_prev, int* warn) {
    return guarded([&] {
        coru::detail::SketchBases sb = coru::detail::sketch_bases(wrap(a, m, n), size_t(ell), q, {seed, stream});
        put(sb.q1, q1);
        put(sb.q2, q2);
        put(sb.c1, c1);
        put(sb.c2_prev, c2_prev);
        *warn = sb.conditioning_warning;
    });
}

// Test-matrix generators of the reference suite (testgen.hpp:48-81).
int ref_gen_fast_decay(int64_t n, int64_t k, uint64_t seed, uint64_t stream, double* out) {
    return guarded([&] { put(coru::gen_fast_decay(size_t(n), size_t(k), {seed, stream}), out); });
}
int ref_gen_noisy_lowrank(int64_t n, int64_t k, double gap, uint64_t seed, uint64_t stream, double* out) {
    return guarded([&] { put(coru::gen_noisy_lowrank(size_t(n), size_t(k), gap, {seed, stream}), out); });
}

// coru::frobenius_norm (matrix.hpp:133-137)
double ref_frobenius(const double* a, int64_t m, int64_t n) { return coru::frobenius_norm(wrap(a, m, n)); }

// coru::alm_rpca (rpca.hpp:95-169). cfg: {lambda, mu0, rho, mu_bar, tol}; icfg: {max_iter, inner,
// corutv_ell, corutv_q, thresholding}. out_i: {iterations, rank_l, s_l0, converged, ell_clamped}.
int ref_alm_rpca(const double* m_, int64_t m, int64_t n, const double* cfg, const int64_t* icfg, uint64_t seed,
                 uint64_t stream, double* l, double* s, double* residuals, int64_t* out_i) {
    return guarded([&] {
        coru::RpcaConfig c;
        c.lambda = cfg[0];
        c.mu0 = cfg[1];
        c.rho = cfg[2];
        c.mu_bar = cfg[3];
        c.tol = cfg[4];
        c.max_iter = int(icfg[0]);
        c.inner = icfg[1] ? coru::RpcaInner::corutv : coru::RpcaInner::svt_exact;
        c.corutv_ell = size_t(icfg[2]);
        c.corutv_q = int(icfg[3]);
        c.corutv_thresholding = icfg[4] ? coru::CorutvThresholding::hard : coru::CorutvThresholding::soft;
        coru::RpcaResult r = coru::alm_rpca(wrap(m_, m, n), c, {seed, stream});
        put(r.l, l);
        put(r.s, s);
        for (size_t i = 0; i < r.residuals.size(); ++i) residuals[i] = r.residuals[i];
        out_i[0] = r.iterations;
        out_i[1] = int64_t(r.rank_l);
        out_i[2] = int64_t(r.s_l0);
        out_i[3] = r.converged;
        out_i[4] = r.ell_clamped;
    });
}

// coru::gen_rpca_instance (testgen.hpp:86-109): m, l_true, s_true (n x n).
int ref_gen_rpca_instance(int64_t n, int64_t r, uint64_t s, double amp, uint64_t seed, uint64_t stream, double* m,
                          double* l, double* sp) {
    return guarded([&] {
        coru::RpcaInstance inst = coru::gen_rpca_instance(size_t(n), size_t(r), s, amp, {seed, stream});
        put(inst.m, m);
        put(inst.l_true, l);
        put(inst.s_true, sp);
    });
}

// coru::spectral_norm (norms.hpp:27)
double ref_spectral_norm(const double* a, int64_t m, int64_t n) { return coru::spectral_norm(wrap(a, m, n)); }

// coru::write_matrix_bin / read_matrix_bin (io.hpp:67-95). Reader: rows/cols out, data (may be NULL).
int ref_write_matrix_bin(const char* path, const double* a, int64_t m, int64_t n) {
    return guarded([&] { coru::write_matrix_bin(path, wrap(a, m, n)); });
}
int ref_read_matrix_bin(const char* path, int64_t* m, int64_t* n, double* out) {
    return guarded([&] {
        Matrix x = coru::read_matrix_bin(path);
        *m = int64_t(x.rows());
        *n = int64_t(x.cols());
        put(x, out);
    });
}

}  // extern "C"
