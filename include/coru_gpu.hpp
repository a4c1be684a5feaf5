// coru_gpu.hpp — header-only C++ mirror of the reference's decomposition API over the C-ABI.
//
// A C++ caller of the reference switches by replacing
//     #include "coru/corutv.hpp"      coru::corutv(a, ell, q, coru::DVariant::exact, {seed, stream})
// with
//     #include "coru_gpu.hpp"         coru_gpu::corutv(a, ell, q, coru_gpu::DVariant::exact, {seed, stream})
// Same argument list and meaning, same output record (UtvApprox, corutv.hpp:23-34), same error
// behaviour (std::invalid_argument for the reference's parameter errors, corutv.hpp:68-70,81 and
// matrix.hpp:29-31); GPU failures throw std::runtime_error. Matrix is row-major fp64 like
// coru::Matrix (matrix.hpp:17-110; construction validation is the reference's own).
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "coru_gpu.h"

namespace coru_gpu {

struct RngSeed {  // rng.hpp:13-16
    std::uint64_t seed = 0;
    std::uint64_t stream = 0;
};
inline RngSeed substream(RngSeed s, std::uint64_t offset) { return {s.seed, s.stream + offset}; }  // rng.hpp:18

enum class DVariant { exact, approx };  // corutv.hpp:17

class Matrix {  // row-major fp64, matrix.hpp:17-110 (the subset the hot path's callers use)
public:
    Matrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), data_(check(rows, cols), 0.0) {}
    Matrix(std::size_t rows, std::size_t cols, std::vector<double> entries)
        : rows_(rows), cols_(cols), data_(std::move(entries)) {
        check(rows, cols);
        if (data_.size() != rows * cols)
            throw std::invalid_argument("Matrix: entries size " + std::to_string(data_.size()) + " does not match " +
                                        std::to_string(rows) + "x" + std::to_string(cols));
        for (double x : data_)
            if (!std::isfinite(x)) throw std::invalid_argument("Matrix: non-finite entry");
    }
    std::size_t rows() const noexcept { return rows_; }
    std::size_t cols() const noexcept { return cols_; }
    std::size_t size() const noexcept { return data_.size(); }
    double operator()(std::size_t i, std::size_t j) const noexcept { return data_[i * cols_ + j]; }
    double& operator()(std::size_t i, std::size_t j) noexcept { return data_[i * cols_ + j]; }
    const std::vector<double>& data() const noexcept { return data_; }
    std::vector<double>& data() noexcept { return data_; }

private:
    static std::size_t check(std::size_t r, std::size_t c) {
        if (r == 0 || c == 0) throw std::invalid_argument("Matrix: dimensions must be positive");
        return r * c;
    }
    std::size_t rows_, cols_;
    std::vector<double> data_;
};

struct UtvApprox {  // corutv.hpp:23-34
    Matrix u, t, v;
    std::size_t ell;
    int q;
    DVariant variant;
    RngSeed seed;
    bool lower = false;
    bool conditioning_warning = false;
    std::vector<std::int64_t> perm;  // QRCP pivots of the core (extra)
};

struct SvdFactors {  // svd.hpp:17-22
    Matrix u;
    std::vector<double> sigma;
    Matrix v;
    bool converged = true;
};

struct SketchBases {  // corutv.hpp:42-47
    Matrix q1, q2, c1, c2_prev;
    bool conditioning_warning = false;
};

namespace detail {
inline void throw_status(int rc) {
    if (rc == CORU_OK) return;
    const std::string msg = coru_last_error();
    if (rc == CORU_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("coru_gpu: " + msg);
}
// One context per thread: the reference is re-entrant across threads (coru_cli.cpp:171-177).
inline coru_ctx* thread_context() {
    struct Holder {
        coru_ctx* c = nullptr;
        ~Holder() { coru_ctx_destroy(c); }
    };
    thread_local Holder h;
    if (!h.c) throw_status(coru_ctx_create(0, &h.c));
    return h.c;
}
}  // namespace detail

// coru::corutv (corutv.hpp:79-100)
inline UtvApprox corutv(const Matrix& a, std::size_t ell, int q, DVariant variant, RngSeed seed) {
    const std::int64_t m = std::int64_t(a.rows()), n = std::int64_t(a.cols()), l = std::int64_t(ell);
    if (ell < 1) throw std::invalid_argument("corutv: ell must be >= 1");
    if (ell >= std::min(a.rows(), a.cols())) throw std::invalid_argument("corutv: ell must be < min(rows, cols)");
    if (q < 0) throw std::invalid_argument("corutv: q must be >= 0");
    UtvApprox f{Matrix(a.rows(), ell), Matrix(ell, ell), Matrix(a.cols(), ell), ell, q, variant, seed,
                false, false, std::vector<std::int64_t>(ell)};
    int lower = 0, warn = 0;
    detail::throw_status(coru_corutv_f64(detail::thread_context(), a.data().data(), m, n, l, q,
                                         variant == DVariant::exact ? CORU_D_EXACT : CORU_D_APPROX, seed.seed,
                                         seed.stream, f.u.data().data(), f.t.data().data(), f.v.data().data(),
                                         f.perm.data(), &lower, &warn));
    f.lower = lower != 0;
    f.conditioning_warning = warn != 0;
    return f;
}

// Zero-copy drop-in for the caller's own row-major fp64 matrix type — coru::Matrix itself
// (matrix.hpp:17-110), or anything with rows(), cols() and contiguous data().data(): A is read
// in place (pageable storage streams through the context's pinned staging ring; it is never
// copied whole), and U, T, V are written straight into matrices of the caller's type (M(rows,
// cols) must zero-construct, as coru::Matrix does). Same argument list and errors as
// coru::corutv (corutv.hpp:79-100).
template <class M>
struct UtvApproxOf {  // corutv.hpp:23-34 with the caller's matrix type
    M u, t, v;
    std::size_t ell;
    int q;
    DVariant variant;
    RngSeed seed;
    bool lower = false;
    bool conditioning_warning = false;
    std::vector<std::int64_t> perm;
};

template <class M, class = std::enable_if_t<!std::is_same<M, Matrix>::value>,
          class = decltype(std::declval<const M&>().data().data())>
inline UtvApproxOf<M> corutv(const M& a, std::size_t ell, int q, DVariant variant, RngSeed seed) {
    if (ell < 1) throw std::invalid_argument("corutv: ell must be >= 1");
    if (ell >= std::min(a.rows(), a.cols())) throw std::invalid_argument("corutv: ell must be < min(rows, cols)");
    if (q < 0) throw std::invalid_argument("corutv: q must be >= 0");
    UtvApproxOf<M> f{M(a.rows(), ell), M(ell, ell), M(a.cols(), ell), ell, q, variant, seed,
                     false, false, std::vector<std::int64_t>(ell)};
    int lower = 0, warn = 0;
    detail::throw_status(coru_corutv_f64(detail::thread_context(), a.data().data(), std::int64_t(a.rows()),
                                         std::int64_t(a.cols()), std::int64_t(ell), q,
                                         variant == DVariant::exact ? CORU_D_EXACT : CORU_D_APPROX, seed.seed,
                                         seed.stream, f.u.data().data(), f.t.data().data(), f.v.data().data(),
                                         f.perm.data(), &lower, &warn));
    f.lower = lower != 0;
    f.conditioning_warning = warn != 0;
    return f;
}

// detail::sketch_bases (corutv.hpp:49-65)
inline SketchBases sketch_bases(const Matrix& a, std::size_t ell, int q, RngSeed seed) {
    SketchBases s{Matrix(a.rows(), ell), Matrix(a.cols(), ell), Matrix(a.rows(), ell), Matrix(a.cols(), ell), false};
    int warn = 0;
    detail::throw_status(coru_sketch_bases_f64(detail::thread_context(), a.data().data(), std::int64_t(a.rows()),
                                               std::int64_t(a.cols()), std::int64_t(ell), q, seed.seed, seed.stream,
                                               s.q1.data().data(), s.q2.data().data(), s.c1.data().data(),
                                               s.c2_prev.data().data(), &warn));
    s.conditioning_warning = warn != 0;
    return s;
}

// gaussian (rng.hpp:107-112): bit-exact host generator.
inline Matrix gaussian(std::size_t rows, std::size_t cols, RngSeed seed) {
    Matrix m(rows, cols);
    detail::throw_status(coru_gaussian(std::int64_t(rows), std::int64_t(cols), seed.seed, seed.stream,
                                       m.data().data(), 1));
    return m;
}

// tsr_svd (baselines.hpp:43-56)
inline SvdFactors tsr_svd(const Matrix& a, std::size_t ell, RngSeed seed) {
    SvdFactors f{Matrix(a.rows(), ell), std::vector<double>(ell), Matrix(a.cols(), ell), true};
    int conv = 0;
    detail::throw_status(coru_tsr_svd_f64(detail::thread_context(), a.data().data(), std::int64_t(a.rows()),
                                          std::int64_t(a.cols()), std::int64_t(ell), seed.seed, seed.stream,
                                          f.u.data().data(), f.sigma.data(), f.v.data().data(), &conv));
    f.converged = conv != 0;
    return f;
}

// sor_svd (baselines.hpp:61-71)
inline Matrix sor_svd(const Matrix& a, std::size_t k, std::size_t ell, int q, RngSeed seed) {
    Matrix out(a.rows(), a.cols());
    detail::throw_status(coru_sor_svd_f64(detail::thread_context(), a.data().data(), std::int64_t(a.rows()),
                                          std::int64_t(a.cols()), std::int64_t(k), std::int64_t(ell), q, seed.seed,
                                          seed.stream, out.data().data()));
    return out;
}

// RpcaInner / CorutvThresholding / RpcaConfig / RpcaResult (rpca.hpp:53-88). inner defaults to corutv,
// the inner step this build provides (svt_exact throws std::runtime_error, CORU_ENOTSUP).
enum class RpcaInner { svt_exact, corutv };
enum class CorutvThresholding { soft, hard };
struct RpcaConfig {
    double lambda = 0.0;
    double mu0 = 0.0;
    double rho = 1.5;
    double mu_bar = 0.0;
    double tol = 1e-5;
    int max_iter = 50;
    RpcaInner inner = RpcaInner::corutv;
    std::size_t corutv_ell = 0;
    int corutv_q = 1;
    CorutvThresholding corutv_thresholding = CorutvThresholding::soft;
};
struct RpcaResult {
    Matrix l, s;
    int iterations;
    std::vector<double> residuals;
    std::size_t rank_l;
    std::size_t s_l0;
    bool converged;
    bool ell_clamped;
};

// alm_rpca (rpca.hpp:95-169) with the CoR-UTV inner step on the GPU.
inline RpcaResult alm_rpca(const Matrix& m, const RpcaConfig& config, RngSeed seed) {
    coru_rpca_config c;
    c.lambda = config.lambda;
    c.mu0 = config.mu0;
    c.rho = config.rho;
    c.mu_bar = config.mu_bar;
    c.tol = config.tol;
    c.max_iter = config.max_iter;
    c.inner = config.inner == RpcaInner::corutv ? CORU_RPCA_CORUTV : CORU_RPCA_SVT_EXACT;
    c.corutv_ell = std::int64_t(config.corutv_ell);
    c.corutv_q = config.corutv_q;
    c.thresholding = config.corutv_thresholding == CorutvThresholding::hard ? CORU_COR_HARD : CORU_COR_SOFT;
    RpcaResult r{Matrix(m.rows(), m.cols()), Matrix(m.rows(), m.cols()), 0, {}, 0, 0, false, false};
    r.residuals.assign(std::size_t(std::max(config.max_iter, 1)), 0.0);
    coru_rpca_result res{};
    res.residuals = r.residuals.data();
    detail::throw_status(coru_alm_rpca_f64(detail::thread_context(), m.data().data(), std::int64_t(m.rows()),
                                           std::int64_t(m.cols()), &c, seed.seed, seed.stream, r.l.data().data(),
                                           r.s.data().data(), &res));
    r.iterations = res.iterations;
    r.residuals.resize(std::size_t(res.iterations));
    r.rank_l = std::size_t(res.rank_l);
    r.s_l0 = std::size_t(res.s_l0);
    r.converged = res.converged != 0;
    r.ell_clamped = res.ell_clamped != 0;
    return r;
}

// Out-of-core corutv (§8 f4): A streamed from host memory in row chunks; the same
// UtvApprox as corutv. chunk_rows = 0: ~512 MB chunks.
inline UtvApprox corutv_streamed(const Matrix& a, std::size_t ell, int q, DVariant variant, RngSeed seed,
                                 std::int64_t chunk_rows = 0) {
    if (ell < 1) throw std::invalid_argument("corutv: ell must be >= 1");
    if (ell >= std::min(a.rows(), a.cols())) throw std::invalid_argument("corutv: ell must be < min(rows, cols)");
    if (q < 0) throw std::invalid_argument("corutv: q must be >= 0");
    UtvApprox f{Matrix(a.rows(), ell), Matrix(ell, ell), Matrix(a.cols(), ell), ell, q, variant, seed,
                false, false, std::vector<std::int64_t>(ell)};
    const std::int64_t l = std::int64_t(ell);
    coru_utv out{f.u.data().data(), l, f.t.data().data(), l, f.v.data().data(), l, f.perm.data(), 0, 0};
    detail::throw_status(coru_corutv_f64_ooc(detail::thread_context(), a.data().data(), std::int64_t(a.rows()),
                                             std::int64_t(a.cols()), std::int64_t(a.cols()), l, q,
                                             variant == DVariant::exact ? CORU_D_EXACT : CORU_D_APPROX, seed.seed,
                                             seed.stream, chunk_rows, &out));
    f.conditioning_warning = out.conditioning_warning != 0;
    f.lower = out.lower != 0;
    return f;
}

// corutv(read_matrix_bin(path), ...) without materialising the matrix (io.hpp:79-95 + corutv.hpp:79).
inline UtvApprox corutv_file(const std::string& path, std::size_t ell, int q, DVariant variant, RngSeed seed,
                             std::int64_t chunk_rows = 0) {
    std::int64_t m = 0, n = 0;
    detail::throw_status(coru_read_matrix_bin_header(path.c_str(), &m, &n));
    UtvApprox f{Matrix(std::size_t(m), ell), Matrix(ell, ell), Matrix(std::size_t(n), ell), ell, q, variant, seed,
                false, false, std::vector<std::int64_t>(ell)};
    const std::int64_t l = std::int64_t(ell);
    coru_utv out{f.u.data().data(), l, f.t.data().data(), l, f.v.data().data(), l, f.perm.data(), 0, 0};
    detail::throw_status(coru_corutv_f64_file(detail::thread_context(), path.c_str(), l, q,
                                              variant == DVariant::exact ? CORU_D_EXACT : CORU_D_APPROX, seed.seed,
                                              seed.stream, chunk_rows, &out));
    f.conditioning_warning = out.conditioning_warning != 0;
    f.lower = out.lower != 0;
    return f;
}

// singular_estimates (corutv.hpp:113-117)
inline std::vector<double> singular_estimates(const UtvApprox& f) {
    std::vector<double> s(f.ell);
    for (std::size_t j = 0; j < f.ell; ++j) s[j] = std::abs(f.t(j, j));
    return s;
}

}  // namespace coru_gpu
