// C++ caller of the drop-in header (include/coru_gpu.hpp), written the way a reference caller
// uses coru::corutv (proj/tests/test_corutv.cpp:31-55, 98-108). Exit 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "coru_gpu.hpp"

using namespace coru_gpu;

static int failures = 0;
#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                            \
        }                                                          \
    } while (0)

static double orth_res(const Matrix& q) {
    double s = 0;
    for (std::size_t i = 0; i < q.cols(); ++i)
        for (std::size_t j = 0; j < q.cols(); ++j) {
            double g = 0;
            for (std::size_t r = 0; r < q.rows(); ++r) g += q(r, i) * q(r, j);
            g -= (i == j);
            s += g * g;
        }
    return std::sqrt(s);
}

static Matrix exact_rank(std::size_t m, std::size_t n, std::size_t r, RngSeed seed) {
    Matrix g1 = gaussian(m, r, substream(seed, 0)), g2 = gaussian(n, r, substream(seed, 1)), a(m, n);
    for (std::size_t i = 0; i < m; ++i)
        for (std::size_t j = 0; j < n; ++j)
            for (std::size_t k = 0; k < r; ++k) a(i, j) += g1(i, k) * g2(j, k);
    return a;
}

static double recon_err(const Matrix& a, const UtvApprox& f) {
    double e = 0, na = 0;
    for (std::size_t i = 0; i < a.rows(); ++i)
        for (std::size_t j = 0; j < a.cols(); ++j) {
            double s = 0;
            for (std::size_t p = 0; p < f.ell; ++p)
                for (std::size_t q = 0; q < f.ell; ++q) s += f.u(i, p) * f.t(p, q) * f.v(j, q);
            e += (a(i, j) - s) * (a(i, j) - s);
            na += a(i, j) * a(i, j);
        }
    return std::sqrt(e / na);
}

int main() {
    // bad parameters -> std::invalid_argument (test_corutv.cpp:31-36)
    const Matrix g = gaussian(10, 8, {1, 0});
    for (auto [ell, q] : {std::pair<std::size_t, int>{0, 0}, {8, 0}, {3, -1}}) {
        bool threw = false;
        try {
            corutv(g, ell, q, DVariant::exact, {1, 0});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    // exact rank-5 recovery (test_corutv.cpp:38-42)
    const Matrix a = exact_rank(30, 20, 5, {3, 0});
    UtvApprox f = corutv(a, 5, 0, DVariant::exact, {4, 0});
    CHECK(recon_err(a, f) <= 1e-8);
    CHECK(!f.lower);
    CHECK(orth_res(f.u) <= 1e-12 * 5 && orth_res(f.v) <= 1e-12 * 5);
    for (std::size_t i = 0; i < 5; ++i)
        for (std::size_t j = 0; j < i; ++j) CHECK(f.t(i, j) == 0.0);
    const auto est = singular_estimates(f);
    for (std::size_t j = 0; j + 1 < est.size(); ++j) CHECK(est[j] >= est[j + 1]);
    // wide input -> ULV (test_corutv.cpp:98-108)
    const Matrix w = exact_rank(20, 35, 4, {11, 0});
    UtvApprox fw = corutv(w, 8, 1, DVariant::exact, {12, 0});
    CHECK(fw.lower);
    CHECK(fw.u.rows() == 20 && fw.v.rows() == 35);
    for (std::size_t i = 0; i < 8; ++i)
        for (std::size_t j = i + 1; j < 8; ++j) CHECK(fw.t(i, j) == 0.0);
    CHECK(recon_err(w, fw) <= 1e-8);
    // sketch stage (test_corutv.cpp:57-65 uses it directly)
    SketchBases sb = sketch_bases(a, 5, 1, {4, 0});
    CHECK(orth_res(sb.q1) <= 1e-12 * 5 && orth_res(sb.q2) <= 1e-12 * 5);
    // approx-D agrees with exact-D on an exact-rank matrix (test_corutv.cpp:87-96)
    const Matrix er = exact_rank(40, 30, 6, {9, 0});
    for (int q : {0, 2}) {
        UtvApprox e = corutv(er, 10, q, DVariant::exact, {10, 0});
        UtvApprox p = corutv(er, 10, q, DVariant::approx, {10, 0});
        CHECK(p.variant == DVariant::approx);
        double diff = 0, nrm = 0;
        for (std::size_t i = 0; i < 40; ++i)
            for (std::size_t j = 0; j < 30; ++j) {
                double se = 0, sp = 0;
                for (std::size_t k = 0; k < 10; ++k)
                    for (std::size_t l = k; l < 10; ++l) {
                        se += e.u(i, k) * e.t(k, l) * e.v(j, l);
                        sp += p.u(i, k) * p.t(k, l) * p.v(j, l);
                    }
                diff += (se - sp) * (se - sp);
                nrm += er(i, j) * er(i, j);
            }
        CHECK(std::sqrt(diff) <= 1e-6 * std::sqrt(nrm));
    }
    // baselines (test_baselines.cpp:99-112): sor_svd recovers exact rank-k input; bad k throws
    {
        const Matrix e5 = exact_rank(25, 18, 5, {22, 0});
        const Matrix s5 = sor_svd(e5, 5, 8, 0, {23, 0});
        double diff = 0, nrm = 0;
        for (std::size_t i = 0; i < e5.data().size(); ++i) {
            diff += (e5.data()[i] - s5.data()[i]) * (e5.data()[i] - s5.data()[i]);
            nrm += e5.data()[i] * e5.data()[i];
        }
        CHECK(std::sqrt(diff) <= 1e-8 * std::sqrt(nrm));
        bool threw = false;
        try {
            (void)sor_svd(e5, 9, 8, 0, {23, 0});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        SvdFactors t = tsr_svd(e5, 6, {20, 3});
        CHECK(orth_res(t.u) <= 1e-9 * std::sqrt(6.0) && orth_res(t.v) <= 1e-9 * std::sqrt(6.0));
        for (std::size_t j = 0; j + 1 < t.sigma.size(); ++j) CHECK(t.sigma[j] >= t.sigma[j + 1]);
    }
    // alm_rpca with the CoR-UTV inner (rpca.hpp:95-169): low rank + sparse recovery, config validation
    {
        const std::size_t n = 60, r = 3;
        Matrix low = exact_rank(n, n, r, {31, 0});
        Matrix mat = low;
        for (std::size_t k = 0; k < 120; ++k) mat.data()[(k * 2654435761ull + k * k * 31) % (n * n)] += (k % 2 ? 50.0 : -50.0);
        RpcaConfig cfg;
        cfg.corutv_ell = 2 * r;
        RpcaResult res = alm_rpca(mat, cfg, {2, 0});
        CHECK(res.converged && res.rank_l == r && res.residuals.size() == std::size_t(res.iterations));
        double diff = 0, nrm = 0;
        for (std::size_t i = 0; i < low.data().size(); ++i) {
            diff += (low.data()[i] - res.l.data()[i]) * (low.data()[i] - res.l.data()[i]);
            nrm += low.data()[i] * low.data()[i];
        }
        CHECK(std::sqrt(diff) <= 1e-3 * std::sqrt(nrm));
        CHECK(res.s_l0 >= 100);  // 111 distinct corrupted entries
        bool threw = false;
        try {
            RpcaConfig bad = cfg;
            bad.rho = 1.0;
            (void)alm_rpca(mat, bad, {2, 0});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    // out-of-core (§8 f4): streamed from host memory and from a CORU .bin file (io.hpp:67-77)
    {
        const Matrix a = exact_rank(300, 120, 6, {41, 0});
        UtvApprox in = corutv(a, 10, 1, DVariant::exact, {5, 0});
        UtvApprox st = corutv_streamed(a, 10, 1, DVariant::exact, {5, 0}, 64);
        CHECK(recon_err(a, st) <= 1e-10 && recon_err(a, in) <= 1e-10);
        for (std::size_t j = 0; j < 10; ++j) CHECK(std::abs(std::abs(st.t(j, j)) - std::abs(in.t(j, j))) <= 1e-8 * std::abs(in.t(0, 0)));
        const std::string path = "/tmp/coru_wrapper_test.bin";
        if (FILE* fp = std::fopen(path.c_str(), "wb")) {
            const std::uint64_t hdr[2] = {a.rows(), a.cols()};
            std::fwrite("CORU", 1, 4, fp);
            std::fwrite(hdr, 8, 2, fp);
            std::fwrite(a.data().data(), 8, a.data().size(), fp);
            std::fclose(fp);
            UtvApprox fl = corutv_file(path, 10, 1, DVariant::exact, {5, 0}, 64);
            CHECK(fl.t.data() == st.t.data() && fl.u.data() == st.u.data());
            std::remove(path.c_str());
        } else {
            CHECK(false);
        }
    }
    std::printf("%s: %d failures\n", failures ? "FAIL" : "OK", failures);
    return failures ? 1 : 0;
}
