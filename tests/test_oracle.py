"""The CPU oracle pinned against the reference (CPU; no GPU needed).

The plain-C restatement (oracle/coru_oracle.c) must reproduce the compiled reference bit-for-bit:
checked against the committed golden fixtures (always) and against oracle/_ref live when it is
present. This is what entitles the GPU parity tests to use the oracle as the checker.
"""
import numpy as np
import pytest

from golden import approx_cases, corutv_cases, kat, pinv_cases, sketch_case, sor_cases, tsr_cases


def test_rng_words_and_gaussian_bitexact(oracle):
    k = kat()
    assert np.array_equal(oracle.xoshiro_words(42, 0, 64), k["xoshiro_42_0"])
    assert np.array_equal(oracle.xoshiro_words(0, 0, 16), k["xoshiro_0_0"])
    for key, (r, c, s, st) in {"gaussian_4x4_1_0": (4, 4, 1, 0), "gaussian_4x4_1_1": (4, 4, 1, 1),
                               "gaussian_7x9_42_3": (7, 9, 42, 3), "gaussian_100x100_42_0": (100, 100, 42, 0),
                               "gaussian_1x5_7_0": (1, 5, 7, 0)}.items():
        assert np.array_equal(oracle.gaussian(r, c, s, st), k[key]), key


def test_gaussian_properties(oracle):
    """test_matcore.cpp:207-230: determinism, distinct streams differ, moments."""
    a = oracle.gaussian(4, 4, 1, 0)
    assert np.array_equal(a, oracle.gaussian(4, 4, 1, 0))
    assert np.abs(a - oracle.gaussian(4, 4, 1, 1)).max() > 0
    g = oracle.gaussian(100, 100, 42, 0)
    assert abs(g.mean()) <= 0.05 and 0.9 <= g.var(ddof=1) <= 1.1


def test_qr_qrcp_bitexact(oracle):
    k = kat()
    q, r = oracle.householder_qr(k["qr_in"])
    assert np.array_equal(q, k["qr_q"]) and np.array_equal(r, k["qr_r"])
    q, r = oracle.householder_qr(np.array([[3.0], [4.0]]))
    assert np.array_equal(q, k["qr34_q"]) and np.array_equal(r, k["qr34_r"])
    assert abs(r[0, 0]) == pytest.approx(5.0) and abs(q[0, 0]) == pytest.approx(0.6)
    q, r = oracle.householder_qr(k["qr_rankdef_in"])
    assert np.array_equal(q, k["qr_rankdef_q"]) and np.array_equal(r, k["qr_rankdef_r"])
    for name in ["qrcp_diag", "qrcp_rank1"] + [f"qrcp_trial{t}" for t in range(12)]:
        src = np.diag([1.0, 5.0, 3.0]) if name == "qrcp_diag" else k[f"{name}_in"]
        q, r, p = oracle.qrcp(src)
        assert np.array_equal(q, k[f"{name}_q"]) and np.array_equal(r, k[f"{name}_r"]), name
        assert np.array_equal(p, k[f"{name}_perm"]), name
    assert oracle.qrcp(np.diag([1.0, 5.0, 3.0]))[2][0] == 1  # test_matcore.cpp:71-80


def test_householder_rejects_wide(oracle):
    with pytest.raises(ValueError):
        oracle.householder_qr(np.zeros((3, 4)))


@pytest.mark.parametrize("case", corutv_cases(), ids=lambda c: c["name"])
def test_corutv_bitexact_vs_golden(oracle, case):
    f = oracle.corutv(case["A"], case["ell"], case["q"], 0, case["seed"], case["stream"])
    assert np.array_equal(f.u, case["U"])
    assert np.array_equal(f.t, case["T"])
    assert np.array_equal(f.v, case["V"])
    assert f.lower == case["lower"] and f.conditioning_warning == case["warning"]


@pytest.mark.parametrize("case", approx_cases(), ids=lambda c: c["name"])
def test_corutv_approx_bitexact_vs_golden(oracle, case):
    """DVariant::approx (corutv.hpp:91-92): sketch products, pinv (svd.hpp) and the core product."""
    f = oracle.corutv(case["A"], case["ell"], case["q"], 1, case["seed"], case["stream"])
    assert np.array_equal(f.u, case["U"])
    assert np.array_equal(f.t, case["T"])
    assert np.array_equal(f.v, case["V"])
    assert f.lower == case["lower"] and f.conditioning_warning == case["warning"]


@pytest.mark.parametrize("case", pinv_cases(), ids=lambda c: c["name"])
def test_pinv_and_jacobi_svd_bitexact_vs_golden(oracle, case):
    """pinv (svd.hpp:167-187) and the square one-sided Jacobi SVD (svd.hpp:31-134, 141-161)."""
    assert np.array_equal(oracle.pinv(case["A"]), case["P"])
    u, s, v, conv = oracle.jacobi_svd_square(case["A"])
    assert np.array_equal(s, case["S"]) and np.array_equal(u, case["U"]) and np.array_equal(v, case["V"])
    assert conv == case["converged"]


def test_pinv_properties(oracle):
    """test_matcore.cpp:178-205: diagonal / zero / orthonormal inputs and the Penrose identities."""
    p = oracle.pinv(np.diag([2.0, 0.0]))
    assert p[0, 0] == 0.5 and p[1, 1] == 0.0
    assert np.max(np.abs(oracle.pinv(np.zeros((3, 3))))) == 0.0
    q, _ = oracle.householder_qr(oracle.gaussian(8, 8, 13, 0))
    assert np.max(np.abs(oracle.pinv(q) - q.T)) <= 1e-12
    a = oracle.gaussian(10, 10, 17, 0)
    ap = oracle.pinv(a)
    sc = np.linalg.norm(a)
    assert np.linalg.norm(a @ ap @ a - a) <= 1e-10 * sc
    assert np.linalg.norm(ap @ a @ ap - ap) <= 1e-9 * sc


def test_approx_agrees_with_exact_on_exact_rank(oracle):
    """test_corutv.cpp:87-96: approx-D and exact-D reconstructions agree on an exact-rank matrix."""
    c = approx_cases()[0]
    a = c["A"]
    for q in (0, 2):
        e = oracle.corutv(a, 10, q, 0, 10, 0)
        p = oracle.corutv(a, 10, q, 1, 10, 0)
        assert np.linalg.norm(e.u @ e.t @ e.v.T - p.u @ p.t @ p.v.T) <= 1e-6 * np.linalg.norm(a)


def test_corutv_threads_do_not_change_bits(oracle):
    case = corutv_cases()[1]
    f1 = oracle.corutv(case["A"], case["ell"], case["q"], 0, case["seed"], 0, threads=1)
    f8 = oracle.corutv(case["A"], case["ell"], case["q"], 0, case["seed"], 0, threads=8)
    assert np.array_equal(f1.u, f8.u) and np.array_equal(f1.t, f8.t) and np.array_equal(f1.v, f8.v)


def test_sketch_bases_bitexact(oracle):
    c = sketch_case()
    q1, q2, c1, c2p, w = oracle.sketch_bases(c["A"], c["ell"], c["q"], c["seed"], c["stream"])
    for got, key in [(q1, "Q1"), (q2, "Q2"), (c1, "C1"), (c2p, "C2prev")]:
        assert np.array_equal(got, c[key]), key
    assert w == c["warning"]


def test_bad_parameters(oracle):
    a = oracle.gaussian(10, 8, 1, 0)
    for ell, q in [(0, 0), (8, 0), (3, -1)]:
        with pytest.raises(ValueError):
            oracle.corutv(a, ell, q, seed=1)


def test_oracle_matches_live_reference(oracle, reference):
    """When oracle/_ref is built (this container), compare against the reference directly."""
    rng = np.random.default_rng(7)
    for (m, n, d, q) in [(200, 150, 12, 0), (150, 200, 10, 1), (300, 120, 30, 2)]:
        a = rng.standard_normal((m, n))
        f = oracle.corutv(a, d, q, 0, 42, 3)
        g = reference.corutv(a, d, q, 0, 42, 3)
        assert np.array_equal(f.u, g.u) and np.array_equal(f.t, g.t) and np.array_equal(f.v, g.v)
        assert f.conditioning_warning == g.conditioning_warning
        f = oracle.corutv(a, d, q, 1, 42, 3)
        g = reference.corutv(a, d, q, 1, 42, 3)
        assert np.array_equal(f.u, g.u) and np.array_equal(f.t, g.t) and np.array_equal(f.v, g.v)
    for n in (1, 3, 16, 33, 64):
        a = rng.standard_normal((n, n)) * (0.5 ** np.arange(n))
        assert np.array_equal(oracle.pinv(a), reference.pinv(a))


def test_reference_threaded_driver_bitexact(reference):
    rng = np.random.default_rng(8)
    a = rng.standard_normal((500, 300))
    f = reference.corutv(a, 20, 1, 0, 5, 0, threads=1)
    g = reference.corutv(a, 20, 1, 0, 5, 0, threads=4)
    assert np.array_equal(f.u, g.u) and np.array_equal(f.t, g.t) and np.array_equal(f.v, g.v)


def test_fp32_restatement_tracks_fp64(oracle):
    """fp32 restatement: |diag T| within the fp32 tolerance (1e-3 absolute), the
    leading k = 20 (signal) estimates to 1e-5 relative."""
    from workloads import make_host
    a = make_host("C1", 300, 300)
    f64 = oracle.corutv(a, 25, 0, seed=42)
    f32 = oracle.corutv(a.astype(np.float32), 25, 0, seed=42)
    d64, d32 = np.abs(np.diag(f64.t)), np.abs(np.diag(f32.t))
    assert np.max(np.abs(d64 - d32)) <= 1e-3
    assert np.max(np.abs(d64 - d32)[:20] / d64[:20]) <= 1e-5


@pytest.mark.parametrize("case", tsr_cases(), ids=lambda c: c["name"])
def test_tsr_svd_bitexact_vs_golden(oracle, case):
    """tsr_svd (baselines.hpp:43-56): two sketches, two QRs, pinv core, square Jacobi SVD, lift."""
    u, s, v, conv = oracle.tsr_svd(case["A"], case["ell"], case["seed"], case["stream"])
    assert np.array_equal(u, case["U"]) and np.array_equal(s, case["S"]) and np.array_equal(v, case["V"])
    assert conv == case["converged"]


@pytest.mark.parametrize("case", sor_cases(), ids=lambda c: c["name"])
def test_sor_svd_bitexact_vs_golden(oracle, case):
    """sor_svd (baselines.hpp:61-71): sketch bases, exact core, truncated SVD, lifted m x n."""
    out = oracle.sor_svd(case["A"], case["k"], case["ell"], case["q"], case["seed"], case["stream"])
    assert np.array_equal(out, case["L"])


def test_sor_svd_equals_corutv_reconstruction_at_k_ell(oracle):
    """test_baselines.cpp:106-112: sor_svd(k = ell) == reconstruct(corutv) for the same seed."""
    c = next(x for x in sor_cases() if x["name"] == "sor_fast_decay_60_k12")
    f = oracle.corutv(c["A"], 12, 0, 0, 25, 0)
    assert np.linalg.norm(c["L"] - f.u @ f.t @ f.v.T) <= 1e-9 * np.linalg.norm(c["A"])


# ---- alm_rpca with the CoR-UTV inner (rpca.hpp:95-169, §8 f2) -------------------------------
from golden import rpca_cases  # noqa: E402


@pytest.mark.parametrize("case", rpca_cases(), ids=lambda c: c["name"])
def test_alm_rpca_bitexact_vs_golden(oracle, case):
    """The numpy/C restatement reproduces the reference's alm_rpca bit for bit (L, S, residual history,
    iteration count, rank, l0 count, flags)."""
    r = oracle.alm_rpca(case["M"], seed=case["seed"], stream=case["stream"], **case["cfg"])
    assert r["iterations"] == case["iterations"]
    assert r["rank_l"] == case["rank_l"] and r["s_l0"] == case["s_l0"]
    assert r["converged"] == case["converged"] and r["ell_clamped"] == case["ell_clamped"]
    assert np.array_equal(r["residuals"], case["residuals"])
    assert np.array_equal(r["l"], case["L"]) and np.array_equal(r["s"], case["S"])


def test_alm_rpca_matches_live_reference(oracle, reference):
    m = reference.gen_rpca_instance(40, 3, 80, 80.0, 22)[0]  # test_cli.cpp:185-195 instance
    for kw in (dict(corutv_ell=6), dict(corutv_ell=6, thresholding=1), dict(corutv_ell=0, max_iter=1)):
        a = reference.alm_rpca(m, seed=4, **kw)
        b = oracle.alm_rpca(m, seed=4, **kw)
        assert a["iterations"] == b["iterations"] and np.array_equal(a["residuals"], b["residuals"])
        assert np.array_equal(a["l"], b["l"]) and np.array_equal(a["s"], b["s"])


def test_alm_rpca_config_validation(oracle):
    m = np.eye(6)
    for kw in (dict(rho=1.0), dict(tol=0.0), dict(max_iter=0), dict(corutv_q=-1)):  # rpca.hpp:72-77
        with pytest.raises(Exception):
            oracle.alm_rpca(m, corutv_ell=2, **kw)


def test_acceptance_criterion7_recovery_fixture():
    """acceptance.cpp:186-230: the reference's CoR-UTV RPCA recovers rank 20 and the sparse support."""
    c = next(x for x in rpca_cases() if x["name"].startswith("acc7"))
    assert c["converged"] and c["rank_l"] == 20 and c["residuals"][-1] < 1e-5 and c["iterations"] <= 20
    st, s = c["S_true"], c["S"]
    assert np.all(np.abs(s[st == 0]) <= 1e-6)
    assert np.all(np.sign(s[st != 0]) == np.sign(st[st != 0]))
