"""SVD-based baselines on the GPU (§8 f3): svd of the square core (svd.hpp:31-161), tsr_svd and
sor_svd (baselines.hpp:43-71), checked against the reference's own outputs
(tests/golden/approx_ref_cases.npz, baselines_ref_cases.npz) and the reference's test properties
(proj/tests/test_baselines.cpp, test_matcore.cpp:119-176). The GPU Jacobi SVD visits pairs in
round-robin order (svd.cu), so results agree with the reference to rounding, not bit-for-bit."""
import numpy as np
import pytest

from conftest import orth_residual
from golden import pinv_cases, sor_cases, tsr_cases

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", pinv_cases(), ids=lambda c: c["name"])
def test_svd_kernel_vs_reference(ctx, case):
    import torch
    import paper_1810_07323_b200 as cg
    a = case["A"]
    n = a.shape[0]
    f = cg.svd(torch.from_numpy(a).cuda(), ctx=ctx)
    u, s, v = f.u.cpu().numpy(), f.sigma.cpu().numpy(), f.v.cpu().numpy()
    assert f.converged == case["converged"]
    sc = max(case["S"][0], 1e-300)
    assert np.all(np.diff(s) <= 0)                                  # non-increasing (svd.hpp:79-82)
    assert np.max(np.abs(s - case["S"])) <= 1e-13 * n * sc          # singular values to rounding
    assert np.linalg.norm((u * s) @ v.T - a) <= 1e-12 * max(np.linalg.norm(a), 1e-300)
    assert orth_residual(v) <= 1e-12 * n
    assert orth_residual(u) <= 1e-12 * n                            # incl. zero-sigma completion


@pytest.mark.parametrize("case", tsr_cases(), ids=lambda c: c["name"])
def test_tsr_svd_vs_reference(ctx, case):
    import paper_1810_07323_b200 as cg
    a, ell = case["A"], case["ell"]
    f = cg.tsr_svd(a, ell, cg.RngSeed(case["seed"], case["stream"]), ctx=ctx)
    assert f.u.shape == (a.shape[0], ell) and f.v.shape == (a.shape[1], ell)
    # test_baselines.cpp:68-79: orthonormal factors, reproducible
    assert orth_residual(f.u) <= 1e-9 * np.sqrt(ell) and orth_residual(f.v) <= 1e-9 * np.sqrt(ell)
    g = cg.tsr_svd(a, ell, cg.RngSeed(case["seed"], case["stream"]), ctx=ctx)
    assert np.array_equal(f.u, g.u) and np.array_equal(f.sigma, g.sigma) and np.array_equal(f.v, g.v)
    # the numerically significant estimates agree with the reference's
    s_ref = case["S"]
    sig = s_ref > 1e-8 * s_ref[0]
    assert np.max(np.abs(f.sigma[sig] - s_ref[sig]) / s_ref[sig]) <= 1e-8
    assert f.converged == case["converged"]


def test_tsr_rank1_leading_estimate(ctx):
    """test_baselines.cpp:57-66."""
    import paper_1810_07323_b200 as cg
    c = next(x for x in tsr_cases() if x["name"] == "tsr_rank1_50x30")
    a = c["A"]
    f = cg.tsr_svd(a, 2, cg.RngSeed(18, 0), ctx=ctx)
    assert abs(f.sigma[0] - np.linalg.norm(a, 2)) <= 0.01 * np.linalg.norm(a, 2)


@pytest.mark.parametrize("case", sor_cases(), ids=lambda c: c["name"])
def test_sor_svd_vs_reference(ctx, case):
    import paper_1810_07323_b200 as cg
    a = case["A"]
    out = cg.sor_svd(a, case["k"], case["ell"], case["q"], cg.RngSeed(case["seed"], case["stream"]), ctx=ctx)
    assert out.shape == a.shape
    tol = 1e-9 if case["q"] == 0 else 1e-6  # power rounds amplify rounding
    assert np.linalg.norm(out - case["L"]) <= tol * np.linalg.norm(a)
    s = np.linalg.svd(out, compute_uv=False)                     # test_baselines.cpp:45-55
    assert s[case["k"]] <= 1e-9 * s[0]


def test_sor_svd_properties(ctx):
    """test_baselines.cpp:99-112: exact rank-k recovery, k = ell equals the corutv reconstruction."""
    import paper_1810_07323_b200 as cg
    c = next(x for x in sor_cases() if x["name"] == "sor_exact_rank_25x18")
    a = c["A"]
    assert np.linalg.norm(a - cg.sor_svd(a, 5, 8, 0, cg.RngSeed(23, 0), ctx=ctx)) <= 1e-8 * np.linalg.norm(a)
    d = next(x for x in sor_cases() if x["name"] == "sor_fast_decay_60_k12")
    s = cg.sor_svd(d["A"], 12, 12, 0, cg.RngSeed(25, 0), ctx=ctx)
    f = cg.corutv(d["A"], 12, 0, seed=cg.RngSeed(25, 0), ctx=ctx)
    assert np.linalg.norm(s - f.u @ f.t @ f.v.T) <= 1e-9 * np.linalg.norm(d["A"])


def test_baselines_bad_parameters(ctx):
    import paper_1810_07323_b200 as cg
    a = cg.gaussian(25, 18, cg.RngSeed(22, 0))
    with pytest.raises(cg.CoruInvalidArgument):
        cg.sor_svd(a, 9, 8, 0, cg.RngSeed(23, 0), ctx=ctx)   # k > ell (test_baselines.cpp:103)
    with pytest.raises(cg.CoruInvalidArgument):
        cg.sor_svd(a, 1, 18, 0, cg.RngSeed(23, 0), ctx=ctx)  # ell >= min(m, n) (:104)
    with pytest.raises(cg.CoruInvalidArgument):
        cg.sor_svd(a, 1, 5, -1, cg.RngSeed(23, 0), ctx=ctx)
    for ell in (0, 18):
        with pytest.raises(cg.CoruInvalidArgument):
            cg.tsr_svd(a, ell, cg.RngSeed(1, 0), ctx=ctx)


def test_baselines_device_entry_matches_host(ctx):
    import torch
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(3)
    a = rng.standard_normal((700, 500)) * (0.98 ** np.arange(500))
    ad = torch.from_numpy(a).cuda()
    h = cg.tsr_svd(a, 30, cg.RngSeed(5, 1), ctx=ctx)
    d = cg.tsr_svd(ad, 30, cg.RngSeed(5, 1), ctx=ctx)
    assert np.array_equal(h.u, d.u.cpu().numpy()) and np.array_equal(h.sigma, d.sigma.cpu().numpy())
    hs = cg.sor_svd(a, 10, 30, 1, cg.RngSeed(5, 1), ctx=ctx)
    ds = cg.sor_svd(ad, 10, 30, 1, cg.RngSeed(5, 1), ctx=ctx)
    assert np.array_equal(hs, ds.cpu().numpy())
    wt = cg.sor_svd(np.ascontiguousarray(a.T), 10, 30, 1, cg.RngSeed(5, 1), ctx=ctx)  # m < n orientation
    assert wt.shape == (500, 700)


@pytest.mark.parametrize("m,n,k,ell,q", [(4000, 4000, 50, 60, 1), (2000, 6000, 100, 110, 1)])
def test_sor_svd_vs_oracle_config_sized(ctx, oracle, m, n, k, ell, q):
    """C2-shaped (and a wide C3-like) sor_svd against the oracle restatement: the rank-k error
    matches the reference's within a small multiple of the corutv floors."""
    import paper_1810_07323_b200 as cg
    from workloads import make_host
    a = make_host("C2q1", m, n)
    out = cg.sor_svd(a, k, ell, q, cg.RngSeed(42, 0), ctx=ctx)
    ref = oracle.sor_svd(a, k, ell, q, 42, 0, threads=16)
    e_g = np.linalg.norm(a - out) / np.linalg.norm(a)
    e_o = np.linalg.norm(a - ref) / np.linalg.norm(a)
    assert e_g <= e_o * 1.01 + 1e-14
