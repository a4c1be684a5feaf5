"""DVariant::approx on the GPU (corutv.hpp:91-92) and its pinv core (svd.hpp:31-187) (gpu marker).

The approx variant forms the core from the sketches, D = (Q1^T C1)·pinv(Q2^T C2prev), instead of a
third pass over A. The GPU pinv runs the reference's one-sided Jacobi rotations in round-robin
instead of cyclic pair order (svd.cu), so factors agree with the reference to rounding (scaled
by the condition number of the kept part), not bit-for-bit. Checked against the reference's own
fixtures (tests/golden/approx_ref_cases.npz) and the CPU oracle.
"""
import numpy as np
import pytest

from conftest import orth_residual, rel_recon_error
from golden import approx_cases, pinv_cases

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


def _pinv_tol(a, s_ref):
    """Rounding-level tolerance for pinv(a) when the kept/dropped split of the singular values
    is clean (no sigma within 10x of the cut d·eps·sigma_1); None when the split is ambiguous."""
    n = a.shape[0]
    if s_ref[0] == 0.0:
        return 0.0
    cut = n * EPS * s_ref[0]
    kept = s_ref[s_ref > cut]
    if np.any((s_ref > cut / 10) & (s_ref < cut * 10)):
        return None
    kappa = kept[0] / kept[-1]
    return 1e-13 * n * kappa


@pytest.mark.parametrize("case", pinv_cases(), ids=lambda c: c["name"])
def test_pinv_kernel_vs_reference(ctx, case):
    import torch
    import paper_1810_07323_b200 as cg
    a = case["A"]
    p, sweeps = cg.pinv(torch.from_numpy(a).cuda(), ctx=ctx)
    p = p.cpu().numpy()
    assert (sweeps > 0) == case["converged"]
    tol = _pinv_tol(a, case["S"])
    nrm = max(np.linalg.norm(case["P"]), 1e-300)
    if tol is not None:
        assert np.linalg.norm(p - case["P"]) <= tol * nrm
    # Penrose identities in any case (test_matcore.cpp:195-205)
    sc = max(np.linalg.norm(a), 1e-300)
    assert np.linalg.norm(a @ p @ a - a) <= 1e-10 * sc


@pytest.mark.parametrize("n", [60, 110, 220, 520])
def test_pinv_kernel_wide_vs_oracle(ctx, oracle, n):
    """Core widths of C2 (60), C3 (110), C4 (220) and C5 (520); the widest run from L2."""
    import torch
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) * (0.97 ** np.arange(n))
    want = oracle.pinv(a)
    got, sweeps = cg.pinv(torch.from_numpy(a).cuda(), ctx=ctx)
    assert 0 < sweeps <= 20
    s = np.linalg.svd(a, compute_uv=False)
    assert np.linalg.norm(got.cpu().numpy() - want) <= 1e-13 * n * (s[0] / s[-1]) * np.linalg.norm(want)


@pytest.mark.parametrize("case", approx_cases(), ids=lambda c: c["name"])
def test_approx_reference_cases(ctx, case):
    import paper_1810_07323_b200 as cg
    a, ell, q = case["A"], case["ell"], case["q"]
    f = cg.corutv(a, ell, q, cg.DVariant.approx, cg.RngSeed(case["seed"], case["stream"]), ctx=ctx)
    assert f.lower == case["lower"] and f.variant == cg.DVariant.approx
    t = f.t
    assert np.all((np.triu(t, 1) if f.lower else np.tril(t, -1)) == 0.0)
    assert orth_residual(f.u) <= 1e-12 * ell and orth_residual(f.v) <= 1e-12 * ell
    e_gpu = rel_recon_error(a, f.u, f.t, f.v)
    e_ref = rel_recon_error(a, case["U"], case["T"], case["V"])
    dg = np.abs(np.abs(np.diag(f.t)) - np.abs(np.diag(case["T"])))
    if q == 0 and not case["warning"]:
        # well-conditioned sketch: the stated fp64 tolerances (BASELINE north_star)
        assert abs(e_gpu - e_ref) <= 1e-10 * max(e_ref, 1e-300) or abs(e_gpu - e_ref) <= 1e-14
        assert dg.max() <= 1e-8
    else:
        assert e_gpu <= 1.5 * e_ref + 1e-13
    assert f.conditioning_warning == case["warning"]


def test_approx_agrees_with_exact_on_exact_rank(ctx):
    """test_corutv.cpp:87-96 on the GPU."""
    import paper_1810_07323_b200 as cg
    a = approx_cases()[0]["A"]
    for q in (0, 2):
        e = cg.corutv(a, 10, q, cg.DVariant.exact, cg.RngSeed(10, 0), ctx=ctx)
        p = cg.corutv(a, 10, q, cg.DVariant.approx, cg.RngSeed(10, 0), ctx=ctx)
        assert np.linalg.norm(e.u @ e.t @ e.v.T - p.u @ p.t @ p.v.T) <= 1e-6 * np.linalg.norm(a)


@pytest.mark.parametrize("name,m,n", [("C1", 1000, 1000), ("C2q1", 4000, 4000)])
def test_approx_config_parity_vs_oracle(ctx, oracle, name, m, n):
    import paper_1810_07323_b200 as cg
    from workloads import CONFIGS, make_host
    c = CONFIGS[name]
    a = make_host(name, m, n)
    f = cg.corutv(a, c.d, c.q, cg.DVariant.approx, cg.RngSeed(42, 0), ctx=ctx)
    o = oracle.corutv(a, c.d, c.q, 1, 42, 0, threads=16)
    e_gpu, e_ora = rel_recon_error(a, f.u, f.t, f.v), rel_recon_error(a, o.u, o.t, o.v)
    dg = np.abs(np.abs(np.diag(f.t)) - np.abs(np.diag(o.t)))
    assert orth_residual(f.u) <= 1e-12 * c.d and orth_residual(f.v) <= 1e-12 * c.d
    if c.q == 0:
        assert abs(e_gpu - e_ora) <= 1e-10 * e_ora
        assert dg.max() <= 1e-8
        assert np.array_equal(f.perm, o.perm)
    else:
        # power rounds: rounding is amplified like in the exact variant (SURVEY.md §8c floors)
        assert e_gpu <= e_ora * 1.05


def test_approx_fp32_vs_fp32_oracle(ctx, oracle):
    import paper_1810_07323_b200 as cg
    from workloads import make_host
    a = make_host("C1", 1000, 1000).astype(np.float32)
    f = cg.corutv(a, 25, 0, cg.DVariant.approx, cg.RngSeed(42, 0), ctx=ctx)
    o = oracle.corutv(a, 25, 0, 1, 42, 0, threads=16)
    a64 = a.astype(np.float64)
    e_gpu = rel_recon_error(a64, *(x.astype(np.float64) for x in (f.u, f.t, f.v)))
    e_ora = rel_recon_error(a64, *(x.astype(np.float64) for x in (o.u, o.t, o.v)))
    assert abs(e_gpu - e_ora) <= 1e-4 * e_ora
    assert np.abs(np.abs(np.diag(f.t)) - np.abs(np.diag(o.t))).max() <= 1e-3


def test_approx_device_entry_and_determinism(ctx):
    import torch
    import paper_1810_07323_b200 as cg
    from workloads import make_host
    a = make_host("C1", 1000, 1000)
    ad = torch.from_numpy(a).cuda()
    f1 = cg.corutv(ad, 25, 1, cg.DVariant.approx, cg.RngSeed(3, 1), ctx=ctx)
    f2 = cg.corutv(ad, 25, 1, cg.DVariant.approx, cg.RngSeed(3, 1), ctx=ctx)
    h = cg.corutv(a, 25, 1, cg.DVariant.approx, cg.RngSeed(3, 1), ctx=ctx)
    for x, y, z in [(f1.u, f2.u, h.u), (f1.t, f2.t, h.t), (f1.v, f2.v, h.v)]:
        x = x.cpu().numpy() if hasattr(x, "cpu") else x
        y = y.cpu().numpy() if hasattr(y, "cpu") else y
        assert np.array_equal(x, y) and np.array_equal(x, z)
