"""Kernel-level parity of the sm_100a kernels against the CPU oracle (gpu marker).

Tolerances:
* GEMM (K1/K2): the reference contract for any alternative matmul is 1e-12 relative per entry
  (matrix.hpp:112-114), stated norm-wise |C - C_ref| <= 1e-12·(|A||X|) because
  relative-per-entry is ill-posed where the sum cancels.
* TSQR: Q R = B to 1e-12·||B||, ||Q^T Q - I|| <= 1e-12·d, diag R >= 0, and agreement with the
  reference Householder Q/R (unique for full-rank input) to 1e-10 relative.
* QRCP: identical pivots, |diag T| to 1e-12 relative, reconstruction M P = Q T.
"""
import numpy as np
import pytest

from conftest import orth_residual

pytestmark = pytest.mark.gpu


def _t(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("m,n,d", [(1000, 1000, 25), (4000, 4000, 60), (777, 1234, 17), (3001, 129, 110),
                                   (64, 64, 8), (5, 3000, 2), (20000, 2000, 110), (2000, 3000, 220)])
@pytest.mark.parametrize("op", [0, 1])
def test_gemm_matches_oracle(ctx, oracle, m, n, d, op):
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(m * 7 + n + d + op)
    a = rng.standard_normal((m, n))
    x = rng.standard_normal((m if op else n, d))
    # leading dimension of X must be even for 16-B cp.async rows: pad to a multiple of 8
    dp = (d + 7) // 8 * 8
    xp = np.zeros((x.shape[0], dp)); xp[:, :d] = x
    c = cg.gemm(_t(a), _t(xp)[:, :d], op=op, ctx=ctx).cpu().numpy()
    want = oracle.matmul(a, x) if op == 0 else oracle.matmul_tn(a, x)
    bound = (np.abs(a) @ np.abs(x)) if op == 0 else (np.abs(a).T @ np.abs(x))
    assert np.all(np.abs(c - want) <= 1e-12 * bound + 1e-300)


@pytest.mark.parametrize("m,n,d,op", [(4000, 4000, 60, 0), (4000, 4000, 60, 1), (1000, 1000, 25, 1),
                                      (20000, 2000, 110, 1), (3001, 129, 110, 0)])
def test_gemm_streamk_fixup_deterministic(ctx, m, n, d, op):
    """Split tiles are summed inside the GEMM by the CTA owning their last k-slab, in segment order:
    repeated launches (fresh epochs over the same workspace) are bitwise identical."""
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(m + n + d)
    a = _t(rng.standard_normal((m, n)))
    x = _t(rng.standard_normal((m if op else n, (d + 7) // 8 * 8)))[:, :d]
    c0 = cg.gemm(a, x, op=op, ctx=ctx).cpu().numpy()
    for _ in range(3):
        assert np.array_equal(cg.gemm(a, x, op=op, ctx=ctx).cpu().numpy(), c0)


def test_gemm_odd_lda_and_views(ctx, oracle):
    """A with odd leading dimension (8-byte cp.async path) and a column view of a wider matrix."""
    import torch
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(5)
    big = rng.standard_normal((301, 157))
    a = big[:, :149]
    x = rng.standard_normal((149, 8))
    ta = _t(big)[:, :149]
    for op, xx, want in [(0, x, oracle.matmul(a, x))]:
        c = cg.gemm(ta, _t(xx), op=op, ctx=ctx).cpu().numpy()
        assert np.all(np.abs(c - want) <= 1e-12 * (np.abs(a) @ np.abs(xx)))
    y = rng.standard_normal((301, 8))
    c = cg.gemm(ta, _t(y), op=1, ctx=ctx).cpu().numpy()
    assert np.all(np.abs(c - oracle.matmul_tn(a, y)) <= 1e-12 * (np.abs(a).T @ np.abs(y)))


@pytest.mark.parametrize("m,d", [(4000, 60), (1000, 25), (200000, 110), (2000, 110), (61, 60), (300, 1),
                                 (5000, 220), (257, 128)])
def test_tsqr_matches_reference_householder(ctx, oracle, m, d):
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(m + d)
    b = rng.standard_normal((m, d))
    q, r = cg.tsqr(_t(b), ctx=ctx)
    q, r = q.cpu().numpy(), r.cpu().numpy()
    assert np.all(np.diag(r) >= 0)
    assert np.all(np.tril(r, -1) == 0.0)
    assert np.linalg.norm(q @ r - b) <= 1e-12 * np.linalg.norm(b)
    assert orth_residual(q) <= 1e-12 * d
    if m * d <= 4000 * 110:
        qo, ro = oracle.householder_qr(b)
        assert np.linalg.norm(q - qo) <= 1e-10 * np.sqrt(d)
        assert np.linalg.norm(r - ro) <= 1e-10 * np.linalg.norm(ro)


def test_qrcp_known_answers(ctx):
    """test_matcore.cpp:71-80: diag(1,5,3) -> perm[0] = 1 and |R| = (5,3,1)."""
    import paper_1810_07323_b200 as cg
    a = np.diag([1.0, 5.0, 3.0])
    q, r, perm = cg.qrcp(_t(a), ctx=ctx)
    r = r.cpu().numpy()
    assert perm[0] == 1
    assert np.allclose(np.abs(np.diag(r)), [5, 3, 1], rtol=1e-14)


@pytest.mark.parametrize("m,d,cond,wide", [(5000, 220, 1e2, True), (5000, 220, 1e2, False), (20000, 520, 50.0, True),
                                          (3000, 130, 1e3, True), (4000, 220, 1e12, True), (1500, 300, 1e9, True)])
def test_wide_qr_cholqr2_and_fallback(m, d, cond, wide, oracle):
    """Wide sketches (d > 128): CholeskyQR2 in fp64 (cholqr.cu) when well-conditioned, the gated
    Householder tree otherwise (cond 1e9 and 1e12 exceed the 1e6 switch): Q R = B to 1e-12,
    orthonormality 1e-12·d, positive diagonal, R equal to the reference Householder R."""
    import paper_1810_07323_b200 as cg
    ctx = cg.Context(0)
    ctx.set_wide_qr(wide)
    rng = np.random.default_rng(m + d)
    x, _ = np.linalg.qr(rng.standard_normal((m, d)))
    y, _ = np.linalg.qr(rng.standard_normal((d, d)))
    b = (x * np.logspace(0, -np.log10(cond), d)) @ y.T
    q, r = cg.tsqr(_t(b), ctx=ctx)
    q, r = q.cpu().numpy(), r.cpu().numpy()
    assert np.all(np.diag(r) > 0)
    assert np.all(np.tril(r, -1) == 0.0)
    assert np.linalg.norm(q @ r - b) <= 1e-12 * np.linalg.norm(b)
    assert orth_residual(q) <= 1e-12 * d
    if cond <= 1e3:
        # unique QR: agrees with the reference Householder factors to rounding (x cond)
        ro = oracle.householder_qr(b)[1] if m * d <= 5000 * 300 else None
        if ro is not None:
            assert np.linalg.norm(r - ro) <= 1e-12 * cond * np.linalg.norm(ro)
    ctx.close()


@pytest.mark.parametrize("n,seed", [(25, 1), (60, 2), (110, 3), (220, 4), (7, 5), (1, 6), (160, 7), (129, 8),
                                    (256, 9), (257, 10), (520, 11), (544, 12)])
def test_qrcp_matches_oracle(ctx, oracle, n, seed):
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(seed)
    # graded columns so pivots are well separated
    a = rng.standard_normal((n, n)) * np.logspace(0, -3, n)[rng.permutation(n)]
    q, r, perm = cg.qrcp(_t(a), ctx=ctx)
    q, r = q.cpu().numpy(), r.cpu().numpy()
    qo, ro, po = oracle.qrcp(a)
    assert np.array_equal(perm, po)
    assert np.all(np.tril(r, -1) == 0.0)
    # backward-stable QR: entry errors ~ eps·||A||, so the absolute part scales with |R(0,0)|·n
    assert np.allclose(np.abs(np.diag(r)), np.abs(np.diag(ro)), rtol=1e-12, atol=1e-15 * n * abs(ro[0, 0]))
    assert np.linalg.norm(q @ r - a[:, perm]) <= 1e-12 * np.linalg.norm(a)
    assert orth_residual(q) <= 1e-12 * n
    # sign convention: the last diagonal keeps its sign (no reflector when sigma == 0, qr.hpp:37)
    assert np.sign(r[-1, -1]) == np.sign(ro[-1, -1])


@pytest.mark.parametrize("n,kind", [(8, "hadamard"), (32, "hadamard"), (64, "hadamard"), (50, "dup"), (100, "dup"),
                                    (33, "zero"), (128, "zero"), (60, "rank5"), (256, "hadamard"), (300, "dup"),
                                    (520, "zero"), (220, "rank5")])
def test_qrcp_ties_and_degenerate(ctx, oracle, n, kind):
    """Tie rule (strict >, lowest position wins, qr.hpp:121-123) and degenerate columns (sigma == 0
    leaves the diagonal unreflected, qr.hpp:37): the pivot order must equal the reference's."""
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(n)
    if kind == "hadamard":  # every column has the same norm: pure tie-breaking
        h = np.array([[1.0]])
        while h.shape[0] < n:
            h = np.block([[h, h], [h, -h]])
        a = h[:n, :n].copy()
    elif kind == "dup":  # duplicated columns: equal norms, and exact cancellation after one of them
        b = rng.standard_normal((n, n // 2))
        a = np.concatenate([b, b], axis=1)[:, rng.permutation(n)]
    elif kind == "zero":
        a = rng.standard_normal((n, n))
        a[:, rng.choice(n, n // 3, replace=False)] = 0.0
    else:
        a = rng.standard_normal((n, 5)) @ rng.standard_normal((5, n))
    q, r, perm = cg.qrcp(_t(a), ctx=ctx)
    q, r = q.cpu().numpy(), r.cpu().numpy()
    qo, ro, po = oracle.qrcp(a)
    # past the numerical rank the pivots are decided by rounding noise
    k = {"rank5": 5, "dup": n // 2}.get(kind, n)
    assert np.array_equal(perm[:k], po[:k])
    assert np.all(np.tril(r, -1) == 0.0)
    assert np.linalg.norm(q @ r - a[:, perm]) <= 1e-12 * np.linalg.norm(a) * n
    assert orth_residual(q) <= 1e-12 * n
    assert np.allclose(np.abs(np.diag(r))[:k], np.abs(np.diag(ro))[:k], rtol=1e-10, atol=1e-12 * np.abs(ro[0, 0]))


@pytest.mark.parametrize("m,n,d,op", [(1000, 1000, 25, 0), (1000, 1000, 25, 1), (4097, 3001, 130, 0),
                                      (4097, 3001, 130, 1), (300, 5000, 520, 0), (5000, 300, 520, 1)])
def test_gemm_f32_matches_oracle(ctx, oracle, m, n, d, op):
    """fp32 A-pass: exact fp32 FMA accumulation; bound |C - C_ref| <= K·2^-23·(|A||X|) (fp32 unit
    roundoff times the reduction length, the standard forward error bound of a dot product)."""
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(m + n + d + op)
    a = rng.standard_normal((m, n)).astype(np.float32)
    x = rng.standard_normal((m if op else n, d)).astype(np.float32)
    c = cg.gemm(_t(a), _t(x), op=op, ctx=ctx).cpu().numpy()
    want = oracle.matmul(a, x) if op == 0 else oracle.matmul_tn(a, x)
    K = n if op == 0 else m
    bound = ((np.abs(a) @ np.abs(x)) if op == 0 else (np.abs(a).T @ np.abs(x))).astype(np.float64)
    assert np.all(np.abs(c.astype(np.float64) - want) <= K * 2.0 ** -23 * bound + 1e-30)


@pytest.mark.parametrize("m,n,d,op", [(1000, 1000, 25, 0), (1000, 1000, 25, 1), (4097, 3001, 130, 0),
                                      (4097, 3001, 130, 1), (300, 5000, 520, 0), (5000, 300, 520, 1),
                                      (129, 131, 16, 0), (131, 129, 16, 1), (2000, 777, 384, 0),
                                      (777, 2000, 400, 1), (1280, 4096, 520, 0), (4096, 1280, 520, 1)])
def test_gemm_f32_tensor_core_matches_oracle(m, n, d, op, oracle):
    """tcgen05 3xTF32 A-pass (gemm_tc32.cu) against the fp32 restatement of matmul (matrix.hpp:115-131).
    Bound: per product the split v = hi + lo loses the lo·lo term and the TF32 truncation of the lo
    parts (<= 2^-19 |a||x|), plus the fp32 accumulation over K (K·2^-22 covers both sides' sums):
    |C - C_ref| <= (2^-19 + K·2^-22)·(|A||X|). Typical errors are far smaller (checked too)."""
    import paper_1810_07323_b200 as cg
    ctx = cg.Context(0)
    ctx.set_f32_path(ctx.F32_TC)
    rng = np.random.default_rng(m + n + d + op)
    a = rng.standard_normal((m, n)).astype(np.float32)
    x = rng.standard_normal((m if op else n, d)).astype(np.float32)
    c = cg.gemm(_t(a), _t(x), op=op, ctx=ctx).cpu().numpy().astype(np.float64)
    want = oracle.matmul(a, x) if op == 0 else oracle.matmul_tn(a, x)
    K = n if op == 0 else m
    bound = ((np.abs(a) @ np.abs(x)) if op == 0 else (np.abs(a).T @ np.abs(x))).astype(np.float64)
    err = np.abs(c - want)
    assert np.all(err <= (2.0 ** -19 + K * 2.0 ** -22) * bound + 1e-30)
    assert np.median(err / bound) < 2.0 ** -22
    ctx.close()


def _ulp_diff(x, y):
    xi = x.astype(np.float64).view(np.int64)
    yi = y.astype(np.float64).view(np.int64)
    return np.abs(xi - yi)


@pytest.mark.parametrize("rows,cols,ld,seed,stream", [(7, 9, 9, 42, 3), (1, 5, 8, 7, 0), (4001, 61, 64, 5, 2),
                                                      (100, 100, 100, 42, 0), (65536, 520, 520, 42, 7)])
def test_device_gaussian_matches_host(ctx, rows, cols, ld, seed, stream):
    """rng_dev.cu vs the bit-exact host generator (rng.hpp:107-112): same xoshiro256++ word stream
    (any word slip would show as O(1) differences), Box–Muller values within 4 ulp (device
    log/sincos vs host libm), padding columns exactly zero."""
    import paper_1810_07323_b200 as cg
    g = cg.gaussian_device(rows, cols, cg.RngSeed(seed, stream), ctx=ctx, ld=ld).cpu().numpy()
    h = cg.gaussian(rows, cols, cg.RngSeed(seed, stream), threads=16)
    assert np.all(g[:, cols:] == 0.0)
    u = _ulp_diff(g[:, :cols], h)
    assert u.max() <= 4, u.max()
    assert np.mean(u > 0) < 0.3


def test_device_phi_corutv_agrees_with_host_exact(oracle):
    """The default (device Φ) and the bit-exact host-Φ modes give the same decomposition to the
    fp64 parity tolerances on a well-conditioned case."""
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(3)
    a = rng.standard_normal((600, 500))
    c_dev, c_host = cg.Context(0), cg.Context(0)
    c_host.set_phi_mode(cg.Context.PHI_HOST_EXACT)
    f1 = cg.corutv(a, 20, 0, seed=cg.RngSeed(4, 1), ctx=c_dev)
    f2 = cg.corutv(a, 20, 0, seed=cg.RngSeed(4, 1), ctx=c_host)
    assert np.array_equal(f1.perm, f2.perm)
    assert np.max(np.abs(np.abs(np.diag(f1.t)) - np.abs(np.diag(f2.t)))) <= 1e-12 * abs(f2.t[0, 0])
    ref = oracle.corutv(a, 20, 0, seed=4, stream=1)
    assert np.max(np.abs(np.abs(np.diag(f2.t)) - np.abs(np.diag(ref.t)))) <= 1e-12 * abs(ref.t[0, 0])


def test_gemm_streamk_planner_sweep(ctx):
    """Randomised stream-K planner sweep: random (rows, K, N, op), a random cap
    on the CTAs per output tile (grouped and ungrouped plans, whole / split tiles), the SAME
    workspace reused by consecutive launches of different plans — every result against a
    float64 numpy product (1e-12·|A||X| entrywise) and bitwise repeatable."""
    import torch
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(20261021)
    ctx.set_f64_engine(1)  # FP64 DMMA for everything: the stream-K kernel under test
    try:
        for trial in range(60):
            op = int(rng.integers(0, 2))
            rows = int(rng.choice([1, 7, 33, 64, 130, 220, 257, 520, 1000, 3000]))
            K = int(rng.choice([8, 40, 129, 1000, 3000, 20000]))
            N = int(rng.choice([1, 8, 25, 60, 110, 130, 220, 256]))
            cap = int(rng.choice([0, 0, 1, 2, 3, 5, 8, 16]))
            cg.debug_gemm_split_cap(cap)
            a = rng.standard_normal((K, rows) if op else (rows, K))
            npad = (N + 7) // 8 * 8
            x = np.zeros((K, npad))
            x[:, :N] = rng.standard_normal((K, N))
            ta, tx = _t(a), _t(x)[:, :N]
            c = cg.gemm(ta, tx, op=op, ctx=ctx).cpu().numpy()
            want = (a.T if op else a) @ x[:, :N]
            bound = np.abs(a.T if op else a) @ np.abs(x[:, :N])
            bad = np.abs(c - want) > 1e-12 * bound + 1e-300
            assert not bad.any(), (trial, op, rows, K, N, cap, int(bad.sum()), float(np.abs(c - want).max()))
            assert np.array_equal(cg.gemm(ta, tx, op=op, ctx=ctx).cpu().numpy(), c), (trial, op, rows, K, N, cap)
    finally:
        cg.debug_gemm_split_cap(0)
        ctx.set_f64_engine(0)


@pytest.mark.parametrize("cap", [1, 2, 4])
@pytest.mark.parametrize("m,d", [(3000, 130), (5000, 220), (2048, 136)])
def test_wide_qr_under_split_caps(ctx, m, d, cap):
    """CholeskyQR2 (Gram + R2·R1 products on the stream-K GEMM, one shared workspace) with the
    planner's split capped: the configuration DESIGN.md (round 1) recorded as producing a wrong
    Gram. Q R = B, orthonormal Q."""
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(m + d + cap)
    b = rng.standard_normal((m, d))
    cg.debug_gemm_split_cap(cap)
    try:
        q, r = cg.tsqr(_t(b), ctx=ctx)
        q, r = q.cpu().numpy(), r.cpu().numpy()
    finally:
        cg.debug_gemm_split_cap(0)
    assert np.linalg.norm(q @ r - b) <= 1e-12 * np.linalg.norm(b) * d
    assert orth_residual(q) <= 1e-12 * d
