"""The fp64 A-pass on the INT8 tensor cores (gemm_oz.cu, Ozaki scheme) — gpu marker.

Accuracy is measured against an extended-precision product (numpy long double, 64-bit
significand) next to the FP64 DMMA kernel's: the emulated product must be at least as accurate
as a native fp64 GEMM up to a small factor, within the reference's
own matmul contract 1e-12·(|A||X|) per entry (matrix.hpp:112-114), bitwise deterministic, and
correct on every shape edge the A-passes see (row / k remainders, N = 25 ... 256, split-K).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _exact(a, x, op):
    al = (a.T if op else a).astype(np.longdouble)
    return al @ x.astype(np.longdouble)


def _run(ctx, a, x, op, engine):
    import torch
    import paper_1810_07323_b200 as cg
    ctx.set_f64_engine(engine)
    try:
        n = x.shape[1]
        xd = torch.zeros((x.shape[0], n + (n & 1)), dtype=torch.float64, device="cuda")  # even ld (16-B rows)
        xd[:, :n] = torch.from_numpy(x).cuda()
        c = cg.gemm(torch.from_numpy(a).cuda(), xd[:, :n], op=op, ctx=ctx)
        torch.cuda.synchronize()
        return c.cpu().numpy()
    finally:
        ctx.set_f64_engine(ctx.F64_AUTO)


SHAPES = [(1000, 776, 25, 0), (1000, 776, 60, 1), (2048, 1024, 112, 0), (1024, 2048, 112, 1), (300, 520, 220, 0),
          (520, 300, 256, 1), (129, 4098, 48, 0), (4100, 258, 64, 1)]


OZ_ENGINES = [2, 3]  # F64_OZAKI_INLINE (digits converted inside the A-pass kernel), F64_OZAKI_PLANES (digit planes)


@pytest.mark.parametrize("engine", OZ_ENGINES)
@pytest.mark.parametrize("m,k,n,op", SHAPES)
def test_oz_accuracy_vs_extended(ctx, m, k, n, op, engine):
    """Dense operands of uniform magnitude (the A-passes' data): the emulated product is within a
    small factor of native fp64 (median entry error <= 4x DMMA's against the exact product;
    measured 2-3x: 54-bit digits against the row / column maximum plus the dropped levels >= 7),
    and 1e-4 of the reference's own per-entry matmul contract."""
    rng = np.random.default_rng(m + k + n + op)
    a = rng.standard_normal((m, k))
    kk = m if op else k
    x = rng.standard_normal((kk, n))
    ex = _exact(a, x, op)
    c_oz = _run(ctx, a, x, op, engine)
    c_dm = _run(ctx, a, x, op, 1)
    scale = (np.abs(a.T if op else a).astype(np.longdouble) @ np.abs(x).astype(np.longdouble))
    err_oz = np.abs(c_oz - ex) / scale
    err_dm = np.abs(c_dm - ex) / scale
    print(f"median rel err ozaki {np.median(err_oz):.3e} dmma {np.median(err_dm):.3e}; "
          f"max ozaki {err_oz.max():.3e} dmma {err_dm.max():.3e}")
    assert float(err_oz.max()) <= 1e-12  # matrix.hpp:112-114 per-entry contract
    assert np.median(err_oz) <= 4 * np.median(err_dm) + 1e-18, (np.median(err_oz), np.median(err_dm))


@pytest.mark.parametrize("engine", OZ_ENGINES)
@pytest.mark.parametrize("m,k,n,op", SHAPES[2:6])
def test_oz_scaled_rows_and_columns(ctx, m, k, n, op, engine):
    """Rows / columns of op(A) and columns of X 2^±20..40 apart: the per-row and per-column
    scales absorb them; the error stays within the scheme's bound (54-bit digits against the
    row / column maximum, dropped levels >= 7) and the per-entry contract 1e-12·(|A||X|)."""
    rng = np.random.default_rng(m * 7 + k + n + op)
    a = rng.standard_normal((m, k))
    a *= np.exp2(rng.integers(-40, 40, size=(m, 1)))
    a *= np.exp2(rng.integers(-20, 20, size=(1, k)))
    kk = m if op else k
    x = rng.standard_normal((kk, n)) * np.exp2(rng.integers(-30, 30, size=(1, n)))
    ex = _exact(a, x, op)
    c_oz = _run(ctx, a, x, op, engine)
    scale = (np.abs(a.T if op else a).astype(np.longdouble) @ np.abs(x).astype(np.longdouble))
    assert float((np.abs(c_oz - ex) / scale).max()) <= 1e-12
    rowmax = np.abs(a.T if op else a).max(axis=1, keepdims=True)
    colmax = np.abs(x).max(axis=0, keepdims=True)
    assert np.all(np.abs(c_oz - ex) <= kk * 2.0 ** -49 * rowmax * colmax)


@pytest.mark.parametrize("engine", OZ_ENGINES)
def test_oz_deterministic_and_zero_rows(ctx, engine):
    """Bitwise repeatable (a multi-wave grid: 20000 rows = 157 row tiles x 2 chunks), exact zeros for
    zero rows / columns, and the two Ozaki engines agree bit for bit (same digits, same MMAs)."""
    rng = np.random.default_rng(5)
    a = rng.standard_normal((20000, 2000))
    a[7] = 0.0            # an all-zero row
    a[:, 11] = 0.0        # an all-zero column (zero output row for op T)
    x = rng.standard_normal((2000, 110))
    c1 = _run(ctx, a, x, 0, engine)
    for _ in range(6):
        assert np.array_equal(_run(ctx, a, x, 0, engine), c1)
    assert np.all(c1[7] == 0.0)
    assert np.array_equal(c1, _run(ctx, a, x, 0, 5 - engine))
    y = rng.standard_normal((20000, 110))
    t1 = _run(ctx, a, y, 1, engine)
    for _ in range(3):
        assert np.array_equal(_run(ctx, a, y, 1, engine), t1)
    assert np.all(t1[11] == 0.0)
    assert np.array_equal(t1, _run(ctx, a, y, 1, 5 - engine))


def test_oz_split_k_large_k(ctx):
    """op T with K = 200000 rows (C3's A^T·B1 shape, narrowed): split-K partials, several flushes
    of the int32 level accumulators per CTA (every 4096 k)."""
    rng = np.random.default_rng(9)
    m, n, d = 200000, 256, 112
    a = rng.standard_normal((m, n))
    y = rng.standard_normal((m, d))
    c = _run(ctx, a, y, 1, 3)
    assert np.array_equal(c, _run(ctx, a, y, 1, 2))
    ref = a.T @ y
    scale = np.abs(a).T @ np.abs(y)
    assert float((np.abs(c - ref) / scale).max()) <= 1e-13


def test_oz_decomposition_matches_dmma(ctx):
    """A whole decomposition on the Ozaki engine agrees with the DMMA engine within the
    well-conditioned (q = 0) tolerances."""
    import paper_1810_07323_b200 as cg
    from workloads import make_host
    a = make_host("C1")
    ctx.set_f64_engine(ctx.F64_DMMA)
    f_dm = cg.corutv(a, 25, 0, seed=cg.RngSeed(42, 0), ctx=ctx)
    ctx.set_f64_engine(ctx.F64_AUTO)
    f_oz = cg.corutv(a, 25, 0, seed=cg.RngSeed(42, 0), ctx=ctx)
    assert np.array_equal(f_dm.perm, f_oz.perm)
    assert np.max(np.abs(np.abs(np.diag(f_dm.t)) - np.abs(np.diag(f_oz.t)))) <= 1e-12


def test_oz_planes_decomposition_bit_identical_to_inline(ctx):
    """A whole decomposition (q = 2, wide sketch) with the digit planes is bit-identical to the one
    that converts A inside every A-pass kernel — the planes hold exactly the digits the kernel
    would produce (both orientations: row scales for A·X, column scales for A^T·Y)."""
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(77)
    a = rng.standard_normal((1500, 900)) * np.exp2(rng.integers(-8, 8, size=(1500, 1)))
    out = {}
    for eng in (ctx.F64_OZAKI_INLINE, ctx.F64_OZAKI_PLANES):
        ctx.set_f64_engine(eng)
        try:
            out[eng] = cg.corutv(a, 130, 2, seed=cg.RngSeed(42, 3), ctx=ctx)
        finally:
            ctx.set_f64_engine(ctx.F64_AUTO)
    f1, f2 = out[ctx.F64_OZAKI_INLINE], out[ctx.F64_OZAKI_PLANES]
    assert np.array_equal(f1.perm, f2.perm)
    assert np.array_equal(f1.t, f2.t) and np.array_equal(f1.u, f2.u) and np.array_equal(f1.v, f2.v)


@pytest.mark.parametrize("shape,d,q", [((1500, 900), 130, 2), ((4000, 1112), 70, 1), ((700, 2600), 40, 1)])
def test_oz_hybrid_decomposition_bit_identical_to_inline(ctx, shape, d, q):
    """Hybrid conversion — the first A·X pass converts in the kernel AND writes the row-scaled digit
    planes with TMA stores, the later A·X passes stream them — gives the bits of the all-in-kernel
    conversion: ragged row tiles and k tails (clipped stores), a wide matrix (ULV: the stored matrix
    is the transpose, so the planes serve the a^T·c1 products)."""
    import torch
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(78)
    a = rng.standard_normal(shape) * np.exp2(rng.integers(-8, 8, size=(shape[0], 1)))
    a_dev = torch.from_numpy(a).cuda()
    out = {}
    for eng in (ctx.F64_OZAKI_INLINE, ctx.F64_OZAKI_HYBRID):
        ctx.set_f64_engine(eng)
        try:
            out[eng] = cg.corutv(a_dev, d, q, seed=cg.RngSeed(42, 3), ctx=ctx)
            if eng == ctx.F64_OZAKI_HYBRID:
                assert ctx.last_f64_engine() == 3
        finally:
            ctx.set_f64_engine(ctx.F64_AUTO)
    f1, f2 = out[ctx.F64_OZAKI_INLINE], out[ctx.F64_OZAKI_HYBRID]
    assert np.array_equal(f1.perm, f2.perm)
    for x, y in ((f1.t, f2.t), (f1.u, f2.u), (f1.v, f2.v)):
        assert np.array_equal(x.cpu().numpy(), y.cpu().numpy())


def test_oz_host_entry_exponents_under_upload(ctx):
    """Host entry on an Ozaki-sized matrix: the exponent pass runs chunk by chunk under the upload
    pipeline (row exponents per chunk, column exponents as a running maximum) and the later passes
    use them — rows and columns scaled over 2^±6 so that wrong exponents would clip digits. Agrees
    with the device entry (whose first power round runs on the Ozaki engine instead of on DMMA
    chunks): leading |t_jj| to 1e-9 relative, equal reconstruction error."""
    import torch
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(79)
    m, n, d = 40000, 512, 100
    x = np.linalg.qr(rng.standard_normal((m, 120)))[0] * (0.97 ** np.arange(120))
    a = x @ np.linalg.qr(rng.standard_normal((n, 120)))[0].T + 1e-4 / np.sqrt(m) * rng.standard_normal((m, n))
    a *= np.exp2(rng.integers(-6, 6, size=(m, 1)).astype(np.float64))
    a *= np.exp2(rng.integers(-6, 6, size=(1, n)).astype(np.float64))
    f_host = cg.corutv(a, d, 1, seed=cg.RngSeed(42, 1), ctx=ctx)
    assert ctx.last_f64_engine() in (1, 3)
    f_dev = cg.corutv(torch.from_numpy(a).cuda(), d, 1, seed=cg.RngSeed(42, 1), ctx=ctx)
    assert ctx.last_f64_engine() in (1, 3)
    th, td = np.abs(np.diag(f_host.t)), np.abs(np.diag(f_dev.t.cpu().numpy()))
    assert np.max(np.abs(th - td)[:20] / td[:20]) <= 1e-9
    na = np.linalg.norm(a)
    eh = np.linalg.norm(a - (f_host.u @ f_host.t) @ f_host.v.T) / na
    ed = np.linalg.norm(a - (f_dev.u.cpu().numpy() @ f_dev.t.cpu().numpy()) @ f_dev.v.cpu().numpy().T) / na
    assert abs(eh - ed) <= 1e-6 * ed
