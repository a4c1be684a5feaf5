"""The row-sharded (multi-rank) C++ path on one GPU: ranks are host threads with their own
contexts, joined by the in-process collective group (coru_threadcomm: stream sync + host
barrier + fixed-order device sums — no kernel ever waits on another). This runs exactly the
orchestration the NCCL build runs at N GPUs (sharded A^T-products, cross-rank TSQR top level by
all-gather, all-reduced core) and checks it against the single-GPU decomposition (gpu marker)."""
import threading

import numpy as np
import pytest

from conftest import orth_residual

pytestmark = pytest.mark.gpu


def _run_sharded(a_dev, d, q, world, seed=42, variant=0):
    import torch
    import paper_1810_07323_b200 as cg
    m, n = a_dev.shape
    group = cg.ThreadGroup(world)
    out = [None] * world
    err = []

    def worker(rank):
        try:
            ctx = cg.Context(0)
            ctx.init_threadcomm(group, rank)
            r0, rows = cg.shard_rows(m, rank, world)
            a_r = a_dev[r0:r0 + rows].contiguous()
            torch.cuda.synchronize()
            f = cg.corutv(a_r, d, q, cg.DVariant(variant), seed=cg.RngSeed(seed, 0), ctx=ctx, m_global=m)
            torch.cuda.synchronize()
            out[rank] = f
        except Exception as e:  # surfaced below (the group releases the other ranks)
            err.append(f"rank {rank}: {e!r}")

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not err, err
    return out


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("m,n,d,q", [(3000, 1500, 40, 1), (4000, 4000, 60, 1), (20000, 2000, 110, 1)])
def test_sharded_matches_single_gpu(ctx, world, m, n, d, q):
    import torch
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(m + n + d + world)
    # rank 2d with sigma from 1 down to 1e-2: the q = 1 sketch stays well conditioned, so the
    # sharded and single-GPU runs must agree to rounding
    r = 2 * d
    x, _ = np.linalg.qr(rng.standard_normal((m, r)))
    y, _ = np.linalg.qr(rng.standard_normal((n, r)))
    a = (x * np.logspace(0, -2, r)) @ y.T + 1e-7 * rng.standard_normal((m, n))
    a_dev = torch.from_numpy(a).cuda()
    single = cg.corutv(a_dev, d, q, seed=cg.RngSeed(42, 0), ctx=ctx)
    parts = _run_sharded(a_dev, d, q, world)
    # replicated outputs are bit-identical on every rank
    for f in parts[1:]:
        assert torch.equal(f.t, parts[0].t) and torch.equal(f.v, parts[0].v)
        assert np.array_equal(f.perm, parts[0].perm)
        assert f.conditioning_warning == parts[0].conditioning_warning
    u = torch.cat([f.u for f in parts]).cpu().numpy()
    t, v = parts[0].t.cpu().numpy(), parts[0].v.cpu().numpy()
    assert orth_residual(u) <= 1e-12 * d and orth_residual(v) <= 1e-12 * d
    e_sh = np.linalg.norm(a - u @ t @ v.T) / np.linalg.norm(a)
    su, st, sv = single.u.cpu().numpy(), single.t.cpu().numpy(), single.v.cpu().numpy()
    e_1 = np.linalg.norm(a - su @ st @ sv.T) / np.linalg.norm(a)
    assert abs(e_sh - e_1) <= 1e-9 * e_1
    assert np.max(np.abs(np.abs(np.diag(t)) - np.abs(np.diag(st)))) <= 1e-9 * abs(st[0, 0])
    assert np.array_equal(parts[0].perm, single.perm)
    # determinism of the sharded path itself
    again = _run_sharded(a_dev, d, q, world)
    assert torch.equal(again[0].t, parts[0].t) and torch.equal(torch.cat([f.u for f in again]), torch.cat([f.u for f in parts]))


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_approx_matches_single_gpu(ctx, world):
    """DVariant::approx sharded: Q1^T C1 is all-reduced, the pinv of Q2^T C2prev is replicated."""
    import torch
    import paper_1810_07323_b200 as cg
    m, n, d, q = 4000, 2000, 40, 1
    rng = np.random.default_rng(world)
    r = 2 * d
    x, _ = np.linalg.qr(rng.standard_normal((m, r)))
    y, _ = np.linalg.qr(rng.standard_normal((n, r)))
    a = (x * np.logspace(0, -2, r)) @ y.T + 1e-7 * rng.standard_normal((m, n))
    a_dev = torch.from_numpy(a).cuda()
    single = cg.corutv(a_dev, d, q, cg.DVariant.approx, seed=cg.RngSeed(42, 0), ctx=ctx)
    parts = _run_sharded(a_dev, d, q, world, variant=1)
    for f in parts[1:]:
        assert torch.equal(f.t, parts[0].t) and torch.equal(f.v, parts[0].v)
    u = torch.cat([f.u for f in parts]).cpu().numpy()
    t, v = parts[0].t.cpu().numpy(), parts[0].v.cpu().numpy()
    assert orth_residual(u) <= 1e-12 * d and orth_residual(v) <= 1e-12 * d
    su, st, sv = single.u.cpu().numpy(), single.t.cpu().numpy(), single.v.cpu().numpy()
    e_sh = np.linalg.norm(a - u @ t @ v.T) / np.linalg.norm(a)
    e_1 = np.linalg.norm(a - su @ st @ sv.T) / np.linalg.norm(a)
    assert abs(e_sh - e_1) <= 1e-8 * e_1
    assert np.max(np.abs(np.abs(np.diag(t)) - np.abs(np.diag(st)))) <= 1e-8 * abs(st[0, 0])


def test_nccl_plumbing_world1(ctx, monkeypatch):
    """The NCCL backend on the one GPU this run has: a world-1 communicator (CORU_NCCL_WORLD1)
    routes the A^T-product and core all-reduces through ncclAllReduce; results must equal the
    communicator-free run bit for bit (a 1-rank sum is the identity)."""
    import torch
    import paper_1810_07323_b200 as cg
    monkeypatch.setenv("CORU_NCCL_WORLD1", "1")
    rng = np.random.default_rng(5)
    a = torch.from_numpy(rng.standard_normal((3000, 1500)) * (0.99 ** np.arange(1500))).cuda()
    ref = [cg.corutv(a, 40, 1, v, seed=cg.RngSeed(42, 0), ctx=ctx) for v in (cg.DVariant.exact, cg.DVariant.approx)]
    c2 = cg.Context(0)
    c2.init_comm(0, 1, cg.Context.unique_id())
    for v, r in zip((cg.DVariant.exact, cg.DVariant.approx), ref):
        f = cg.corutv(a, 40, 1, v, seed=cg.RngSeed(42, 0), ctx=c2, m_global=3000)
        assert torch.equal(f.u, r.u) and torch.equal(f.t, r.t) and torch.equal(f.v, r.v)
    c2.close()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("decay", [-2.0, -9.0])
def test_sharded_wide_sketch_cholqr2(ctx, world, decay):
    """Wide sketch (d = 136 > 128) row-sharded: the Q1 sketch is factored by CholeskyQR2 over all
    ranks (all-reduced Gram matrices, local triangular solves) — decay -2: the well-conditioned case
    it accepts; decay -9 with q = 1: cond(sketch) ~ 1e27 trips the device-side status and every rank
    falls back to the gated Householder tree with its cross-rank top level. Either way the result
    matches the single-GPU decomposition and replicated outputs are bit-identical across ranks."""
    import torch
    import paper_1810_07323_b200 as cg
    m, n, d, q = 6000, 1200, 136, 1
    rng = np.random.default_rng(world + int(-decay))
    r = 2 * d
    x, _ = np.linalg.qr(rng.standard_normal((m, r)))
    y, _ = np.linalg.qr(rng.standard_normal((n, r)))
    a = (x * np.logspace(0, decay, r)) @ y.T + 1e-9 * rng.standard_normal((m, n))
    a_dev = torch.from_numpy(a).cuda()
    single = cg.corutv(a_dev, d, q, seed=cg.RngSeed(42, 0), ctx=ctx)
    parts = _run_sharded(a_dev, d, q, world)
    for f in parts[1:]:
        assert torch.equal(f.t, parts[0].t) and torch.equal(f.v, parts[0].v)
        assert np.array_equal(f.perm, parts[0].perm)
    u = torch.cat([f.u for f in parts]).cpu().numpy()
    t, v = parts[0].t.cpu().numpy(), parts[0].v.cpu().numpy()
    assert orth_residual(u) <= 1e-12 * d and orth_residual(v) <= 1e-12 * d
    su, st, sv = single.u.cpu().numpy(), single.t.cpu().numpy(), single.v.cpu().numpy()
    e_sh = np.linalg.norm(a - u @ t @ v.T) / np.linalg.norm(a)
    e_1 = np.linalg.norm(a - su @ st @ sv.T) / np.linalg.norm(a)
    assert e_sh <= 1.05 * e_1 + 1e-15
    k = 60  # leading, well-determined part of the spectrum
    assert np.max(np.abs(np.abs(np.diag(t))[:k] - np.abs(np.diag(st))[:k])) <= 1e-8 * abs(st[0, 0])
    again = _run_sharded(a_dev, d, q, world)
    assert torch.equal(again[0].t, parts[0].t)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("m,n,d,q", [(20000, 2000, 110, 1), (6000, 1200, 136, 2)])
def test_sharded_b2_allreduce_per_chunk(ctx, monkeypatch, world, m, n, d, q):
    """The sharded power rounds with the A^T-product issued per 64-column chunk and each chunk's
    all-reduce (plus scatter) on the aux stream under the next chunk's product (the large-message
    schedule, forced here with CORU_B2_OVERLAP=1): the same decomposition as the one-message
    schedule — both reduce identical per-rank partials in rank order."""
    import torch
    import paper_1810_07323_b200 as cg
    rng = np.random.default_rng(m + d + world)
    r = 2 * d
    x, _ = np.linalg.qr(rng.standard_normal((m, r)))
    y, _ = np.linalg.qr(rng.standard_normal((n, r)))
    a_dev = torch.from_numpy((x * np.logspace(0, -2, r)) @ y.T + 1e-7 * rng.standard_normal((m, n))).cuda()
    monkeypatch.setenv("CORU_B2_OVERLAP", "0")
    one = _run_sharded(a_dev, d, q, world)
    monkeypatch.setenv("CORU_B2_OVERLAP", "1")
    per = _run_sharded(a_dev, d, q, world)
    for f in per[1:]:
        assert torch.equal(f.t, per[0].t) and torch.equal(f.v, per[0].v)
    # the chunked product sums over k in a different split order than the full-width one: agree to rounding
    t1, t2 = one[0].t.cpu().numpy(), per[0].t.cpu().numpy()
    assert np.array_equal(one[0].perm, per[0].perm)
    assert np.max(np.abs(np.abs(np.diag(t1)) - np.abs(np.diag(t2)))) <= 1e-9 * abs(t1[0, 0])
    u = torch.cat([f.u for f in per]).cpu().numpy()
    assert orth_residual(u) <= 1e-12 * d
