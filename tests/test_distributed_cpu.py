"""Multi-rank (row-sharded) CoR-UTV logic on CPU: world_size 2, gloo backend.

Restates, step for step, the sharded branch of the product's orchestration
(paper_1810_07323_b200/csrc/capi.cu, `run()` with world > 1) with the CPU oracle
for the local math and torch.distributed (gloo) for the collectives:
  rows of A split by the product's coru_shard_rows; Φ from the product's host generator;
  B2 = allreduce_sum(A_g^T B1_g); QR(B1) = local tree root R_g -> allgather -> redundant top QR
  -> Q1_g = Q_local_g · Q_top[g]; Q2, QRCP and V redundant; D = allreduce_sum(Q1_g^T A_g Q2).
The result must reproduce the single-process oracle decomposition (up to rounding) and be
bit-identical across ranks where the product promises it (T, V, perm, the flag).
"""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def _allgather(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return np.concatenate([o.numpy() for o in out], axis=0)


def sharded_corutv(a_full, d, q, seed, stream, rank, world):
    """One rank of the row-sharded algorithm; returns (U_g, T, V, perm, warn, rows)."""
    import paper_1810_07323_b200 as cg
    from oracle import Oracle
    o = Oracle()
    m, n = a_full.shape
    r0, rows = cg.shard_rows(m, rank, world)
    a = np.ascontiguousarray(a_full[r0:r0 + rows])
    phi = cg.gaussian(n, d, cg.RngSeed(seed, stream))          # replicated, bit-exact
    b2 = phi
    for _ in range(q + 1):
        b1 = o.matmul(a, b2)                                     # local rows
        b2 = _allreduce(o.matmul_tn(a, b1))                      # sum_g A_g^T B1_g
    # TSQR of B1 across ranks: local factor, all-gather the d x d roots, redundant top QR.
    q_loc, r_loc = o.householder_qr(b1)
    stack = _allgather(r_loc)                                    # (world*d) x d
    q_top, r1 = o.householder_qr(stack)
    q1 = q_loc @ q_top[rank * d:(rank + 1) * d]
    warn = abs(r1[d - 1, d - 1]) <= 1e-14 * abs(r1[0, 0])
    q2, _ = o.householder_qr(b2)                                  # replicated
    core = _allreduce(q1.T @ (a @ q2))                           # D = sum_g Q1_g^T A_g Q2
    qm, t, perm = o.qrcp(core)
    return q1 @ qm, t, q2[:, perm], perm, warn, (r0, rows)


def _worker(rank, world, init_file, a_full, d, q, seed, out_dir):
    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank, world_size=world)
    try:
        u, t, v, perm, warn, (r0, rows) = sharded_corutv(a_full, d, q, seed, 0, rank, world)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), u=u, t=t, v=v, perm=perm, warn=warn, r0=r0, rows=rows)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,d,q", [(400, 300, 20, 1), (1001, 200, 25, 0), (600, 600, 30, 2)])
def test_row_sharded_matches_single_process(tmp_path, oracle, m, n, d, q):
    rng = np.random.default_rng(m + n + d)
    x, _ = np.linalg.qr(rng.standard_normal((m, 60)))
    y, _ = np.linalg.qr(rng.standard_normal((n, 60)))
    # mild decay: the q = 2 sketch stays well conditioned, so the split must agree to rounding
    a = (x * (0.95 ** np.arange(60))) @ y.T + 1e-6 * rng.standard_normal((m, n))
    world = 2
    init_file = os.path.join(tempfile.mkdtemp(), "pg_init")
    mp.start_processes(_worker, args=(world, init_file, a, d, q, 42, str(tmp_path)), nprocs=world,
                       join=True, start_method="fork")
    res = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    # replicated outputs are bit-identical across ranks
    for key in ("t", "v", "perm", "warn"):
        assert np.array_equal(res[0][key], res[1][key]), key
    u = np.concatenate([r["u"] for r in res], axis=0)
    assert u.shape == (m, d)
    t, v = res[0]["t"], res[0]["v"]
    ref = oracle.corutv(a, d, q, seed=42)
    e_sh = np.linalg.norm(a - u @ t @ v.T) / np.linalg.norm(a)
    e_ref = np.linalg.norm(a - ref.u @ ref.t @ ref.v.T) / np.linalg.norm(a)
    assert abs(e_sh - e_ref) <= 1e-8 * e_ref + 1e-14
    assert np.max(np.abs(np.abs(np.diag(t)) - np.abs(np.diag(ref.t)))) <= 1e-10 * abs(ref.t[0, 0])
    assert np.array_equal(res[0]["perm"], ref.perm)
    assert np.linalg.norm(u.T @ u - np.eye(d)) <= 1e-12 * d
    assert np.all(np.diag(np.linalg.qr(u)[1]) != 0)


def test_shard_rows_cover_all_rows_evenly():
    import paper_1810_07323_b200 as cg
    for m in (4000, 200000, 32768, 65536, 1001):
        for world in (2, 4, 8):
            spans = [cg.shard_rows(m, r, world) for r in range(world)]
            assert [s[0] for s in spans] == [m * r // world for r in range(world)]
            assert sum(s[1] for s in spans) == m


def sharded_corutv_wide(a_full, d, q, seed, stream, rank, world, chunk_cols=64):
    """The wide-sketch (d > 128) variant of the sharded orchestration (capi.cu run_impl, sharded
    branch with ts1.chol): B2 all-reduced per 64-column chunk, Q1 by CholeskyQR2 over all ranks —
    both Gram matrices all-reduced, R1 = R2·R1', Q1_g = B1_g R1'^{-1} R2^{-1} — no all-gather."""
    import paper_1810_07323_b200 as cg
    from oracle import Oracle
    o = Oracle()
    m, n = a_full.shape
    r0, rows = cg.shard_rows(m, rank, world)
    a = np.ascontiguousarray(a_full[r0:r0 + rows])
    b2 = cg.gaussian(n, d, cg.RngSeed(seed, stream))
    for _ in range(q + 1):
        b1 = o.matmul(a, b2)
        nxt = np.empty((n, d))
        for c0 in range(0, d, chunk_cols):                      # one message per column chunk
            nxt[:, c0:c0 + chunk_cols] = _allreduce(o.matmul_tn(a, np.ascontiguousarray(b1[:, c0:c0 + chunk_cols])))
        b2 = nxt
    g1 = _allreduce(b1.T @ b1)
    r1a = np.linalg.cholesky(g1).T
    q1a = np.linalg.solve(r1a.T, b1.T).T
    g2 = _allreduce(q1a.T @ q1a)
    r2 = np.linalg.cholesky(g2).T
    q1 = np.linalg.solve(r2.T, q1a.T).T
    r1 = r2 @ r1a
    warn = abs(r1[d - 1, d - 1]) <= 1e-14 * abs(r1[0, 0])
    q2, _ = o.householder_qr(b2)
    core = _allreduce(q1.T @ (a @ q2))
    qm, t, perm = o.qrcp(core)
    return q1 @ qm, t, q2[:, perm], perm, warn, (r0, rows)


def _worker_wide(rank, world, init_file, a_full, d, q, seed, out_dir):
    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank, world_size=world)
    try:
        u, t, v, perm, warn, (r0, rows) = sharded_corutv_wide(a_full, d, q, seed, 0, rank, world)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), u=u, t=t, v=v, perm=perm, warn=warn, r0=r0, rows=rows)
    finally:
        dist.destroy_process_group()


def test_row_sharded_wide_sketch_cholqr2(tmp_path, oracle):
    """d = 136 > 128, world 2 (gloo): CholeskyQR2 with all-reduced Gram matrices and chunked B2
    all-reduces reproduce the single-process oracle decomposition; replicated outputs bit-identical."""
    m, n, d, q = 900, 400, 136, 1
    rng = np.random.default_rng(m + n + d)
    x, _ = np.linalg.qr(rng.standard_normal((m, 2 * d)))
    y, _ = np.linalg.qr(rng.standard_normal((n, 2 * d)))
    a = (x * np.logspace(0, -1.5, 2 * d)) @ y.T + 1e-7 * rng.standard_normal((m, n))
    world = 2
    init_file = os.path.join(tempfile.mkdtemp(), "pg_init")
    mp.start_processes(_worker_wide, args=(world, init_file, a, d, q, 42, str(tmp_path)), nprocs=world,
                       join=True, start_method="fork")
    res = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    for key in ("t", "v", "perm", "warn"):
        assert np.array_equal(res[0][key], res[1][key]), key
    u = np.concatenate([r["u"] for r in res], axis=0)
    t, v = res[0]["t"], res[0]["v"]
    ref = oracle.corutv(a, d, q, seed=42)
    e_sh = np.linalg.norm(a - u @ t @ v.T) / np.linalg.norm(a)
    e_ref = np.linalg.norm(a - ref.u @ ref.t @ ref.v.T) / np.linalg.norm(a)
    assert abs(e_sh - e_ref) <= 1e-7 * e_ref + 1e-14
    k = 60
    assert np.max(np.abs(np.abs(np.diag(t))[:k] - np.abs(np.diag(ref.t))[:k])) <= 1e-9 * abs(ref.t[0, 0])
    assert np.linalg.norm(u.T @ u - np.eye(d)) <= 1e-12 * d
