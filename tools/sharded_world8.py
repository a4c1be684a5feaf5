"""World-8 run of the row-sharded orchestration on ONE B200: the ranks are host
threads joined by the in-process collective group (coru_threadcomm), so the eight ranks share the
GPU — wall times say nothing about scaling; what the record shows is that the d > 128 sharded path
(CholeskyQR2 with all-reduced Gram matrices, per-chunk B2 all-reduce) runs at the C4 / C5 shapes,
what it agrees with (the single-GPU decomposition), and how each rank's time splits into its own
A-passes and everything else (replicated Q2 tree / QRCP, collectives, waiting for the other ranks).

    python tools/sharded_world8.py [--configs C4,C5] [--c5-size 32768] > gpurun_out/r02_sharded_world8.json
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def run_sharded(cg, torch, a_dev, d, q, world):
    m, n = a_dev.shape
    group = cg.ThreadGroup(world)
    out, prof, wall, err = [None] * world, [None] * world, [0.0] * world, []

    def worker(rank):
        try:
            ctx = cg.Context(0)
            ctx.init_threadcomm(group, rank)
            r0, rows = cg.shard_rows(m, rank, world)
            a_r = a_dev[r0:r0 + rows]
            ctx.set_profiling(True)
            t0 = time.perf_counter()
            out[rank] = cg.corutv(a_r, d, q, seed=cg.RngSeed(42, 0), ctx=ctx, m_global=m)
            torch.cuda.synchronize()
            wall[rank] = time.perf_counter() - t0
            prof[rank] = ctx.profile_apass()
        except Exception as e:  # noqa: BLE001
            err.append(f"rank {rank}: {e!r}")

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise RuntimeError(err)
    return out, prof, wall


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C4,C5")
    ap.add_argument("--c5-size", type=int, default=32768)
    ap.add_argument("--world", type=int, default=8)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_1810_07323_b200 as cg
    from workloads import CONFIGS, make_device
    res = {}
    for name in args.configs.split(","):
        c = CONFIGS[name]
        size = args.c5_size if name == "C5" else None
        a = make_device(name, m=size, n=size)
        torch.cuda.synchronize()
        ctx = cg.Context(0)
        t0 = time.perf_counter()
        single = cg.corutv(a, c.d, c.q, seed=cg.RngSeed(42, 0), ctx=ctx)
        torch.cuda.synchronize()
        t_single = time.perf_counter() - t0
        ctx.close()
        run_sharded(cg, torch, a, c.d, c.q, args.world)  # warm-up (arenas, plans)
        parts, prof, wall = run_sharded(cg, torch, a, c.d, c.q, args.world)
        u = torch.cat([f.u for f in parts])
        d_sh, d_1 = parts[0].t.double().diagonal().abs(), single.t.double().diagonal().abs()
        dt = (d_sh - d_1).abs().max().item()
        kk = c.k // 2  # leading half of the target rank: well separated from the noise floor
        dt_lead = (d_sh - d_1)[:kk].abs().max().item()
        from parity_util import rel_err
        e_sh = rel_err(a, u, parts[0].t, parts[0].v)
        e_1 = rel_err(a, single.u, single.t, single.v)
        same = all(torch.equal(f.t, parts[0].t) and torch.equal(f.v, parts[0].v) for f in parts[1:])
        eye = torch.eye(c.d, dtype=torch.float64, device=u.device)
        orth = float(torch.linalg.norm(u.double().T @ u.double() - eye))
        res[f"{name}_{a.shape[0]}x{a.shape[1]}"] = {
            "world": args.world, "backend": "coru_threadcomm (one B200, ranks = host threads)",
            "d": c.d, "q": c.q, "dtype": c.dtype,
            "single_gpu_wall_s": t_single, "sharded_wall_s_max_over_ranks": max(wall),
            "per_rank": [{"rank": r, "wall_s": wall[r], "apass_ms": prof[r]["ms"], "apass_launches": prof[r]["launches"],
                          "other_ms": wall[r] * 1e3 - prof[r]["ms"]} for r in range(args.world)],
            "replicated_outputs_bit_identical_across_ranks": bool(same),
            "absdiag_T_maxdiff_vs_single_gpu": dt, "absdiag_T_maxdiff_leading_half_k": dt_lead,
            "t11": float(single.t[0, 0].abs()), "rel_err_sharded": e_sh, "rel_err_single_gpu": e_1,
            "pivots_equal_single_gpu": bool(np.array_equal(parts[0].perm, single.perm)),
            "orth_u": orth,
        }
        print(json.dumps({name: res[f"{name}_{a.shape[0]}x{a.shape[1]}"]}), file=sys.stderr, flush=True)
        del a, parts, single, u
        torch.cuda.empty_cache()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
