"""Full-size parity of C4 (fp64 32768^2, d=220, q=2) and C5 (fp32, d=520, q=2; default 32768^2,
--c5-size 65536 for the full config) against the bit-exact oracle and its two floors
(tests/parity_util.py). Runs on the GPU box (minutes of oracle time on all host cores):

    python tools/parity_fullsize.py [--configs C4,C5] [--c5-size 32768] > gpurun_out/r02_parity_fullsize.json

One JSON object per config (A SHA-256, rel-err diff, |diag T| diffs on the determined prefix and
overall, first pivot divergence, flags, both floors, the verdict under the protocol).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C4,C5")
    ap.add_argument("--c5-size", type=int, default=32768)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_1810_07323_b200 as cg
    from parity_util import parity_record
    from workloads import CONFIGS, make_device, sha256
    ctx = cg.Context(0)
    out = {}
    for name in args.configs.split(","):
        c = CONFIGS[name]
        m = n = args.c5_size if name == "C5" else None
        t0 = time.perf_counter()
        a_dev = make_device(name, m=m, n=n)
        torch.cuda.synchronize()
        a = a_dev.cpu().numpy()
        sha = sha256(a)
        f = cg.corutv(a_dev, c.d, c.q, seed=cg.RngSeed(42, 0), ctx=ctx)
        torch.cuda.synchronize()
        del a_dev
        torch.cuda.empty_cache()
        eye = np.eye(c.d)
        u64, v64 = f.u.cpu().numpy().astype(np.float64), f.v.cpu().numpy().astype(np.float64)
        orth = (float(np.linalg.norm(u64.T @ u64 - eye)), float(np.linalg.norm(v64.T @ v64 - eye)))
        rec, ok = parity_record(a, f, c.d, c.q, c.k, dtype=c.dtype, a_sha=sha)
        rec.update(config=f"{name} {a.shape[0]}x{a.shape[1]}", orth_u=orth[0], orth_v=orth[1],
                   seconds=time.perf_counter() - t0, host_threads=os.cpu_count())
        out[f"{name}_{a.shape[0]}x{a.shape[1]}"] = rec
        print(json.dumps({name: rec}), file=sys.stderr, flush=True)
        del a
    print(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
