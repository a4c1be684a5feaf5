"""TSQR tree-shape sweep: time coru_tsqr_f64_dev (factor + explicit Q) on an m x d sketch for a set
of block-row targets (CORU_TSQR_TARGET, read by plan_tsqr on every call).

    python tools/tsqr_sweep.py [--m 200000] [--d 110] [--targets 512,768,1024,1352,2048]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=200000)
    ap.add_argument("--d", type=int, default=110)
    ap.add_argument("--targets", default="0,512,768,1024,1352,1400,2048,2704")
    ap.add_argument("--decay", type=float, default=3.0 / 20.0, help="column scale 10^(-decay*j)")
    args = ap.parse_args()
    import torch
    import paper_1810_07323_b200 as cg
    ctx = cg.Context(0)
    g = torch.Generator(device="cuda").manual_seed(1)
    b = torch.randn(args.m, args.d, dtype=torch.float64, device="cuda", generator=g)
    b *= 10.0 ** (-args.decay * torch.arange(args.d, dtype=torch.float64, device="cuda"))
    for t in [int(x) for x in args.targets.split(",")]:
        if t:
            os.environ["CORU_TSQR_TARGET"] = str(t)
        else:
            os.environ.pop("CORU_TSQR_TARGET", None)
        cg.tsqr(b, ctx=ctx)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n = 5
        for _ in range(n):
            q, r = cg.tsqr(b, ctx=ctx)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / n * 1e3
        err = float(torch.linalg.norm(q @ r - b) / torch.linalg.norm(b))
        print(f"target {t or 'default':>8}: {ms:8.3f} ms  (QR-B rel {err:.1e})", flush=True)


if __name__ == "__main__":
    main()
