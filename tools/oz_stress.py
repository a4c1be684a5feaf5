"""Determinism stress of the Ozaki A-pass kernel: repeated products of the same operands must be
bitwise identical (tooling; CORU_LIB_VARIANT selects an A/B build)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1810_07323_b200 as cg
    ctx = cg.Context(0)
    rng = np.random.default_rng(5)
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    for (m, k, n, op) in [(3000, 2000, 110, 0), (3000, 2000, 110, 1), (20000, 2000, 110, 0), (2048, 4096, 60, 0)]:
        a = torch.from_numpy(rng.standard_normal((k, m) if op else (m, k))).cuda()
        x = torch.zeros((k, n + (n & 1)), dtype=torch.float64, device="cuda")
        x[:, :n] = torch.from_numpy(rng.standard_normal((k, n))).cuda()
        ref = cg.gemm(a, x[:, :n], op=op, ctx=ctx).clone()
        bad = 0
        worst = 0.0
        for _ in range(reps):
            c = cg.gemm(a, x[:, :n], op=op, ctx=ctx)
            if not torch.equal(c, ref):
                bad += 1
                diff = (c - ref).abs()
                worst = max(worst, float(diff.max()))
                idx = torch.nonzero(diff > 0)
                if bad == 1:
                    print("   first mismatch: count", idx.shape[0], "rows", idx[:, 0].unique()[:10].tolist(), "cols",
                          idx[:, 1].unique()[:10].tolist())
        print(f"variant {os.environ.get('CORU_LIB_VARIANT', 'default')} shape {(m, k, n, op)}: {bad}/{reps} mismatching runs, "
              f"max diff {worst:.3e}", flush=True)


if __name__ == "__main__":
    main()
