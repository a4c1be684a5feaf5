"""Layout debugging for the tcgen05 fp32 A-pass (tooling only): structured inputs whose products
identify which A row / K index / X column each output element picked up."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_07323_b200 as cg

ctx = cg.Context(0)
ctx.set_f32_path(ctx.F32_TC)
for op in (0, 1):
    for (Mo, K, N) in [(128, 128, 16), (128, 128, 64), (256, 256, 272)]:
        a = np.zeros((Mo, K), np.float32)
        for i in range(Mo):
            a[i, i % K] = 1.0
        x = (np.arange(K)[:, None] * 1000 + np.arange(N)[None, :]).astype(np.float32)
        if op == 1:
            at = np.ascontiguousarray(a.T)  # K x Mo, op T computes at^T x = a x
            c = cg.gemm(torch.from_numpy(at).cuda(), torch.from_numpy(x).cuda(), op=1, ctx=ctx).cpu().numpy()
        else:
            c = cg.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda(), op=0, ctx=ctx).cpu().numpy()
        want = a @ x
        bad = np.argwhere(c != want)
        print(f"op={op} Mo={Mo} K={K} N={N}: wrong {len(bad)}/{c.size}")
        for (i, j) in bad[:12]:
            v = c[i, j]
            print(f"   C[{i},{j}] = {v:.1f} want {want[i, j]:.1f}  -> krow {v // 1000:.0f} col {v % 1000:.0f}")
        if len(bad):
            rows = sorted(set(int(i) for i, _ in bad))
            print("   bad rows (first 40):", rows[:40])
