"""Time the approx-D pinv kernel (Jacobi SVD + assembly) on cores of the config widths."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1810_07323_b200 as cg
ctx = cg.Context(0)
for n, decay in [(25, 0.9), (60, 0.75), (60, 1.0), (110, 0.9), (220, 0.97), (520, 0.99)]:
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) * (decay ** np.arange(n))
    ad = torch.from_numpy(a).cuda()
    cg.pinv(ad, ctx=ctx)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 5 if n < 200 else 2
    for _ in range(reps):
        p, sw = cg.pinv(ad, ctx=ctx)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    err = np.linalg.norm(p.cpu().numpy() - np.linalg.pinv(a)) / np.linalg.norm(np.linalg.pinv(a))
    print(f"n={n} decay={decay} sweeps={sw} ms={dt*1e3:.3f} rel_err_vs_numpy={err:.2e}", flush=True)
