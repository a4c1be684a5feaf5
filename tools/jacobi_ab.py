"""Time the one-CTA Jacobi SVD (coru_svd_f64_dev) on RPCA-like and graded cores; run under
CORU_JACOBI_VARIANT=0/1/2 to compare launch shapes."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_1810_07323_b200 as cg  # noqa: E402

ctx = cg.Context(0)
rng = np.random.default_rng(0)
out = {}
for d, kind in ((60, "graded"), (80, "rpca"), (110, "graded"), (110, "rpca")):
    if kind == "rpca":
        x, _ = np.linalg.qr(rng.standard_normal((d, d)))
        y, _ = np.linalg.qr(rng.standard_normal((d, d)))
        s = np.concatenate([np.linspace(100, 50, d // 2), 1e-3 * rng.random(d - d // 2)])
    else:
        x, _ = np.linalg.qr(rng.standard_normal((d, d)))
        y, _ = np.linalg.qr(rng.standard_normal((d, d)))
        s = np.arange(1, d + 1, dtype=float) ** -2.0
    a = torch.from_numpy((x * s) @ y.T).cuda()
    for _ in range(3):
        f = cg.svd(a, ctx=ctx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f = cg.svd(a, ctx=ctx)
    e1.record()
    torch.cuda.synchronize()
    err = float(np.max(np.abs(np.sort(f.sigma.cpu().numpy())[::-1] - np.sort(s)[::-1])) / s.max())
    print(f"variant {os.environ.get('CORU_JACOBI_VARIANT', '0')} d={d} {kind}: {e0.elapsed_time(e1) / 10:.3f} ms "
          f"(incl. host sync) sweeps={f.converged} sigma err {err:.1e}", flush=True)
