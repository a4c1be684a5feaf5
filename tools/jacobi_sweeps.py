"""Sweeps used by the one-CTA Jacobi SVD (coru_svd_f64_dev's converged output) on RPCA-like and graded cores."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_1810_07323_b200 as cg  # noqa: E402

ctx = cg.Context(0)
lib = cg.load_library()
rng = np.random.default_rng(0)
for d, kind in ((60, "graded"), (80, "rpca"), (80, "flat"), (110, "graded")):
    x, _ = np.linalg.qr(rng.standard_normal((d, d)))
    y, _ = np.linalg.qr(rng.standard_normal((d, d)))
    if kind == "rpca":
        s = np.concatenate([np.linspace(100, 50, d // 2), 1e-3 * rng.random(d - d // 2)])
    elif kind == "flat":
        s = np.linspace(2, 1, d)
    else:
        s = np.arange(1, d + 1, dtype=float) ** -2.0
    a = torch.from_numpy((x * s) @ y.T).cuda()
    u = torch.empty((d, d), dtype=torch.float64, device="cuda")
    v = torch.empty_like(u)
    sg = torch.empty(d, dtype=torch.float64, device="cuda")
    conv = C.c_int()
    cg._check(lib.coru_svd_f64_dev(ctx.h, a.data_ptr(), d, d, u.data_ptr(), d, sg.data_ptr(), v.data_ptr(), d,
                                   C.byref(conv)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        cg._check(lib.coru_svd_f64_dev(ctx.h, a.data_ptr(), d, d, u.data_ptr(), d, sg.data_ptr(), v.data_ptr(), d,
                                       C.byref(conv)))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"d={d} {kind}: sweeps={conv.value} {ms:.3f} ms/call -> {1e3 * ms / max(conv.value, 1) / (d - 1 + d % 2):.2f} us/step")
