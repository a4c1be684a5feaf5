"""A/B of the host-entry upload pipeline (CORU_NO_UPLOAD_PIPE) on C2q1, interleaved (tooling)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1810_07323_b200 as cg
from workloads import make_host
a = torch.from_numpy(make_host("C2q1")).pin_memory().numpy()
ctx = cg.Context(0)
res = {"pipe": [], "nopipe": []}
for rep in range(6):
    for mode in ("pipe", "nopipe"):
        if mode == "nopipe": os.environ["CORU_NO_UPLOAD_PIPE"] = "1"
        else: os.environ.pop("CORU_NO_UPLOAD_PIPE", None)
        cg.corutv(a, 60, 1, seed=cg.RngSeed(42, 0), ctx=ctx)
        t0 = time.perf_counter()
        for s in range(5):
            cg.corutv(a, 60, 1, seed=cg.RngSeed(42, s), ctx=ctx)
        res[mode].append((time.perf_counter() - t0) / 5 * 1e3)
for k, v in res.items():
    print(k, "median %.3f ms  min %.3f" % (np.median(v), min(v)))
