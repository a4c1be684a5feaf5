"""Host-side costs of one C2 decomposition on the GPU box: Φ generation vs the whole call."""
import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import torch
import paper_1810_07323_b200 as cg
from workloads import make_device
for thr in (1, 4, 8, 16):
    t = time.perf_counter()
    for s in range(10):
        cg.gaussian(4000, 60, cg.RngSeed(42, s), threads=thr)
    print(f"phi 4000x60 threads={thr}: {(time.perf_counter() - t) / 10 * 1e3:.3f} ms")
ctx = cg.Context(0)
a = make_device("C2q1")
for i in range(3):
    cg.corutv(a, 60, 1, seed=cg.RngSeed(42, i), ctx=ctx)
torch.cuda.synchronize()
t = time.perf_counter()
for i in range(20):
    cg.corutv(a, 60, 1, seed=cg.RngSeed(42, 100 + i), ctx=ctx)
torch.cuda.synchronize()
print(f"corutv C2q1 wall: {(time.perf_counter() - t) / 20 * 1e3:.3f} ms")
