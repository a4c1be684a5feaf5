"""Where the C2q1 e2e (host-buffer) call spends its time: H2D of A alone, D2H of the outputs, the
device decomposition, and the full host entry (tooling)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1810_07323_b200 as cg
from workloads import make_host
a = make_host("C2q1")
ctx = cg.Context(0)
ah = torch.from_numpy(a).pin_memory()
ad = torch.empty_like(ah, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(3):
    ad.copy_(ah, non_blocking=True)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    ev[0].record(); ad.copy_(ah, non_blocking=True); ev[1].record(); torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
print("H2D 128 MB pinned: %.3f ms (%.1f GB/s)" % (np.median(ts), 128e6 / np.median(ts) / 1e6))
u = np.empty((4000, 60)); t = np.empty((60, 60)); v = np.empty((4000, 60))
ahn = ah.numpy()
for _ in range(3):
    cg.corutv(ahn, 60, 1, seed=cg.RngSeed(42, 0), ctx=ctx)
t0 = time.perf_counter()
for s in range(10):
    cg.corutv(ahn, 60, 1, seed=cg.RngSeed(42, s), ctx=ctx)
print("host entry (numpy wrapper, pinned A): %.3f ms" % ((time.perf_counter() - t0) / 10 * 1e3))
t0 = time.perf_counter()
for s in range(10):
    f = cg.corutv(ad, 60, 1, seed=cg.RngSeed(42, s), ctx=ctx)
torch.cuda.synchronize()
print("device entry: %.3f ms" % ((time.perf_counter() - t0) / 10 * 1e3))
