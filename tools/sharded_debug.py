import faulthandler, sys, threading, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
faulthandler.dump_traceback_later(60, exit=True)
import numpy as np, torch
import paper_1810_07323_b200 as cg
from test_gpu_sharded import _run_sharded
rng = np.random.default_rng(0)
m, n, d, q, world = 3000, 1500, 40, 1, 2
a = torch.from_numpy(rng.standard_normal((m, n))).cuda()
ctx = cg.Context(0)
f = cg.corutv(a, d, q, seed=cg.RngSeed(42, 0), ctx=ctx)
print("single ok", flush=True)
for it in range(3):
    t0 = time.time()
    parts = _run_sharded(a, d, q, world)
    print("run", it, "ok", time.time() - t0, flush=True)
