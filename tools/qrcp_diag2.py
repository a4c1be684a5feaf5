import os, sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1810_07323_b200 as cg
from workloads import make_host
ctx = cg.Context(0)
a = make_host("C4", 4096, 4096)
def run():
    f = cg.corutv(a, 220, 2, seed=cg.RngSeed(42, 0), ctx=ctx)
    return f, np.linalg.norm(a - f.u @ f.t @ f.v.T) / np.linalg.norm(a)
f1, e1 = run()
os.environ["CORU_QRCP_CTA"] = "1"
f2, e2 = run()
print("grid err", e1, "cta err", e2, "perm eq", np.array_equal(f1.perm, f2.perm), "T maxdiff", np.abs(f1.t - f2.t).max(),
      "U maxdiff", np.abs(f1.u - f2.u).max())
print("perm grid", f1.perm[:10], "cta", f2.perm[:10])
del os.environ["CORU_QRCP_CTA"]
ad = torch.from_numpy(a).cuda()
g = cg.corutv(ad, 220, 2, seed=cg.RngSeed(42, 0), ctx=ctx)
print("dev entry T diff vs cta", np.abs(g.t.cpu().numpy() - f2.t).max(), "perm", g.perm[:10])
