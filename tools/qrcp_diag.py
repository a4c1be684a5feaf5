import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1810_07323_b200 as cg
from oracle import Oracle
o = Oracle(); ctx = cg.Context(0)
def check(a, tag):
    t = torch.from_numpy(a).cuda()
    q, r, perm = cg.qrcp(t, ctx=ctx)
    q, r = q.cpu().numpy(), r.cpu().numpy()
    qo, ro, po = o.qrcp(np.ascontiguousarray(a))
    print(tag, "perm_eq", np.array_equal(perm, po), "first diff", np.argmax(perm != po) if not np.array_equal(perm, po) else -1,
          "recon", np.linalg.norm(q @ r - a[:, perm]) / np.linalg.norm(a), "orth", np.linalg.norm(q.T @ q - np.eye(len(q))))
rng = np.random.default_rng(0)
check(rng.standard_normal((220, 220)), "randn220")
big = rng.standard_normal((220, 224)); check(big[:, :220], "strided220")
from workloads import make_host
a = make_host("C4", 4096, 4096)
sb = cg.sketch_bases(a, 220, 2, cg.RngSeed(42, 0), ctx=ctx)
D = sb.q1.T @ a @ sb.q2
check(D, "C4core")
s = np.linalg.svd(D, compute_uv=False); print("core sv", s[:3], s[-3:])
