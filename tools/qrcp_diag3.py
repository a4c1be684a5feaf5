import os, sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1810_07323_b200 as cg
from workloads import make_host
a = make_host("C4", 4096, 4096)
def run(tag, wide=True, env=None):
    if env: os.environ[env] = "1"
    ctx = cg.Context(0); ctx.set_wide_qr(wide)
    for _ in range(3):
        f = cg.corutv(a, 220, 2, seed=cg.RngSeed(42, 0), ctx=ctx)
        print(tag, "err %.6f" % (np.linalg.norm(a - f.u @ f.t @ f.v.T) / np.linalg.norm(a)), f.perm[:6], flush=True)
    if env: del os.environ[env]
run("default")
run("early", env="CORU_QR1_EARLY")
run("nowide", wide=False)
run("ctaqrcp", env="CORU_QRCP_CTA")
