"""GPU alm_rpca vs the reference fixtures: per-case discrepancy report (JSON lines)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1810_07323_b200 as cg  # noqa: E402
from golden import rpca_cases  # noqa: E402

ctx = cg.Context(0)
for c in rpca_cases():
    cfg = cg.RpcaConfig(**{k: v for k, v in c["cfg"].items() if k != "thresholding"},
                        corutv_thresholding=cg.CorutvThresholding(c["cfg"]["thresholding"]))
    t = time.time()
    try:
        r = cg.alm_rpca(c["M"], cfg, cg.RngSeed(c["seed"], c["stream"]), ctx=ctx)
    except Exception as e:  # report and continue
        print(json.dumps(dict(name=c["name"], error=repr(e))), flush=True)
        continue
    dt = time.time() - t
    n = min(len(r.residuals), len(c["residuals"]))
    rr = np.asarray(r.residuals[:n]); cr = c["residuals"][:n]
    print(json.dumps(dict(
        name=c["name"], sec=round(dt, 3), it=(r.iterations, c["iterations"]), rank=(r.rank_l, c["rank_l"]),
        s_l0=(r.s_l0, c["s_l0"]), conv=(r.converged, c["converged"]), clamped=(r.ell_clamped, c["ell_clamped"]),
        l_rel=float(np.linalg.norm(r.l - c["L"]) / max(np.linalg.norm(c["L"]), 1e-300)),
        s_rel=float(np.linalg.norm(r.s - c["S"]) / max(np.linalg.norm(c["S"]), 1e-300)),
        supp_diff=int(np.sum((r.s != 0) != (c["S"] != 0))),
        zeta_rel=float(np.max(np.abs(rr - cr) / cr)) if n else None)), flush=True)
