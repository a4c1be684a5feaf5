"""Full-size C3 (fp64 200000 x 2000, d = 110, q = 1) against the bit-exact oracle (gpu marker).

A is generated once (tests/workloads.make_device), the GPU decomposes it from HBM with the
reference's Φ (host-exact mode, the default), and the oracle (oracle/coru_oracle.c, bit-identical
to the compiled reference; pinned in test_oracle.py) runs on all host cores on the same bytes,
together with its two floors (tests/parity_util.py). C4 and C5 at full / near-full size run in
tools/parity_fullsize.py (minutes of oracle time) -> profiles/r02_parity_fullsize.json.
"""
import json
import os

import numpy as np
import pytest

from conftest import orth_residual

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _save(name, rec):
    out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")
    if os.path.isdir(out):
        p = os.path.join(out, "parity_fullsize.json")
        data = json.load(open(p)) if os.path.exists(p) else {}
        data[name] = rec
        with open(p, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


def test_c3_fullsize_vs_oracle(ctx):
    import torch
    import paper_1810_07323_b200 as cg
    from parity_util import parity_record
    from workloads import CONFIGS, make_device, sha256
    c = CONFIGS["C3"]
    a_dev = make_device("C3")
    torch.cuda.synchronize()
    a = a_dev.cpu().numpy()
    f = cg.corutv(a_dev, c.d, c.q, seed=cg.RngSeed(42, 0), ctx=ctx)
    u = f.u.cpu().numpy()
    v = f.v.cpu().numpy()
    t = f.t.cpu().numpy()
    del a_dev
    torch.cuda.empty_cache()
    assert np.all(np.tril(t, -1) == 0.0)
    ou, ov = orth_residual(u), orth_residual(v)
    assert ou <= 1e-12 * c.d and ov <= 1e-12 * c.d
    rec, ok = parity_record(a, f, c.d, c.q, c.k, a_sha=sha256(a))
    rec.update(orth_u=ou, orth_v=ov, config="C3 full size")
    _save("C3_200000x2000", rec)
    assert ok["err"] and ok["never_worse"], rec
    assert ok["diag"], rec
    assert ok["flag"], rec
