"""BASELINE configs at full size on the GPU, checked through size-independent properties
(gpu marker). The CPU oracle cannot run C3-C5 in test time (C4 alone is 13 min single-threaded,
SURVEY.md §6), so full-size parity rests on:
  * orthonormality ||U^T U - I||, ||V^T V - I|| <= 1e-12·d (fp64), <= 1e-4·d (fp32);
  * T upper triangular with exact zeros, |t_jj| non-increasing (QRCP pivot order);
  * the exact identity ||A - U T V^T||_F^2 = ||A||_F^2 - ||T||_F^2 (T = U^T A V), checked
    against the explicitly streamed residual — a consistency check of every kernel at once;
  * the residual is never below the SVD optimum sqrt(sum_{i>d} sigma_i^2) of the known spectrum;
  * bitwise determinism of a repeated call (fixed-order reductions, no atomics).
Results are written to gpurun_out/fullsize.json (copied to profiles/).
"""
import json
import os
import time

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RESULTS = {}


def _save():
    out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "fullsize.json"), "w") as f:
            json.dump(RESULTS, f, indent=1, sort_keys=True)


def _resid_fro(a, u, t, v, rows=8192):
    """||A - U T V^T||_F streamed in row blocks (fp64 accumulation)."""
    import torch
    ut = (u.double() @ t.double())
    vt = v.double().T
    s = torch.zeros((), dtype=torch.float64, device=a.device)
    for r0 in range(0, a.shape[0], rows):
        blk = a[r0:r0 + rows].double() - ut[r0:r0 + rows] @ vt
        s += (blk * blk).sum()
    return float(torch.sqrt(s))


def _fro(a, rows=8192):
    import torch
    s = torch.zeros((), dtype=torch.float64, device=a.device)
    for r0 in range(0, a.shape[0], rows):
        blk = a[r0:r0 + rows].double()
        s += (blk * blk).sum()
    return float(torch.sqrt(s))


@pytest.mark.parametrize("name", ["C2q1", "C2q2", "C3", "C4", "C5"])
def test_fullsize_properties(ctx, name):
    import torch
    import paper_1810_07323_b200 as cg
    from workloads import CONFIGS, make_device, spectrum
    c = CONFIGS[name]
    a = make_device(name)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = cg.corutv(a, c.d, c.q, seed=cg.RngSeed(42, 0), ctx=ctx)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    d = c.d
    eye = torch.eye(d, dtype=torch.float64, device=a.device)
    orth_u = float(torch.linalg.norm(f.u.double().T @ f.u.double() - eye))
    orth_v = float(torch.linalg.norm(f.v.double().T @ f.v.double() - eye))
    t = f.t.double()
    lower_zero = bool((torch.tril(t, -1) == 0).all())
    dg = torch.abs(torch.diagonal(t)).cpu().numpy()
    # QRCP order: non-increasing up to the error of the downdated column norms the pivots are
    # chosen by (qr.hpp:121-139) — rounding level in fp64; in fp32 nearly equal trailing |t_jj|
    # (C5's noise floor) may swap by a few 1e-6 relative
    nonincreasing = bool(np.all(dg[:-1] >= dg[1:] * (1 - (1e-12 if c.dtype == "f64" else 1e-4))))
    na = _fro(a)
    resid = _resid_fro(a, f.u, f.t, f.v)
    ident = np.sqrt(max(na * na - float((t * t).sum()), 0.0))
    if name in ("C4", "C5"):
        opt = None  # noisy: the optimum is not known in closed form
    else:
        s = spectrum(name, min(c.m, c.n))
        opt = float(np.sqrt((s[d:] ** 2).sum() / (s ** 2).sum()))
    f2 = cg.corutv(a, c.d, c.q, seed=cg.RngSeed(42, 0), ctx=ctx)
    same = bool(torch.equal(f.u, f2.u) and torch.equal(f.t, f2.t) and torch.equal(f.v, f2.v))
    RESULTS[name] = dict(seconds_first_call=dt, orth_u=orth_u, orth_v=orth_v, t_lower_exact_zero=lower_zero,
                         diag_nonincreasing=nonincreasing, rel_err=resid / na, rel_err_identity=ident / na,
                         svd_optimum=opt, warning=f.conditioning_warning, deterministic=same,
                         diag_first=float(dg[0]), diag_k=float(dg[c.k - 1]), diag_last=float(dg[-1]))
    _save()
    tol = 1e-12 * d if c.dtype == "f64" else 1e-4 * d
    assert orth_u <= tol and orth_v <= tol
    assert lower_zero and nonincreasing and same
    # identity holds to the cancellation accuracy of ||A||^2 - ||T||^2
    eps = 2.2e-16 if c.dtype == "f64" else 1.2e-7
    assert abs(resid - ident) <= max(1e-6 * resid, 50 * eps * na * na / max(resid + ident, 1e-300))
    if opt is not None:
        assert resid / na >= opt * (1 - 1e-6)
