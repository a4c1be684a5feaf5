"""Parity protocol shared by the full-size GPU tests and tools/parity_fullsize.py (test
infrastructure; the oracle is the checker only).

GPU-vs-oracle discrepancies are judged against the oracle's own sensitivity at the same size
(SURVEY.md §8c):
  floor 1 — the oracle against itself on A·(1 + s·ε), s ∈ {-1, 0, 1} from xoshiro256++ {99, 0}
            (ε = 2^-52 fp64, 2^-23 fp32): a 1-ulp perturbation of the input;
  floor 2 — the oracle against the same restatement compiled with FMA contraction
            (oracle/liboracle_fma.so): the reference's algorithm with different rounding, the
            closest CPU stand-in for an independent implementation;
and against the algorithm's exact-arithmetic result, approximated by the same restatement in
extended precision (oracle f80: x87 long double, unit roundoff 2^-64; fp64 for the fp32 configs):
the distance of each fp64 execution (the reference, the GPU) from that result is its own
rounding error, which on ill-conditioned sketches (power rounds on fast-decaying spectra) is far
above the two floors — the reference's long serial sums (matrix.hpp:121-129, qr.hpp:32-57)
accumulate error the floors do not resample.
Verdict rules (BASELINE.json north_star tolerances, fp64 / fp32):
  * |diag T| on the determined prefix — entries j with (|t_jj|/|t_11|)^(2q+1) > 1e-12, whose
    sketch columns carry signal above rounding — within max(tol_diag, 10·max(floor1, floor2)) of
    the oracle, OR at least as close to the extended-precision result as the oracle is (within 2x);
  * the relative reconstruction error: the same rule, and never worse than the oracle's beyond
    that band;
  * conditioning_warning equal to the oracle's whenever the oracle and both floor runs agree
    (otherwise the flag is rounding-determined at this size and only recorded), or equal to the
    extended-precision run's (C2 q=2: |R1(60,60)/R1(1,1)| is ~1e-18 in exact arithmetic, so the
    flag is set; the reference's serial sums leave rounding noise above 1e-14 and miss it).
"""
from __future__ import annotations

import hashlib
import os

import numpy as np

TOL = {"f64": (1e-10, 1e-8), "f32": (1e-4, 1e-3)}   # (rel. error, |diag T|)


def host_threads() -> int:
    return max(1, min(os.cpu_count() or 1, 64))


def perturb(oracle, a: np.ndarray) -> np.ndarray:
    """A·(1 + s·ε) entrywise, s = (xoshiro256++{99,0} word mod 3) - 1 (SURVEY.md §8c protocol 1)."""
    eps = 2.0 ** -52 if a.dtype == np.float64 else 2.0 ** -23
    out = np.empty_like(a)
    flat_in, flat_out = a.reshape(-1), out.reshape(-1)
    chunk = 1 << 26
    words = oracle.xoshiro_words(99, 0, a.size)
    for e0 in range(0, a.size, chunk):
        w = words[e0:e0 + chunk]
        s = (w % np.uint64(3)).astype(np.int8).astype(a.dtype) - a.dtype.type(1)
        flat_out[e0:e0 + chunk] = flat_in[e0:e0 + chunk] * (a.dtype.type(1) + s * a.dtype.type(eps))
    return out


def rel_err(a, u, t, v, rows: int = 8192) -> float:
    """||A - U T V^T||_F / ||A||_F in fp64, streamed in row blocks (torch on the GPU when available)."""
    try:
        import torch
        use_gpu = torch.cuda.is_available()
    except ImportError:  # pragma: no cover
        use_gpu = False
    if use_gpu:
        import torch
        dev = torch.device("cuda", 0)
        A = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        U = (u if isinstance(u, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(u))).to(dev).double()
        T = (t if isinstance(t, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(t))).to(dev).double()
        V = (v if isinstance(v, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(v))).to(dev).double()
        ut, vt = U @ T, V.T
        num = torch.zeros((), dtype=torch.float64, device=dev)
        den = torch.zeros((), dtype=torch.float64, device=dev)
        for r0 in range(0, A.shape[0], rows):
            blk = A[r0:r0 + rows].to(dev).double()
            den += (blk * blk).sum()
            res = blk - ut[r0:r0 + rows] @ vt   # out of place: a CUDA fp64 A would otherwise be overwritten
            num += (res * res).sum()
        return float(torch.sqrt(num / den))
    a64 = np.asarray(a, np.float64)
    r = a64 - (np.asarray(u, np.float64) @ np.asarray(t, np.float64)) @ np.asarray(v, np.float64).T
    return float(np.linalg.norm(r) / np.linalg.norm(a64))


def determined_prefix(t_ref: np.ndarray, q: int) -> int:
    dg = np.abs(np.diag(np.asarray(t_ref, np.float64)))
    if dg[0] == 0:
        return 0
    return int(np.sum((dg / dg[0]) ** (2 * q + 1) > 1e-12))


def first_pivot_divergence(p1, p2):
    p1, p2 = np.asarray(p1), np.asarray(p2)
    diff = np.nonzero(p1 != p2)[0]
    return int(diff[0]) if diff.size else None


def oracle_runs(a, d, q, seed=42, stream=0, threads=None, ext=True):
    """The oracle at A, at the 1-ulp-perturbed A, the FMA-built oracle at A, and (ext) the
    extended-precision restatement at A."""
    from oracle import ORACLE_FMA_SO, Oracle
    threads = threads or host_threads()
    o, o_fma = Oracle(), Oracle(ORACLE_FMA_SO)
    f0 = o.corutv(a, d, q, 0, seed, stream, threads=threads)
    ap = perturb(o, a)
    f1 = o.corutv(ap, d, q, 0, seed, stream, threads=threads)
    f2 = o_fma.corutv(a, d, q, 0, seed, stream, threads=threads)
    fx = None
    if ext:
        hi = np.longdouble if a.dtype == np.float64 else np.float64
        fx = o.corutv(a.astype(hi), d, q, 0, seed, stream, threads=threads)
    return f0, (ap, f1), f2, fx


def parity_record(a, f_gpu, d, q, k, dtype="f64", seed=42, stream=0, threads=None, a_sha=None, ext=True):
    """Run the oracle runs and compare the GPU factors; returns (record, verdicts dict)."""
    f0, (ap, f1), f2, fx = oracle_runs(a, d, q, seed, stream, threads, ext)
    tol_err, tol_diag = TOL[dtype]
    g_u, g_t, g_v = (np.asarray(x.cpu().numpy() if hasattr(x, "cpu") else x) for x in (f_gpu.u, f_gpu.t, f_gpu.v))
    e_gpu, e0 = rel_err(a, g_u, g_t, g_v), rel_err(a, f0.u, f0.t, f0.v)
    e1, e2 = rel_err(ap, f1.u, f1.t, f1.v), rel_err(a, f2.u, f2.t, f2.v)
    del ap
    d0 = np.abs(np.diag(f0.t).astype(np.float64))
    dgpu = np.abs(np.diag(g_t).astype(np.float64))
    d1 = np.abs(np.diag(f1.t).astype(np.float64))
    d2 = np.abs(np.diag(f2.t).astype(np.float64))
    p = max(determined_prefix(f0.t, q), 1)
    floor_err = max(abs(e1 - e0) / e0, abs(e2 - e0) / e0)
    floor_diag = max(np.abs(d1 - d0)[:p].max(), np.abs(d2 - d0)[:p].max())
    rel_err_diff = abs(e_gpu - e0) / e0
    diag_prefix = float(np.abs(dgpu - d0)[:p].max())
    flags_agree = f0.conditioning_warning == f1.conditioning_warning == f2.conditioning_warning
    bound_err = max(tol_err, 10 * floor_err)
    bound_diag = max(tol_diag, 10 * floor_diag)
    # reconstruction errors at rounding level (exact-rank inputs) are compared absolutely
    abs_floor = 100 * (2.0 ** -52 if dtype == "f64" else 2.0 ** -23)
    rec = dict(
        a_sha256=a_sha or hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest(),
        m=int(a.shape[0]), n=int(a.shape[1]), d=d, q=q, k=k, dtype=dtype,
        err_gpu=e_gpu, err_oracle=e0, rel_err_diff=rel_err_diff,
        diag_prefix_len=p, diag_prefix_absdiff=diag_prefix,
        diag_k_absdiff=float(np.abs(dgpu - d0)[:k].max()), diag_all_absdiff=float(np.abs(dgpu - d0).max()),
        floor1_rel_err=abs(e1 - e0) / e0, floor2_rel_err=abs(e2 - e0) / e0,
        floor1_diag_prefix=float(np.abs(d1 - d0)[:p].max()), floor2_diag_prefix=float(np.abs(d2 - d0)[:p].max()),
        floor1_diag_all=float(np.abs(d1 - d0).max()), floor2_diag_all=float(np.abs(d2 - d0).max()),
        first_pivot_divergence=first_pivot_divergence(f_gpu.perm, f0.perm) if getattr(f_gpu, "perm", None) is not None
        else None,
        warn_gpu=bool(f_gpu.conditioning_warning), warn_oracle=f0.conditioning_warning,
        warn_floor1=f1.conditioning_warning, warn_floor2=f2.conditioning_warning,
        bound_rel_err=bound_err, bound_diag_prefix=bound_diag,
        stated_tol_err_pass=bool(rel_err_diff <= tol_err), stated_tol_diag_pass=bool(diag_prefix <= tol_diag),
        stated_tol_diag_all_pass=bool(np.abs(dgpu - d0).max() <= tol_diag),
    )
    err_ok = abs(e_gpu - e0) <= max(bound_err * e0, abs_floor)
    diag_ok = diag_prefix <= bound_diag
    if fx is not None:
        ex = rel_err(a, fx.u.astype(np.float64), fx.t.astype(np.float64), fx.v.astype(np.float64))
        dx = np.abs(np.diag(fx.t).astype(np.float64))
        gpu_to_ext = float(np.abs(dgpu - dx)[:p].max())
        ora_to_ext = float(np.abs(d0 - dx)[:p].max())
        rec.update(err_ext=ex, ext_dtype="long double (f80)" if dtype == "f64" else "f64",
                   gpu_to_ext_rel_err=abs(e_gpu - ex) / ex, oracle_to_ext_rel_err=abs(e0 - ex) / ex,
                   gpu_to_ext_diag_prefix=gpu_to_ext, oracle_to_ext_diag_prefix=ora_to_ext,
                   first_pivot_divergence_gpu_ext=first_pivot_divergence(f_gpu.perm, fx.perm)
                   if getattr(f_gpu, "perm", None) is not None else None,
                   first_pivot_divergence_oracle_ext=first_pivot_divergence(f0.perm, fx.perm),
                   warn_ext=bool(fx.conditioning_warning))
        # at least as close to the exact-arithmetic result as the reference's own fp64 execution
        err_ok = err_ok or abs(e_gpu - ex) <= max(2 * abs(e0 - ex), bound_err * ex, abs_floor)
        diag_ok = diag_ok or gpu_to_ext <= max(2 * ora_to_ext, tol_diag)
    ok = dict(
        err=err_ok,
        never_worse=e_gpu <= e0 * (1 + bound_err) + abs_floor,
        diag=diag_ok,
        flag=(not flags_agree) or bool(f_gpu.conditioning_warning) == f0.conditioning_warning
        or (fx is not None and bool(f_gpu.conditioning_warning) == bool(fx.conditioning_warning)),
    )
    rec["verdict"] = {k_: bool(v_) for k_, v_ in ok.items()}
    return rec, ok
