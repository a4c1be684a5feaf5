"""Benchmark of the ALM-RPCA solve with the CoR-UTV inner step (§8 f2; rpca.hpp:95-169).

    python bench_rpca.py [--n 8000] [--rank 40] [--steps 3] [--warmup 3] [--no-cpu-baseline]

One step = one alm_rpca solve (corutv inner, soft thresholding, ell = 2·rank, q = 1 — the settings of
acceptance.cpp:204-220) of a synthetic gen_rpca_instance-shaped problem (testgen.hpp:86-109): M = G1·G2^T +
S with n x rank Gaussian factors and 5 % of the entries corrupted by ±80, generated on the GPU from a fixed
seed. mu0 = 1.25/||M||_2 is estimated once by power iteration and passed to every arm (the reference's
default would run a full Jacobi SVD of M). Prints one JSON line like bench.py: value (solves/s, M resident
in HBM, device-timed), e2e (host-buffer entry, M in / L, S out each step), the roofline of the dominant
kernel (the FP64 A-pass GEMM over the iterate) and of the fused lift + ALM update kernel (HBM-bound,
40 B per entry), cpu_baseline (the compiled reference, one ALM iteration of the same instance on one core,
scaled by the GPU's iteration count), clocks and gpu_launches. Single GPU (alm_rpca is a single-GPU entry).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from bench import ClockSampler, measured_fp64_peak_tflops, measured_peaks  # noqa: E402

METRIC = "ALM-RPCA (CoR-UTV inner) solves/sec & kernel roofline on B200"
UNIT = "solves/s"


def make_instance(torch, n, r, frac, amp, seed, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    g1 = torch.randn(n, r, dtype=torch.float64, device=dev, generator=g)
    g2 = torch.randn(n, r, dtype=torch.float64, device=dev, generator=g)
    m = g1 @ g2.T
    nnz = int(frac * n * n)
    idx = torch.randperm(n * n, device=dev, generator=g)[:nnz]
    sgn = torch.where(torch.rand(nnz, device=dev, generator=g, dtype=torch.float64) < 0.5, amp, -amp)
    m.view(-1)[idx] += sgn
    return m


def spectral_estimate(torch, m, iters=60):
    v = torch.ones(m.shape[1], 1, dtype=m.dtype, device=m.device)
    s = 0.0
    for _ in range(iters):
        w = m.T @ (m @ v)
        s = float(torch.linalg.vector_norm(w))
        v = w / s
    return float(np.sqrt(s))


def ncu_update_traffic():
    """DRAM bytes per launch of the fused update kernel from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "r01_ncu_full_rpca_update.json")
    try:
        with open(path) as f:
            d = json.load(f)
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, unit = d[k].split()
            tot += float(v) * scale[unit]
        return tot
    except (OSError, KeyError, ValueError):
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8000)
    ap.add_argument("--rank", type=int, default=40)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    import torch
    import paper_1810_07323_b200 as cg

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n, r = args.n, args.rank
    m = make_instance(torch, n, r, 0.05, 80.0, 1234, dev)
    mu0 = 1.25 / spectral_estimate(torch, m)
    cfg = cg.RpcaConfig(mu0=mu0, corutv_ell=2 * r, corutv_q=1)
    ctx = cg.Context(0)
    stream = torch.cuda.Stream(dev)
    ctx.set_stream(stream.cuda_stream)
    torch.cuda.synchronize()
    res = None
    for w in range(args.warmup):
        res = cg.alm_rpca(m, cfg, cg.RngSeed(7, 100 + w), ctx=ctx)
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ctx.set_profiling(True)
    ctx.profile_apass()
    ctx.profile_rpca_update()
    cg.launch_count(reset=True)
    iters = []
    with ClockSampler(0) as clk:
        for s in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                evs[s][0].record(stream)
            res = cg.alm_rpca(m, cfg, cg.RngSeed(7, s), ctx=ctx)
            evs[s][1].record(stream)
            iters.append(res.iterations)
        torch.cuda.synchronize()
    launches = cg.launch_count(reset=True)
    ap_prof = ctx.profile_apass()
    up_prof = ctx.profile_rpca_update()
    ctx.set_profiling(False)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    value = args.steps / (total_ms * 1e-3)

    # e2e: host entry, pinned M in, L and S out, every step
    m_h = m.cpu().pin_memory()
    lib = cg.load_library()
    import ctypes as C
    l_h = torch.empty_like(m_h).pin_memory()
    s_h = torch.empty_like(m_h).pin_memory()
    resid = np.zeros(cfg.max_iter)
    rr = cg._RpcaResult()
    rr.residuals = resid.ctypes.data
    ccfg = cfg._c()
    ctx.set_stream(None)

    def e2e_step(s):
        cg._check(lib.coru_alm_rpca_f64(ctx.h, m_h.data_ptr(), n, n, C.byref(ccfg), 7, 500 + s, l_h.data_ptr(),
                                        s_h.data_ptr(), C.byref(rr)))
    e2e_step(0)
    t0 = time.perf_counter()
    for s in range(args.steps):
        e2e_step(s)
    e2e_s = (time.perf_counter() - t0) / args.steps

    peaks, psrc = measured_peaks()
    fp64 = measured_fp64_peak_tflops(torch)
    ap_avg = ap_prof["ms"] / max(ap_prof["launches"], 1)
    ap_tf = ap_prof["flops"] / max(ap_prof["launches"], 1) / (ap_avg * 1e-3) / 1e12
    up_avg = up_prof["ms"] / max(up_prof["launches"], 1)
    up_bytes = up_prof["bytes"] / max(up_prof["launches"], 1)
    up_gbs = up_bytes / (up_avg * 1e-3) / 1e9
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    roof = {"bound": "tensor", "achieved": ap_tf, "peak": fp64, "unit": "TFLOP/s", "frac": ap_tf / fp64,
            "traffic": None, "kernel": "k_gemm_f64 (FP64 DMMA passes over the iterate X: sketch, power, projection)",
            "avg_launch_ms": ap_avg, "launches": ap_prof["launches"],
            "algorithmic_flops_per_launch": ap_prof["flops"] / max(ap_prof["launches"], 1),
            "share_of_step": ap_prof["ms"] / total_ms,
            "peak_source": "cuBLAS DGEMM 8192^3 burst measured in this run"}
    roof_upd = {"bound": "hbm", "achieved": up_gbs, "peak": hbm, "unit": "GB/s", "frac": up_gbs / hbm,
                "traffic": ncu_update_traffic() if n == 8000 and r == 40 else None,
                "kernel": "k_rpca_lift_update (L = Tp·V^T in registers + shrink / multiplier / next iterate; "
                          "reads M, Y, writes S, Y, X)", "algorithmic_bytes_per_launch": up_bytes,
                "avg_launch_ms": up_avg, "launches": up_prof["launches"], "share_of_step": up_prof["ms"] / total_ms,
                "peak_source": psrc}
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import Reference, has_reference, Oracle
        mh = m_h.numpy()
        kw = dict(mu0=mu0, corutv_ell=2 * r, corutv_q=1, max_iter=1, seed=7, stream=0)
        if has_reference():
            fn, kind = (lambda: Reference().alm_rpca(mh, **kw)), "reference"
        else:
            fn, kind = (lambda: Oracle().alm_rpca(mh, **kw)), "port"
        t0 = time.perf_counter()
        fn()
        it_s = time.perf_counter() - t0
        per_solve = it_s * statistics.mean(iters)
        cpu = {"value": 1.0 / per_solve, "unit": UNIT, "cores": 1, "kind": kind,
               "sample": f"1 ALM iteration of the same {n}x{n} instance on one core ({it_s:.1f} s) x the GPU "
                         f"solve's {statistics.mean(iters):.1f} iterations", "host_cores_total": os.cpu_count()}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "none", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"RPCA{n}: M = G1·G2^T (n={n}, rank {r}) + 5% entries ±80 (gen_rpca_instance "
                               f"shape), alm_rpca corutv inner soft, ell={2 * r}, q=1, tol 1e-5, mu0=1.25/||M||_2",
                   "iterations": iters, "rank_l": res.rank_l, "s_l0": res.s_l0, "converged": res.converged,
                   "l2": "flushed between steps (256 MB write outside the per-step events)"},
        "e2e": {"value": 1.0 / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(n * n * 8),
                "d2h_bytes_per_step": int(2 * n * n * 8), "api": "coru_alm_rpca_f64 (host buffers, pinned)"},
        "roofline": roof, "roofline_update": roof_upd, "cpu_baseline": cpu, "gpu_launches": launches,
        "clocks": clk.summary(),
        "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
    }
    print(json.dumps(line), flush=True)
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
