"""Benchmark of the CoR-UTV hot path (BASELINE.json metric: decompositions/s and A-pass TFLOP/s vs roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2q1] [--impl ours|reference]

One "step" is one coru::corutv-equivalent decomposition (corutv.hpp:79-100) of the synthetic
BASELINE config (default C2: fp64 4000x4000, sigma_i = i^-2, d = 60, q = 1; BASELINE.json
configs[1], the config the metric is quoted on that fits one GPU). With N > 1 (torchrun) A is
row-block sharded over the ranks and one decomposition spans all of them (strong scaling).

Our arm prints one JSON line with: value (decomps/s, A resident in HBM, device-timed with CUDA
events, max over ranks), e2e (same metric through the host-buffer C-ABI with the H2D of A and the
D2H of U,T,V inside the timed region), roofline of the dominant kernel (the FP64 A-pass GEMM,
timed live with CUDA events on its launch stream inside the library), cpu_baseline (the compiled
reference on one host core, rank 0 at N=1), clocks sampled during the timed region, and
gpu_launches. `--impl reference` times the unmodified reference (oracle/_ref/libcoru_ref.so,
compiled from the reference headers) on the host's cores with its own trial-level fan-out.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from workloads import CONFIGS, make_device, make_host  # noqa: E402

METRIC = "CoR-UTV decomps/sec & A-pass TFLOPS / HBM GB/s vs roofline at 1/2/4/8 B200"
UNIT = "decomps/s"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ---- clocks sampling ----------------------------------------------------------------------------
class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region.

    NVML is polled every ~2 ms from a host thread (the C2 timed region is only ~15 ms, far below
    nvidia-smi's 200 ms minimum interval); one sample is always taken at entry. Falls back to
    `nvidia-smi -lms 200` when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu_index: int, period_s: float = 0.002):
        self.gpu = gpu_index
        self.period = period_s
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._nvml = None

    def _sample(self):
        nv, h = self._nvml, self._h
        self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                             nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
                             nv.nvmlDeviceGetCurrentClocksEventReasons(h)))

    def _loop(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                return
            time.sleep(self.period)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nvml = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(self._physical_index())
            self._sample()
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        except Exception:  # noqa: BLE001
            self._nvml = None
        return self

    def _physical_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [x.strip() for x in vis.split(",") if x.strip()]
            if self.gpu < len(ids) and ids[self.gpu].isdigit():
                return int(ids[self.gpu])
        return self.gpu

    def __exit__(self, *a):
        self._stop.set()
        if self._nvml is not None:
            self._t.join(timeout=1)
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": "unavailable"}
        reasons = set()
        for nm, attr in self.REASONS:
            bit = getattr(self._nvml, attr, 0)
            if any(s[2] & bit for s in self.samples):
                reasons.add(nm)
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": sorted(reasons),
                "samples": len(self.samples), "source": "NVML polled every 2 ms during the timed region"}


# ---- peaks ----------------------------------------------------------------------------------------
def measured_fp64_peak_tflops(torch):
    """FP64 roofline denominator: cuBLAS DGEMM 8192^3 burst, measured in this run
    (MEASURED_PEAKS.json carries only HBM and bf16 figures)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b, c
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def measured_tf32_peak_tflops(torch):
    """Dense TF32 tensor-core throughput: cuBLAS fp32 8192^3 GEMM with TF32 allowed, burst (best of 5)."""
    n = 8192
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(n, n, dtype=torch.float32, device="cuda")
    b = torch.randn(n, n, dtype=torch.float32, device="cuda")
    c = torch.empty_like(a)
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    torch.backends.cuda.matmul.allow_tf32 = prev
    del a, b, c
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def ncu_traffic(config_name):
    """dram bytes per A-pass launch from the committed ncu --set full summary (profiles/), if any."""
    p = os.path.join(ROOT, "profiles", "ncu_apass_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get(config_name, {}).get("dram_bytes_per_launch")
    return None


# ---- CPU baselines ----------------------------------------------------------------------------------
def cpu_baseline_sample(cfg, a_host, variant=0):
    """The compiled reference (oracle/_ref) on ONE host core: bounded sample of whole decompositions."""
    from oracle import Reference, has_reference, Oracle
    if has_reference():
        ref, kind = Reference(), "reference"
        run = lambda s: ref.corutv(a_host, cfg.d, cfg.q, variant, 42, s)  # noqa: E731
    else:
        ora, kind = Oracle(), "port"
        run = lambda s: ora.corutv(a_host, cfg.d, cfg.q, variant, 42, s, threads=1)  # noqa: E731
    times = []
    budget = 12.0
    t_all = time.perf_counter()
    s = 0
    while True:
        t0 = time.perf_counter()
        run(s)
        times.append(time.perf_counter() - t0)
        s += 1
        if time.perf_counter() - t_all > budget or s >= 5:
            break
    per = sum(times) / len(times)
    return {"value": 1.0 / per, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{len(times)} full {cfg.name} decompositions, single thread, s/decomp={per:.3f}",
            "host_cores_total": os.cpu_count()}


def run_reference_arm(args, cfg):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    from oracle import Reference, has_reference, Oracle
    a = make_host(cfg.name)
    threads = min(os.cpu_count() or 1, 64)
    if has_reference():
        ref, kind = Reference(), "reference"
        batch = lambda s0: ref.corutv_batch(a, cfg.d, cfg.q, 42, s0, threads, threads)  # noqa: E731
    else:
        ora, kind = Oracle(), "port"

        def batch(s0):
            import concurrent.futures as cf
            with cf.ThreadPoolExecutor(threads) as ex:
                list(ex.map(lambda i: ora.corutv(a, cfg.d, cfg.q, 0, 42, s0 + i, threads=1), range(threads)))
    for w in range(args.warmup):
        batch(10_000 + w * threads)
    t0 = time.perf_counter()
    for s in range(args.steps):
        batch(s * threads)
    dt = time.perf_counter() - t0
    value = args.steps * threads / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype.replace("f", "f"),
        "data": "synthetic", "config": config_block(cfg, args, l2="n/a (CPU)"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"each step = {threads} concurrent unmodified corutv calls (trial fan-out, "
                                   f"coru_cli.cpp:171-177), one per host thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_block(cfg, args, l2):
    return {"workload": f"{cfg.name}: {cfg.dtype} {cfg.m}x{cfg.n}, {cfg.desc}, d={cfg.d}, q={cfg.q}, k={cfg.k}",
            "m": cfg.m, "n": cfg.n, "d": cfg.d, "q": cfg.q, "k": cfg.k, "seed": "RngSeed{42, step}",
            "variant": args.variant, "passes_over_A": 2 * cfg.q + (3 if args.variant == "exact" else 2),
            "parallelism": f"row-sharded x{args.gpus}" if args.gpus > 1 else "single GPU", "l2": l2}


# ---- our arm --------------------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    import paper_1810_07323_b200 as cg

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = cg.Context(local)
    if world > 1:
        uid = [cg.Context.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.init_comm(rank, world, uid[0])
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)
    ctx.set_stream(stream.cuda_stream)

    # A: generated on the GPU (identical on every rank), this rank keeps its row block.
    a_full = make_device(cfg.name, device=dev)
    row0, rows = cg.shard_rows(cfg.m, rank, world)
    a = a_full[row0:row0 + rows].contiguous()
    del a_full
    torch.cuda.empty_cache()
    dt = torch.float64 if cfg.dtype == "f64" else torch.float32
    m_local, n, d = rows, cfg.n, cfg.d
    u = torch.empty((m_local, d), dtype=dt, device=dev)
    t = torch.empty((d, d), dtype=dt, device=dev)
    v = torch.empty((n, d), dtype=dt, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    lib = cg.load_library()
    sfx = "f64" if cfg.dtype == "f64" else "f32"
    fn = getattr(lib, f"coru_corutv_{sfx}_dev")
    perm = np.zeros(d, np.int64)
    out = cg._Utv(u.data_ptr(), d, t.data_ptr(), d, v.data_ptr(), d, perm.ctypes.data, 0, 0)
    import ctypes as C

    def step(s):
        cg._check(fn(ctx.h, a.data_ptr(), m_local, cfg.m, n, a.stride(0), d, cfg.q, args.variant_id, 42, s,
                      C.byref(out)))

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for w in range(args.warmup):
        step(1_000_000 + w)
    torch.cuda.synchronize()

    # Timed region: K steps; each step device-timed with CUDA events on the library's stream,
    # L2 flushed between steps outside the events. Max over ranks.
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ctx.set_profiling(True)
    cg.launch_count(reset=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for s in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                evs[s][0].record(stream)
            step(s)
            evs[s][1].record(stream)
        torch.cuda.synchronize()
        barrier()
        wall = time.perf_counter() - wall0
    launches = cg.launch_count(reset=True)
    prof = ctx.profile_apass()
    ctx.set_profiling(False)
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    total_ms = sum(step_ms)
    if world > 1:
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    value = args.steps / (total_ms * 1e-3)

    # e2e: the same decomposition through host buffers (pinned A in, U/T/V out) every step.
    e2e = run_e2e(args, cfg, ctx, a, world, rank, local, dev, barrier)

    peaks, peak_src = measured_peaks()
    roof = None
    if prof["launches"]:
        avg_ms = prof["ms"] / prof["launches"]
        flops_per = prof["flops"] / prof["launches"]
        bytes_per = prof["bytes"] / prof["launches"]
        achieved = flops_per / (avg_ms * 1e-3) / 1e12
        traffic = ncu_traffic(cfg.name)
        if cfg.dtype == "f64":
            peak = measured_fp64_peak_tflops(torch)
            kernel = "k_gemm_f64 (FP64 DMMA A-pass: B1=A·B2, B2=A^T·B1, W=A·Q2; stream-K fix-up fused)"
            peak_src = ("cuBLAS DGEMM 8192^3 burst measured in this run (no FP64 entry in "
                        f"{peak_src})")
        else:
            tf32 = measured_tf32_peak_tflops(torch)
            peak = tf32 / 3.0
            kernel = ("k_apass_tf32x3 (tcgen05.mma kind::tf32, 3xTF32 split, TMA-fed, A hi/lo in TMEM) "
                      "+ k_split_xt (X hi/lo transpose)")
            peak_src = (f"cuBLAS TF32 8192^3 burst measured in this run ({tf32:.0f} TFLOP/s) / 3: the "
                        "3xTF32 scheme issues three TF32 MMAs per fp32 product")
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": kernel, "peak_source": peak_src,
                "algorithmic_flops_per_launch": flops_per, "algorithmic_bytes_per_launch": bytes_per,
                "avg_launch_ms": avg_ms, "launches": prof["launches"],
                "hbm_gbs": bytes_per / (avg_ms * 1e-3) / 1e9, "hbm_peak_gbs": peaks.get("hbm_gbs"),
                "hbm_frac": bytes_per / (avg_ms * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
                "apass_share_of_step": prof["ms"] / max(sum(step_ms), 1e-9)}

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(cfg, make_host(cfg.name), args.variant_id)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
            "config": config_block(cfg, args, l2="flushed between steps (256 MB write outside the per-step events)"),
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "gpu_launches": launches,
            "clocks": clk.summary(), "wall_s_timed_region": wall,
            "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    ctx.close()
    return 0


def run_e2e(args, cfg, ctx, a, world, rank, local, dev, barrier):
    import ctypes as C
    import torch
    import paper_1810_07323_b200 as cg
    lib = cg.load_library()
    m_local, n, d = a.shape[0], cfg.n, cfg.d
    dt = a.dtype
    a_host = a.cpu().pin_memory()
    u_h = torch.empty((m_local, d), dtype=dt).pin_memory()
    t_h = torch.empty((d, d), dtype=dt).pin_memory()
    v_h = torch.empty((n, d), dtype=dt).pin_memory()
    perm = np.zeros(d, np.int64)
    lower, warn = C.c_int(), C.c_int()
    sfx = "f64" if cfg.dtype == "f64" else "f32"
    if world == 1:
        fn = getattr(lib, f"coru_corutv_{sfx}")

        def step(s):
            cg._check(fn(ctx.h, a_host.data_ptr(), cfg.m, n, d, cfg.q, args.variant_id, 42, 500_000 + s,
                         u_h.data_ptr(), t_h.data_ptr(), v_h.data_ptr(), perm.ctypes.data, C.byref(lower),
                         C.byref(warn)))
    else:
        a_dev = torch.empty_like(a)
        u = torch.empty((m_local, d), dtype=dt, device=dev)
        t = torch.empty((d, d), dtype=dt, device=dev)
        v = torch.empty((n, d), dtype=dt, device=dev)
        out = cg._Utv(u.data_ptr(), d, t.data_ptr(), d, v.data_ptr(), d, perm.ctypes.data, 0, 0)
        fn = getattr(lib, f"coru_corutv_{sfx}_dev")
        s_ = torch.cuda.Stream(dev)
        ctx.set_stream(s_.cuda_stream)

        def step(s):
            with torch.cuda.stream(s_):
                a_dev.copy_(a_host, non_blocking=True)
            cg._check(fn(ctx.h, a_dev.data_ptr(), m_local, cfg.m, n, a_dev.stride(0), d, cfg.q, args.variant_id, 42,
                         500_000 + s, C.byref(out)))
            with torch.cuda.stream(s_):
                u_h.copy_(u, non_blocking=True)
                t_h.copy_(t, non_blocking=True)
                v_h.copy_(v, non_blocking=True)
            s_.synchronize()
    for w in range(min(args.warmup, 2)):
        step(w + 100)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(args.steps):
        step(s)
    torch.cuda.synchronize()
    barrier()
    el = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([el], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = float(tt.item())
    es = a.element_size()
    return {"value": args.steps / el, "unit": UNIT, "h2d_bytes_per_step": int(a.numel() * es),
            "d2h_bytes_per_step": int((m_local * d + d * d + n * d) * es + d * 8 + 8),
            "api": f"coru_corutv_{sfx} (host buffers, pinned)" if world == 1 else
                   f"coru_corutv_{sfx}_dev + per-step H2D(A shard)/D2H(U,T,V)",
            "timer": "host wall clock (each call returns synchronised), max over ranks"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2q1", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--variant", default="exact", choices=["exact", "approx"],
                    help="DVariant (corutv.hpp:17); the BASELINE metric is quoted on exact")
    args = ap.parse_args()
    args.variant_id = 0 if args.variant == "exact" else 1
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
