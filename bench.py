"""Benchmark of the CoR-UTV hot path (BASELINE.json metric: decompositions/s and A-pass TFLOP/s vs roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

One "step" is one coru::corutv-equivalent decomposition (corutv.hpp:79-100) of a synthetic
BASELINE config. Default: C3 (fp64 200000x2000, sigma_i = 10^(-i/20), d = 110, q = 1) — the
largest fp64 config the metric is quoted on at 1/2/4/8 GPUs whose reference arm fits the driver's
window; --config C1 / C2q1 / C2q2 / C4 / C5 select the others. With N > 1 A is row-block sharded
over N ranks and one decomposition spans all of them (strong scaling); `--gpus N` without torchrun
re-launches itself under torch.distributed.run.

A is generated ONCE per arm by tests/workloads.make_device (seeded torch CUDA generator) and both
arms decompose the identical bytes (its SHA-256 is in `config`). Φ is the reference's
gaussian() bit for bit (host-exact mode, the library default), generated inside every timed step.

Our arm prints one JSON line with: value (decomps/s, A resident in HBM, device-timed with CUDA
events, max over ranks), e2e (same metric through the host-buffer C-ABI coru_corutv_f64 with a
PAGEABLE A — the drop-in caller's std::vector storage — H2D of A and D2H of U,T,V inside the
timed region; e2e_pinned: the same with page-locked A), roofline of the dominant kernel (the A-pass,
timed live with CUDA events on its launch stream inside the library), cpu_baseline (the compiled
reference, rank 0 at N=1), clocks sampled during the timed region, and gpu_launches.
`--impl reference` times the reference itself (oracle/_ref/libcoru_ref.so, compiled from the
reference headers: ref_corutv_mt = coru::corutv's exact-D steps with its products spread over all
host cores in the reference's per-entry summation order, bit-identical) — one decomposition per
step on the same A bytes.
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

from workloads import CONFIGS, make_device, make_host, sha256  # noqa: E402

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


def measured_int8_peak_tops(torch):
    """Dense INT8 tensor-core throughput: cuBLASLt int8 GEMM (torch._int_mm) 8192^3, burst (best of 5)."""
    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    for _ in range(2):
        c = torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = torch._int_mm(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
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


# ---- workload ---------------------------------------------------------------------------------------
def make_workload(cfg, want_host=True, device=None):
    """A generated once (seeded torch CUDA generator, tests/workloads.py) -> (device tensor or None,
    host numpy array or None, sha256 of the host bytes). Without a GPU (reference arm on a CPU-only
    host) the numpy generator stands in and the SHA says which bytes were used."""
    import torch
    if torch.cuda.is_available():
        a_dev = make_device(cfg.name, device=device or torch.device("cuda", 0))
        torch.cuda.synchronize()
        a_host = a_dev.cpu().numpy() if want_host else None
        return a_dev, a_host, (sha256(a_host) if a_host is not None else None), "workloads.make_device (torch CUDA)"
    a_host = make_host(cfg.name)
    return None, a_host, sha256(a_host), "workloads.make_host (numpy; no GPU on this host)"


def config_block(cfg, args, a_sha, gen):
    """Identical in both arms (the driver compares them)."""
    return {"workload": f"{cfg.name}: {cfg.dtype} {cfg.m}x{cfg.n}, {cfg.desc}, d={cfg.d}, q={cfg.q}, k={cfg.k}",
            "m": cfg.m, "n": cfg.n, "d": cfg.d, "q": cfg.q, "k": cfg.k, "seed": "RngSeed{42, step}",
            "variant": args.variant, "passes_over_A": 2 * cfg.q + (3 if args.variant == "exact" else 2),
            "parallelism": f"row-sharded x{args.gpus}" if args.gpus > 1 else "single GPU",
            "phi": "host-exact: coru::gaussian bit for bit (rng.hpp:86-112), generated inside every step",
            "a_sha256": a_sha, "a_generator": gen,
            "l2": ("GPU arm: 256 MB write between steps outside the per-step events (126 MB L2); "
                   "reference arm: n/a (CPU)"),
            "launch": ("small configs (rows x cols <= 2^24): the library replays the decomposition from a CUDA graph "
                       "from the third call on the same buffers on; larger ones: plain launches")}


# ---- CPU reference ------------------------------------------------------------------------------
def reference_runner(cfg, a_host, variant_id):
    """One whole decomposition of the reference on all host cores, as a callable of the seed stream.

    fp64 exact-D, m >= n: ref_corutv_mt (oracle/_ref: the reference headers compiled in place; its
    gaussian / householder_qr / qrcp / flag are the reference's own serial functions, the A-products
    run over all cores in the reference's per-entry order — bit-identical to coru::corutv).
    Otherwise coru::corutv itself (single thread) or, for fp32 (no fp32 reference exists), the
    bit-exact-restatement oracle in fp32 on all cores."""
    from oracle import Oracle, Reference, has_reference
    threads = os.cpu_count() or 1
    if cfg.dtype == "f64" and has_reference():
        ref = Reference()
        if variant_id == 0 and cfg.m >= cfg.n:
            return (lambda s: ref.corutv(a_host, cfg.d, cfg.q, 0, 42, s, threads=threads)), threads, "reference", \
                "ref_corutv_mt: the reference's corutv steps, products over all host cores (bit-identical)"
        return (lambda s: ref.corutv(a_host, cfg.d, cfg.q, variant_id, 42, s)), 1, "reference", \
            "coru::corutv, single thread"
    ora = Oracle()
    return (lambda s: ora.corutv(a_host, cfg.d, cfg.q, variant_id, 42, s, threads=threads)), threads, "port", \
        "oracle/coru_oracle.c (bit-exact restatement; fp32 instantiation for the fp32 config) on all cores"


def cpu_baseline_sample(cfg, a_host, variant_id, budget_s=12.0):
    """Bounded sample of whole reference decompositions (>= 1, stop after ~budget_s)."""
    run, cores, kind, what = reference_runner(cfg, a_host, variant_id)
    times = []
    t_all = time.perf_counter()
    s = 0
    while True:
        t0 = time.perf_counter()
        run(10_000 + s)
        times.append(time.perf_counter() - t0)
        s += 1
        if time.perf_counter() - t_all > budget_s or s >= 5:
            break
    per = sum(times) / len(times)
    return {"value": 1.0 / per, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{len(times)} full {cfg.name} decomposition(s) on the same A, {what}, s/decomp={per:.3f}",
            "host_cores_total": os.cpu_count()}


def run_reference_arm(args, cfg):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    _, a_host, a_sha, gen = make_workload(cfg)
    run, cores, kind, what = reference_runner(cfg, a_host, args.variant_id)
    for w in range(args.warmup):
        run(1_000_000 + w)
    times = []
    for s in range(args.steps):
        t0 = time.perf_counter()
        run(s)
        times.append(time.perf_counter() - t0)
    dt = sum(times)
    value = args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype,
        "data": "synthetic", "config": config_block(cfg, args, a_sha, gen),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"each step = one whole {cfg.name} decomposition of the same A: {what}",
                         "host_cores_total": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_s": {"min": min(times), "median": statistics.median(times), "max": max(times)},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- our arm --------------------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    import paper_1810_07323_b200 as cg

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
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

    # A: generated on the GPU (identical bytes on every rank and in the reference arm); this rank
    # keeps its row block. Rank 0 keeps a host copy for the e2e leg, the CPU baseline and the SHA.
    a_full, a_host_full, a_sha, gen = make_workload(cfg, want_host=(rank == 0), device=dev)
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
    # Small configs (C1, C2) are replayed from a CUDA graph by the library, which excludes the
    # in-library A-pass events: their timed region runs without them and the A-pass durations are
    # collected over a second loop of the same K steps (plain launches, the same kernels).
    graph_cfg = world == 1 and cfg.m * cfg.n <= (1 << 24) and cfg.d <= 112
    ctx.set_profiling(not graph_cfg)
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
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    graph_replays = ctx.graph_replays()
    prof_step_ms = step_ms
    if graph_cfg:
        ctx.set_profiling(True)
        pevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for s in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                pevs[s][0].record(stream)
            step(s)
            pevs[s][1].record(stream)
        torch.cuda.synchronize()
        prof_step_ms = [e0.elapsed_time(e1) for e0, e1 in pevs]
        cg.launch_count(reset=True)
    prof = ctx.profile_apass()
    ctx.set_profiling(False)
    total_ms = sum(step_ms)
    if world > 1:
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    value = args.steps / (total_ms * 1e-3)

    # e2e: the same decomposition through host buffers every step (pageable A = the drop-in
    # caller's storage; then page-locked A).
    e2e = run_e2e(args, cfg, ctx, a, a_host_full, world, rank, local, dev, barrier, pinned=False)
    e2e_pinned = run_e2e(args, cfg, ctx, a, a_host_full, world, rank, local, dev, barrier, pinned=True)

    peaks, peak_src = measured_peaks()
    roof = None
    if prof["launches"]:
        # The roofline is the kernel's: its launch duration is averaged over the A-passes of the timed
        # steps that had the GPU to themselves. Passes issued while the call's second stream runs QR
        # kernels (the Q1 tree under the last A^T pass of tall sketches, and under the projection
        # pass) share the SMs with them; their average is reported next to it.
        avg_all_ms = prof["ms"] / prof["launches"]
        n_ex = prof.get("launches_exclusive", 0)
        avg_ms = prof["ms_exclusive"] / n_ex if n_ex else avg_all_ms
        flops_per = prof["flops"] / prof["launches"]
        bytes_per = prof["bytes"] / prof["launches"]
        achieved = flops_per / (avg_ms * 1e-3) / 1e12
        traffic = ncu_traffic(cfg.name)
        engine = ctx.last_f64_engine() if cfg.dtype == "f64" else -1
        if cfg.dtype == "f64" and engine == 0:
            # small matrix: the library kept the A-passes on the FP64 tensor path (DMMA stream-K)
            dgemm = measured_fp64_peak_tflops(torch)
            t_tensor = flops_per / (dgemm * 1e12)
            t_hbm = bytes_per / (peaks.get("hbm_gbs", 6650.0) * 1e9)
            roof = {"bound": "tensor" if t_tensor >= t_hbm else "hbm",
                    "achieved": achieved if t_tensor >= t_hbm else bytes_per / (avg_ms * 1e-3) / 1e9,
                    "peak": dgemm if t_tensor >= t_hbm else peaks.get("hbm_gbs"),
                    "unit": "TFLOP/s" if t_tensor >= t_hbm else "GB/s",
                    "frac": max(t_tensor, t_hbm) / (avg_ms * 1e-3), "traffic": traffic,
                    "kernel": "k_gemm_f64 (FP64 DMMA m16n8k8, stream-K; matrices under two waves of int8 CTAs)",
                    "peak_source": (f"cuBLAS DGEMM 8192^3 burst measured in this run ({dgemm:.1f} TFLOP/s); "
                                    f"HBM {peaks.get('hbm_gbs')} GB/s from {peak_src}"),
                    "t_tensor_ms": t_tensor * 1e3, "t_hbm_ms": t_hbm * 1e3,
                    "algorithmic_flops_per_launch": flops_per, "algorithmic_bytes_per_launch": bytes_per,
                    "avg_launch_ms": avg_ms, "launches": prof["launches"],
                    "hbm_gbs": bytes_per / (avg_ms * 1e-3) / 1e9, "hbm_peak_gbs": peaks.get("hbm_gbs"),
                    "hbm_frac": bytes_per / (avg_ms * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
                    "apass_share_of_step": prof["ms"] / max(sum(prof_step_ms), 1e-9)}
        elif cfg.dtype == "f64":
            # The fp64 A-pass runs on the INT8 tensor cores (Ozaki scheme, gemm_oz.cu): per launch
            # 28 slice products (levels 0..6 of 7 x 7 digit pairs) over the padded width d16.
            dgemm = measured_fp64_peak_tflops(torch)
            int8 = measured_int8_peak_tops(torch)
            d16 = (cfg.d + 15) // 16 * 16
            int8_ops = 28 * 2.0 * (cfg.m // world) * cfg.n * d16
            t_tensor = int8_ops / (int8 * 1e12)
            t_hbm = bytes_per / (peaks.get("hbm_gbs", 6650.0) * 1e9)
            achieved_int8 = int8_ops / (avg_ms * 1e-3) / 1e12
            kname = ("k_apass_oz (fp64 A-pass on the INT8 tensor cores: tcgen05.mma kind::i8, Ozaki scheme with 7 "
                     "balanced 8-bit digit slices per operand, levels 0..6 = 28 slice products; A TMA-staged, "
                     "converted in-kernel; + X split / exponent kernels)") if engine == 1 else (
                     "k_apass_ozp (fp64 A-pass on the INT8 tensor cores over digit planes converted once per "
                     "decomposition by k_oz_planes: pure TMA -> tcgen05.mma kind::i8, 28 slice products)"
                     ) if engine == 2 else (
                     "k_apass_oz / k_apass_ozp, hybrid (fp64 A-pass on the INT8 tensor cores: tcgen05.mma kind::i8, "
                     "Ozaki scheme, 28 slice products; the first A.X pass converts A in the kernel and TMA-stores "
                     "the row-scaled digit planes, the later A.X passes stream them (k_apass_ozp), the A^T.Y "
                     "passes convert in the kernel; + X split / exponent kernels)")
            roof = {"bound": "tensor" if t_tensor >= t_hbm else "hbm",
                    "achieved": achieved_int8 if t_tensor >= t_hbm else bytes_per / (avg_ms * 1e-3) / 1e9,
                    "peak": int8 if t_tensor >= t_hbm else peaks.get("hbm_gbs"),
                    "unit": "TOP/s (int8)" if t_tensor >= t_hbm else "GB/s",
                    "frac": max(t_tensor, t_hbm) / (avg_ms * 1e-3), "traffic": traffic,
                    "kernel": kname,
                    "peak_source": (f"cuBLASLt int8 GEMM 8192^3 burst measured in this run ({int8:.0f} TOP/s); "
                                    f"HBM {peaks.get('hbm_gbs')} GB/s from {peak_src}"),
                    "algorithmic_int8_ops_per_launch": int8_ops, "t_tensor_ms": t_tensor * 1e3,
                    "t_hbm_ms": t_hbm * 1e3,
                    "algorithmic_flops_per_launch": flops_per, "algorithmic_bytes_per_launch": bytes_per,
                    "avg_launch_ms": avg_ms, "launches": prof["launches"],
                    "fp64_equiv_tflops": achieved, "dgemm_peak_tflops": dgemm,
                    "fp64_equiv_vs_dgemm_peak": achieved / dgemm,
                    "hbm_gbs": bytes_per / (avg_ms * 1e-3) / 1e9, "hbm_peak_gbs": peaks.get("hbm_gbs"),
                    "hbm_frac": bytes_per / (avg_ms * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
                    "apass_share_of_step": prof["ms"] / max(sum(prof_step_ms), 1e-9)}
        else:
            tf32_cublas = measured_tf32_peak_tflops(torch)
            # dense TF32 = half the dense bf16 rate: cuBLAS's TF32 GEMM does not reach it, so the
            # larger of the two is the roofline
            tf32_from_bf16 = float(peaks.get("bf16_tflops", 0.0)) / 2.0
            tf32 = max(tf32_cublas, tf32_from_bf16)
            peak = tf32 / 3.0
            kernel = ("k_apass_tf32x3 (tcgen05.mma kind::tf32, 3xTF32 split, TMA-fed, A hi/lo in TMEM) "
                      "+ k_split_xt (X hi/lo transpose)")
            peak_src = (f"max(cuBLAS TF32 8192^3 burst measured in this run = {tf32_cublas:.0f} TFLOP/s, dense bf16 burst "
                        f"of {peak_src} / 2 = {tf32_from_bf16:.0f} TFLOP/s) / 3: the 3xTF32 scheme issues three TF32 "
                        "MMAs per fp32 product")
            roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic, "kernel": kernel, "peak_source": peak_src,
                    "algorithmic_flops_per_launch": flops_per, "algorithmic_bytes_per_launch": bytes_per,
                    "avg_launch_ms": avg_ms, "launches": prof["launches"],
                    "hbm_gbs": bytes_per / (avg_ms * 1e-3) / 1e9, "hbm_peak_gbs": peaks.get("hbm_gbs"),
                    "hbm_frac": bytes_per / (avg_ms * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
                    "apass_share_of_step": prof["ms"] / max(sum(prof_step_ms), 1e-9)}

    if roof is not None:
        roof["launches_timed_alone"] = int(n_ex) if n_ex else int(prof["launches"])
        roof["avg_launch_ms_all_passes"] = avg_all_ms
        roof["avg_launch_ms_note"] = ("avg_launch_ms / achieved / frac: A-passes of the timed steps that ran alone on the GPU; "
                                      "avg_launch_ms_all_passes includes those sharing the SMs with the QR stream")
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(cfg, a_host_full, args.variant_id)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
            "config": config_block(cfg, args, a_sha, gen),
            "e2e": e2e, "e2e_pinned": e2e_pinned, "roofline": roof, "cpu_baseline": cpu, "gpu_launches": launches,
            "cuda_graph_replays": graph_replays,
            "clocks": clk.summary(), "wall_s_timed_region": wall,
            "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    ctx.close()
    return 0


def run_e2e(args, cfg, ctx, a, a_host_full, world, rank, local, dev, barrier, pinned):
    """Host buffers in, host buffers out, every step. Single GPU: the drop-in host entry
    coru_corutv_{f64,f32} (validation, H2D of A overlapped with the first power round, D2H of
    U/T/V). N > 1: per-rank H2D of the A shard + the device entry + D2H, max over ranks."""
    import ctypes as C
    import torch
    import paper_1810_07323_b200 as cg
    lib = cg.load_library()
    m_local, n, d = a.shape[0], cfg.n, cfg.d
    dt = a.dtype
    if world == 1:
        a_np = np.ascontiguousarray(a_host_full)
        a_h = torch.from_numpy(a_np).pin_memory() if pinned else None
        a_ptr = a_h.data_ptr() if pinned else a_np.ctypes.data
    else:
        a_h = a.cpu()
        if pinned:
            a_h = a_h.pin_memory()
        a_ptr = a_h.data_ptr()
    mk = (lambda *s: torch.empty(s, dtype=dt).pin_memory()) if pinned else (lambda *s: torch.empty(s, dtype=dt))
    u_h, t_h, v_h = mk(m_local, d), mk(d, d), mk(n, d)
    perm = np.zeros(d, np.int64)
    lower, warn = C.c_int(), C.c_int()
    sfx = "f64" if cfg.dtype == "f64" else "f32"
    if world == 1:
        fn = getattr(lib, f"coru_corutv_{sfx}")

        def step(s):
            cg._check(fn(ctx.h, a_ptr, cfg.m, n, d, cfg.q, args.variant_id, 42, 500_000 + s,
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
                a_dev.copy_(a_h, non_blocking=True)
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
    kind = "page-locked" if pinned else "pageable"
    return {"value": args.steps / el, "unit": UNIT, "h2d_bytes_per_step": int(a.numel() * es),
            "d2h_bytes_per_step": int((m_local * d + d * d + n * d) * es + d * 8 + 8),
            "host_memory": kind,
            "api": (f"coru_corutv_{sfx} (host buffers, {kind})" if world == 1 else
                    f"coru_corutv_{sfx}_dev + per-step H2D(A shard)/D2H(U,T,V), {kind} host buffers"),
            "timer": "host wall clock (each call returns synchronised), max over ranks"}


def spawn_ranks(args):
    """`--gpus N` outside torchrun: re-launch under torch.distributed.run (one rank per GPU)."""
    import socket
    import subprocess
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--variant", default="exact", choices=["exact", "approx"],
                    help="DVariant (corutv.hpp:17); the BASELINE metric is quoted on exact")
    args = ap.parse_args()
    args.variant_id = 0 if args.variant == "exact" else 1
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
