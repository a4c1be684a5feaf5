"""B200-native CoR-UTV (arXiv:1810.07323) — Python mirror of the reference's decomposition API.

The product is ``libcoru_gpu.so`` (hand-written sm_100a kernels behind the C-ABI declared in
``include/coru_gpu.h``). This module binds that C-ABI with ctypes and mirrors the reference
interface of the hot path, ``proj/include/coru/corutv.hpp`` and ``rng.hpp``:

=====================================  =================================================
reference (C++)                        here
=====================================  =================================================
``RngSeed{seed, stream}`` rng.hpp:13   ``RngSeed(seed, stream)``
``DVariant`` corutv.hpp:17             ``DVariant.exact`` / ``DVariant.approx``
``UtvApprox`` corutv.hpp:23-34         ``UtvApprox`` (u, t, v, ell, q, variant, seed, lower,
                                       conditioning_warning, plus ``perm``)
``corutv(a, ell, q, variant, seed)``   ``corutv(a, ell, q, variant, seed)``
  corutv.hpp:79-100
``detail::sketch_bases`` :49-65        ``sketch_bases(a, ell, q, seed)``
``reconstruct`` :102                   ``reconstruct(f)``
``truncate_rank_k`` :106-110           ``truncate_rank_k(f, k)``
``singular_estimates`` :113-117        ``singular_estimates(f)``
``gaussian(rows, cols, seed)``         ``gaussian(rows, cols, seed)``
  rng.hpp:107-112
=====================================  =================================================

``a`` may be a host ``numpy`` array (the host-buffer C-ABI entry: upload, decompose, download)
or a CUDA ``torch`` tensor (the device entry; outputs are CUDA tensors). Errors mirror the
reference: ``std::invalid_argument`` -> :class:`CoruInvalidArgument` (a ``ValueError``).
There is no CPU fallback: without the built library or an sm_100 GPU every call raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Any, Optional

import numpy as np

__all__ = [
    "RngSeed", "DVariant", "UtvApprox", "SketchBases", "Context", "CoruInvalidArgument", "CoruError",
    "corutv", "sketch_bases", "project", "gaussian", "reconstruct", "truncate_rank_k",
    "singular_estimates", "shard_rows", "library_path", "load_library", "launch_count",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libcoru_gpu.so")
if os.environ.get("CORU_LIB_VARIANT"):  # tooling: A/B builds of the same library (tools/oz_variants.sh)
    _LIB_PATH = os.path.join(_HERE, f"libcoru_gpu_{os.environ['CORU_LIB_VARIANT']}.so")

CORU_OK, CORU_EINVAL, CORU_ECUDA, CORU_ENCCL, CORU_ENOMEM, CORU_ENOTSUP, CORU_EIO = range(7)


class CoruError(RuntimeError):
    """Non-argument failure of the GPU path (CUDA, NCCL, allocation)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[coru_gpu status {code}] {msg}")
        self.code = code


class CoruInvalidArgument(ValueError):
    """Mirrors the reference's std::invalid_argument (corutv.hpp:68-70,81; matrix.hpp:29-31)."""


@dataclass(frozen=True)
class RngSeed:
    """rng.hpp:13-16. Identical (seed, stream) pairs reproduce identical output."""
    seed: int = 0
    stream: int = 0


def substream(s: RngSeed, offset: int) -> RngSeed:
    """rng.hpp:18-20."""
    return RngSeed(s.seed, s.stream + offset)


class DVariant(enum.IntEnum):
    """corutv.hpp:17."""
    exact = 0
    approx = 1


@dataclass
class UtvApprox:
    """corutv.hpp:23-34 — u·t·v^T; ``perm`` are the QRCP pivots of the core (extra)."""
    u: Any
    t: Any
    v: Any
    ell: int
    q: int
    variant: DVariant
    seed: RngSeed
    lower: bool = False
    conditioning_warning: bool = False
    perm: Optional[np.ndarray] = None


@dataclass
class SketchBases:
    """corutv.hpp:42-47."""
    q1: Any
    q2: Any
    c1: Any
    c2_prev: Any
    conditioning_warning: bool = False


# --------------------------------------------------------------------------------------------
_lib = None


def library_path() -> str:
    return _LIB_PATH


class _Utv(C.Structure):
    _fields_ = [("u", C.c_void_p), ("ldu", C.c_int64), ("t", C.c_void_p), ("ldt", C.c_int64),
                ("v", C.c_void_p), ("ldv", C.c_int64), ("perm", C.c_void_p),
                ("lower", C.c_int), ("conditioning_warning", C.c_int)]


def load_library():
    """Load the in-tree libcoru_gpu.so. Fails loudly: there is no fallback implementation."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(_LIB_PATH)
    i64, u64, i32, p = C.c_int64, C.c_uint64, C.c_int, C.c_void_p
    L.coru_abi_version.restype = i32
    L.coru_last_error.restype = C.c_char_p
    L.coru_launch_count.argtypes = [i32]
    L.coru_launch_count.restype = i64
    L.coru_debug_gemm_split_cap.argtypes = [i32]
    L.coru_debug_gemm_split_cap.restype = None
    L.coru_ctx_create.argtypes = [i32, C.POINTER(p)]
    L.coru_ctx_destroy.argtypes = [p]
    L.coru_ctx_destroy.restype = None
    L.coru_ctx_set_stream.argtypes = [p, p]
    L.coru_ctx_set_host_threads.argtypes = [p, i32]
    L.coru_ctx_set_phi_mode.argtypes = [p, i32]
    L.coru_ctx_set_f32_path.argtypes = [p, i32]
    L.coru_ctx_set_wide_qr.argtypes = [p, i32]
    L.coru_ctx_set_f64_engine.argtypes = [p, i32]
    L.coru_ctx_last_f64_engine.argtypes = [p]
    L.coru_ctx_graph_replays.argtypes = [p]
    L.coru_ctx_graph_replays.restype = i64
    L.coru_comm_unique_id.argtypes = [p]
    L.coru_ctx_init_comm.argtypes = [p, i32, i32, p]
    L.coru_ctx_set_profiling.argtypes = [p, i32]
    L.coru_ctx_profile_apass.argtypes = [p, C.POINTER(C.c_double), C.POINTER(i64), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]
    L.coru_ctx_profile_apass_exclusive.argtypes = [p, C.POINTER(C.c_double), C.POINTER(i64)]
    L.coru_threadcomm_create.argtypes = [i32]
    L.coru_threadcomm_create.restype = p
    L.coru_threadcomm_destroy.argtypes = [p]
    L.coru_threadcomm_destroy.restype = None
    L.coru_ctx_init_threadcomm.argtypes = [p, p, i32]
    L.coru_shard_rows.argtypes = [i64, i32, i32, C.POINTER(i64), C.POINTER(i64)]
    L.coru_shard_rows.restype = None
    for sfx in ("f64", "f32"):
        getattr(L, f"coru_corutv_{sfx}_dev").argtypes = [p, p, i64, i64, i64, i64, i64, i32, i32, u64, u64,
                                                         C.POINTER(_Utv)]
        getattr(L, f"coru_corutv_{sfx}").argtypes = [p, p, i64, i64, i64, i32, i32, u64, u64, p, p, p, p,
                                                     C.POINTER(i32), C.POINTER(i32)]
    for sfx in ("f64", "f32"):
        getattr(L, f"coru_corutv_{sfx}_ooc").argtypes = [p, p, i64, i64, i64, i64, i32, i32, u64, u64, i64, p]
    L.coru_read_matrix_bin_header.argtypes = [C.c_char_p, C.POINTER(i64), C.POINTER(i64)]
    L.coru_corutv_f64_file.argtypes = [p, C.c_char_p, i64, i32, i32, u64, u64, i64, p]
    L.coru_sketch_bases_f64_dev.argtypes = [p, p, i64, i64, i64, i64, i64, i32, u64, u64, p, i64, p, i64, p, i64,
                                            p, i64, C.POINTER(i32)]
    L.coru_sketch_bases_f64.argtypes = [p, p, i64, i64, i64, i32, u64, u64, p, p, p, p, C.POINTER(i32)]
    L.coru_project_f64_dev.argtypes = [p, p, i64, i64, i64, p, i64, p, i64, i64, p, i64]
    L.coru_gaussian.argtypes = [i64, i64, u64, u64, p, i32]
    L.coru_gaussian_f64_dev.argtypes = [p, i64, i64, u64, u64, p, i64]
    L.coru_gemm_f64_dev.argtypes = [p, i32, p, i64, p, i64, p, i64, i64, i64, i64]
    L.coru_gemm_f32_dev.argtypes = [p, i32, p, i64, p, i64, p, i64, i64, i64, i64]
    L.coru_tsqr_f64_dev.argtypes = [p, p, i64, i64, i64, p, i64, p, i64]
    L.coru_qrcp_f64_dev.argtypes = [p, p, i64, i64, p, i64, p, i64, p]
    L.coru_pinv_f64_dev.argtypes = [p, p, i64, i64, p, i64, C.POINTER(i32)]
    L.coru_svd_f64_dev.argtypes = [p, p, i64, i64, p, i64, p, p, i64, C.POINTER(i32)]
    L.coru_tsr_svd_f64_dev.argtypes = [p, p, i64, i64, i64, i64, u64, u64, p, i64, p, p, i64, C.POINTER(i32)]
    L.coru_tsr_svd_f64.argtypes = [p, p, i64, i64, i64, u64, u64, p, p, p, C.POINTER(i32)]
    L.coru_sor_svd_f64_dev.argtypes = [p, p, i64, i64, i64, i64, i64, i32, u64, u64, p, i64]
    L.coru_sor_svd_f64.argtypes = [p, p, i64, i64, i64, i64, i32, u64, u64, p]
    L.coru_rpca_config_default.argtypes = [p]
    L.coru_ctx_profile_rpca_update.argtypes = [p, C.POINTER(C.c_double), C.POINTER(i64), C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.coru_rpca_config_default.restype = None
    L.coru_alm_rpca_f64_dev.argtypes = [p, p, i64, i64, i64, p, u64, u64, p, i64, p, i64, p]
    L.coru_alm_rpca_f64.argtypes = [p, p, i64, i64, p, u64, u64, p, p, p]
    _lib = L
    return L


def _check(rc: int):
    if rc == CORU_OK:
        return
    msg = load_library().coru_last_error().decode(errors="replace")
    if rc == CORU_EINVAL:
        raise CoruInvalidArgument(msg)
    if rc == CORU_ENOTSUP:
        raise NotImplementedError(msg)
    if rc == CORU_EIO:
        raise CoruIoError(msg)
    raise CoruError(rc, msg)


def launch_count(reset: bool = False) -> int:
    """Kernels this library launched on the calling thread (bench evidence)."""
    return int(load_library().coru_launch_count(1 if reset else 0))


def debug_gemm_split_cap(cap: int) -> None:
    """Test tooling: cap the stream-K CTAs per output tile of the FP64 GEMM planner (0 = default)."""
    load_library().coru_debug_gemm_split_cap(int(cap))


def shard_rows(m: int, rank: int, world: int) -> tuple[int, int]:
    """Row block (row0, rows) of ``rank`` — coru_shard_rows."""
    a, b = C.c_int64(), C.c_int64()
    load_library().coru_shard_rows(m, rank, world, C.byref(a), C.byref(b))
    return a.value, b.value


class Context:
    """One coru_ctx: device, stream, workspace arena, pinned staging, optional NCCL communicator."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        _check(self.lib.coru_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self.rank, self.world = 0, 1

    def close(self):
        if getattr(self, "h", None):
            self.lib.coru_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int | None):
        _check(self.lib.coru_ctx_set_stream(self.h, C.c_void_p(stream_handle or 0)))

    def set_host_threads(self, n: int):
        _check(self.lib.coru_ctx_set_host_threads(self.h, n))

    PHI_DEVICE, PHI_HOST_EXACT = 0, 1

    def set_phi_mode(self, mode: int):
        """PHI_HOST_EXACT (default): host-generated, bit-identical to the reference's gaussian()
        (rng.hpp:86-112); PHI_DEVICE (opt-in): Φ generated on the GPU (reference word stream
        bit-for-bit, Box–Muller values within a few ulp of the host libm's)."""
        _check(self.lib.coru_ctx_set_phi_mode(self.h, mode))

    F32_AUTO, F32_SIMT, F32_TC = 0, 1, 2

    def set_f32_path(self, mode: int):
        """fp32 A-pass engine: F32_AUTO (default: tcgen05 3xTF32 tensor cores for A-pass-sized
        products), F32_SIMT (CUDA-core FFMA), F32_TC (tensor cores wherever the shape allows)."""
        _check(self.lib.coru_ctx_set_f32_path(self.h, mode))

    F64_AUTO, F64_DMMA, F64_OZAKI_INLINE, F64_OZAKI_PLANES, F64_OZAKI_HYBRID = 0, 1, 2, 3, 4

    def set_f64_engine(self, mode: int):
        """fp64 A-pass engine: F64_AUTO (default: INT8 tensor cores, Ozaki scheme, for A-pass-sized
        products over the caller's A; digits converted inside each pass or once per decomposition
        into digit planes, by a cost model), F64_DMMA (FP64 DMMA for everything),
        F64_OZAKI_INLINE / F64_OZAKI_PLANES / F64_OZAKI_HYBRID (force where the conversion happens;
        hybrid = the first A·X pass converts in the kernel and writes the row-scaled planes that the
        later A·X passes stream)."""
        _check(self.lib.coru_ctx_set_f64_engine(self.h, mode))

    def last_f64_engine(self) -> int:
        """Engine of the last fp64 decomposition's A-passes: 0 DMMA, 1 Ozaki (in-kernel digits),
        2 Ozaki (digit planes), 3 Ozaki hybrid."""
        return int(self.lib.coru_ctx_last_f64_engine(self.h))

    def graph_replays(self) -> int:
        """CUDA-graph replays of small decompositions so far (coru_ctx_graph_replays)."""
        return int(self.lib.coru_ctx_graph_replays(self.h))

    def set_wide_qr(self, on: bool):
        """QR of sketches wider than 128 columns: CholeskyQR2 in fp64 with a device-side Householder
        fall-back (default), or the Householder tree only."""
        _check(self.lib.coru_ctx_set_wide_qr(self.h, 1 if on else 0))

    def set_profiling(self, on: bool):
        _check(self.lib.coru_ctx_set_profiling(self.h, 1 if on else 0))

    def profile_apass(self) -> dict:
        """Summed device time of the A-passes since the last read (CUDA events on the launch stream);
        ms_exclusive / launches_exclusive: the passes not sharing the GPU with the call's QR stream."""
        ems, en = C.c_double(), C.c_int64()
        _check(self.lib.coru_ctx_profile_apass_exclusive(self.h, C.byref(ems), C.byref(en)))
        ms, n, fl, by = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        _check(self.lib.coru_ctx_profile_apass(self.h, C.byref(ms), C.byref(n), C.byref(fl), C.byref(by)))
        return {"ms": ms.value, "launches": n.value, "flops": fl.value, "bytes": by.value,
                "ms_exclusive": ems.value, "launches_exclusive": en.value}

    def profile_rpca_update(self) -> dict:
        """Summed device time of alm_rpca's fused lift + update kernel since the last read."""
        ms, n, fl, by = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        _check(self.lib.coru_ctx_profile_rpca_update(self.h, C.byref(ms), C.byref(n), C.byref(fl), C.byref(by)))
        return {"ms": ms.value, "launches": n.value, "flops": fl.value, "bytes": by.value}

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        _check(load_library().coru_comm_unique_id(buf))
        return bytes(buf)

    def init_threadcomm(self, group: "ThreadGroup", rank: int):
        """Join an in-process collective group (ranks = host threads, one context each)."""
        _check(self.lib.coru_ctx_init_threadcomm(self.h, group.h, rank))
        self.rank, self.world = rank, group.world

    def init_comm(self, rank: int, world: int, uid: bytes):
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        _check(self.lib.coru_ctx_init_comm(self.h, rank, world, buf))
        self.rank, self.world = rank, world


class ThreadGroup:
    """coru_threadcomm: the in-process alternative to NCCL for row-sharded decompositions."""

    def __init__(self, world: int):
        self.lib = load_library()
        self.world = world
        self.h = self.lib.coru_threadcomm_create(world)
        if not self.h:
            raise CoruInvalidArgument("world must be >= 1")

    def close(self):
        if getattr(self, "h", None):
            self.lib.coru_threadcomm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _np_dtype_suffix(dt) -> str:
    dt = np.dtype(dt)
    if dt == np.float64:
        return "f64"
    if dt == np.float32:
        return "f32"
    raise CoruInvalidArgument(f"unsupported dtype {dt}")


_CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: torch's default stream reports handle 0


def _torch_sync_stream(ctx: Context, a):
    """Enqueue the library's work on torch's current stream (ordered with the tensors' producers
    and consumers). Handle 0 would select the context's own non-blocking stream instead."""
    import torch
    h = torch.cuda.current_stream(a.device).cuda_stream
    ctx.set_stream(h if h else _CUDA_STREAM_LEGACY)


def corutv(a, ell: int, q: int, variant: DVariant = DVariant.exact, seed: RngSeed = RngSeed(),
           ctx: Optional[Context] = None, m_global: Optional[int] = None) -> UtvApprox:
    """corutv.hpp:79-100. ``a``: numpy (host entry) or CUDA torch tensor (device entry).

    With a communicator on ``ctx`` (``Context.init_comm``), ``a`` is this rank's row block of
    the global ``m_global x n`` matrix and ``u`` holds this rank's rows.
    """
    variant = DVariant(variant)
    if _is_torch(a):
        import torch
        if not a.is_cuda:
            raise CoruInvalidArgument("torch input must be a CUDA tensor (use numpy for host input)")
        if a.dim() != 2 or a.stride(1) != 1:
            raise CoruInvalidArgument("a must be a 2-D row-major (stride(1) == 1) matrix")
        ctx = ctx or default_context(a.device.index or 0)
        m_local, n = a.shape
        m = m_global if m_global is not None else m_local
        sfx = {torch.float64: "f64", torch.float32: "f32"}.get(a.dtype)
        if sfx is None:
            raise CoruInvalidArgument(f"unsupported dtype {a.dtype}")
        ur = m_local if m >= n else m
        u = torch.empty((max(ur, 1), max(ell, 1)), dtype=a.dtype, device=a.device)
        t = torch.empty((max(ell, 1), max(ell, 1)), dtype=a.dtype, device=a.device)
        v = torch.empty((max(n, 1), max(ell, 1)), dtype=a.dtype, device=a.device)
        perm = np.zeros(max(ell, 1), np.int64)
        out = _Utv(u.data_ptr(), max(ell, 1), t.data_ptr(), max(ell, 1), v.data_ptr(), max(ell, 1),
                   perm.ctypes.data, 0, 0)
        _torch_sync_stream(ctx, a)
        _check(getattr(ctx.lib, f"coru_corutv_{sfx}_dev")(ctx.h, a.data_ptr(), m_local, m, n, a.stride(0), ell, q,
                                                           int(variant), seed.seed, seed.stream, C.byref(out)))
        return UtvApprox(u, t, v, ell, q, variant, seed, bool(out.lower), bool(out.conditioning_warning), perm)
    a = np.ascontiguousarray(a)
    if a.ndim != 2:
        raise CoruInvalidArgument("a must be a 2-D matrix")
    sfx = _np_dtype_suffix(a.dtype)
    ctx = ctx or default_context(0)
    m, n = a.shape
    if ell < 1 or ell >= min(m, n) or q < 0:
        # Same checks and order as check_corutv_params; done by the library too.
        _check(getattr(ctx.lib, f"coru_corutv_{sfx}")(ctx.h, None, m, n, ell, q, int(variant), seed.seed,
                                                      seed.stream, None, None, None, None, None, None))
    u = np.empty((m, ell), a.dtype)
    t = np.empty((ell, ell), a.dtype)
    v = np.empty((n, ell), a.dtype)
    perm = np.empty(ell, np.int64)
    lower, warn = C.c_int(), C.c_int()
    _check(getattr(ctx.lib, f"coru_corutv_{sfx}")(ctx.h, a.ctypes.data, m, n, ell, q, int(variant), seed.seed,
                                                  seed.stream, u.ctypes.data, t.ctypes.data, v.ctypes.data,
                                                  perm.ctypes.data, C.byref(lower), C.byref(warn)))
    return UtvApprox(u, t, v, ell, q, variant, seed, bool(lower.value), bool(warn.value), perm)


def sketch_bases(a, ell: int, q: int, seed: RngSeed = RngSeed(), ctx: Optional[Context] = None,
                 m_global: Optional[int] = None) -> SketchBases:
    """detail::sketch_bases (corutv.hpp:49-65), fp64."""
    if _is_torch(a):
        import torch
        ctx = ctx or default_context(a.device.index or 0)
        m_local, n = a.shape
        m = m_global if m_global is not None else m_local
        mk = lambda r: torch.empty((r, ell), dtype=torch.float64, device=a.device)  # noqa: E731
        q1, q2, c1, c2 = mk(m_local), mk(n), mk(m_local), mk(n)
        w = C.c_int()
        _torch_sync_stream(ctx, a)
        _check(ctx.lib.coru_sketch_bases_f64_dev(ctx.h, a.data_ptr(), m_local, m, n, a.stride(0), ell, q, seed.seed,
                                                 seed.stream, q1.data_ptr(), ell, q2.data_ptr(), ell,
                                                 c1.data_ptr(), ell, c2.data_ptr(), ell, C.byref(w)))
        return SketchBases(q1, q2, c1, c2, bool(w.value))
    a = np.ascontiguousarray(a, np.float64)
    ctx = ctx or default_context(0)
    m, n = a.shape
    q1, q2 = np.empty((m, ell)), np.empty((n, ell))
    c1, c2 = np.empty((m, ell)), np.empty((n, ell))
    w = C.c_int()
    _check(ctx.lib.coru_sketch_bases_f64(ctx.h, a.ctypes.data, m, n, ell, q, seed.seed, seed.stream,
                                         q1.ctypes.data, q2.ctypes.data, c1.ctypes.data, c2.ctypes.data,
                                         C.byref(w)))
    return SketchBases(q1, q2, c1, c2, bool(w.value))


def project(a, q1, q2, ctx: Optional[Context] = None):
    """D = (q1^T a) q2 (corutv.hpp:90), summed over ranks; CUDA fp64 tensors."""
    import torch
    ctx = ctx or default_context(a.device.index or 0)
    ell = q1.shape[1]
    d = torch.empty((ell, ell), dtype=torch.float64, device=a.device)
    _torch_sync_stream(ctx, a)
    _check(ctx.lib.coru_project_f64_dev(ctx.h, a.data_ptr(), a.shape[0], a.shape[1], a.stride(0), q1.data_ptr(),
                                        q1.stride(0), q2.data_ptr(), q2.stride(0), ell, d.data_ptr(), ell))
    return d


def gaussian(rows: int, cols: int, seed: RngSeed = RngSeed(), threads: int = 1) -> np.ndarray:
    """rng.hpp:107-112 — host generator of the test matrix Φ, bit-exact with the reference."""
    out = np.empty((rows, cols), np.float64)
    _check(load_library().coru_gaussian(rows, cols, seed.seed, seed.stream, out.ctypes.data, threads))
    return out


def gaussian_device(rows: int, cols: int, seed: RngSeed = RngSeed(), ctx: "Context | None" = None, ld: int | None = None):
    """Device generator of Φ (the CORU_PHI_DEVICE path): a (rows, ld) float64 CUDA tensor whose first
    `cols` columns hold gaussian(rows, cols, seed) and the rest zeros."""
    import torch
    ctx = ctx or default_context()
    ld = ld or cols
    out = torch.empty((rows, ld), dtype=torch.float64, device=f"cuda:{ctx.device}")
    _torch_sync_stream(ctx, out)
    _check(ctx.lib.coru_gaussian_f64_dev(ctx.h, rows, cols, seed.seed, seed.stream, out.data_ptr(), ld))
    return out


def _mm(x, y):
    return x @ y


def _T(x):
    return x.T if not _is_torch(x) else x.transpose(0, 1)


def reconstruct(f: UtvApprox):
    """corutv.hpp:102 — u·t·v^T."""
    return _mm(_mm(f.u, f.t), _T(f.v))


def truncate_rank_k(f: UtvApprox, k: int):
    """corutv.hpp:106-110."""
    if k < 1 or k > f.ell:
        raise CoruInvalidArgument("truncate_rank_k: k out of range")
    if f.lower:
        return _mm(_mm(f.u, f.t[:, :k]), _T(f.v[:, :k]))
    return _mm(_mm(f.u[:, :k], f.t[:k, :]), _T(f.v))


def singular_estimates(f: UtvApprox) -> np.ndarray:
    """corutv.hpp:113-117 — |t_jj|."""
    t = f.t.detach().cpu().numpy() if _is_torch(f.t) else f.t
    return np.abs(np.diag(t)).copy()


# kernel-level entry points (parity tests / benchmarks) ----------------------------------------
def gemm(a, x, op: int = 0, ctx: Optional[Context] = None, out=None):
    """C = op(a)·x on the A-pass kernel (op 0: a·x, op 1: a^T·x); CUDA fp64 or fp32 tensors."""
    import torch
    ctx = ctx or default_context(a.device.index or 0)
    rows = a.shape[0] if op == 0 else a.shape[1]
    K = a.shape[1] if op == 0 else a.shape[0]
    N = x.shape[1]
    c = out if out is not None else torch.empty((rows, N), dtype=a.dtype, device=a.device)
    fn = ctx.lib.coru_gemm_f64_dev if a.dtype == torch.float64 else ctx.lib.coru_gemm_f32_dev
    _torch_sync_stream(ctx, a)
    _check(fn(ctx.h, op, a.data_ptr(), a.stride(0), x.data_ptr(), x.stride(0), c.data_ptr(), c.stride(0), rows, K, N))
    return c


def tsqr(b, ctx: Optional[Context] = None):
    """householder_qr (qr.hpp:85-99) through the TSQR tree; CUDA fp64 tensor, rows > cols."""
    import torch
    ctx = ctx or default_context(b.device.index or 0)
    m, n = b.shape
    q = torch.zeros((m, n), dtype=torch.float64, device=b.device)
    r = torch.empty((n, n), dtype=torch.float64, device=b.device)
    _torch_sync_stream(ctx, b)
    _check(ctx.lib.coru_tsqr_f64_dev(ctx.h, b.data_ptr(), b.stride(0), m, n, q.data_ptr(), n, r.data_ptr(), n))
    return q, r


def qrcp(mat, ctx: Optional[Context] = None):
    """qrcp (qr.hpp:106-143) of a square CUDA fp64 tensor -> (q, r, perm)."""
    import torch
    ctx = ctx or default_context(mat.device.index or 0)
    n = mat.shape[0]
    q = torch.empty((n, n), dtype=torch.float64, device=mat.device)
    r = torch.empty((n, n), dtype=torch.float64, device=mat.device)
    perm = np.empty(n, np.int64)
    _torch_sync_stream(ctx, mat)
    _check(ctx.lib.coru_qrcp_f64_dev(ctx.h, mat.data_ptr(), mat.stride(0), n, q.data_ptr(), n, r.data_ptr(), n,
                                     perm.ctypes.data))
    return q, r, perm


def pinv(mat, ctx: Optional[Context] = None):
    """pinv (svd.hpp:167-187) of a square CUDA fp64 tensor -> (p, sweeps); sweeps = Jacobi sweeps
    used, 0 when the 60-sweep cap was hit (SvdFactors::converged == false)."""
    import torch
    ctx = ctx or default_context(mat.device.index or 0)
    n = mat.shape[0]
    assert mat.shape == (n, n) and mat.dtype == torch.float64 and mat.is_cuda
    out = torch.empty((n, n), dtype=torch.float64, device=mat.device)
    conv = C.c_int(0)
    _torch_sync_stream(ctx, mat)
    _check(ctx.lib.coru_pinv_f64_dev(ctx.h, mat.data_ptr(), mat.stride(0), n, out.data_ptr(), n, C.byref(conv)))
    return out, int(conv.value)


@dataclass
class SvdFactors:
    """SvdFactors (svd.hpp:17-22): u, sigma (non-increasing), v, converged."""
    u: object
    sigma: object
    v: object
    converged: bool


def svd(mat, ctx: Optional[Context] = None) -> SvdFactors:
    """svd (svd.hpp:141-161) of a square CUDA fp64 tensor (the Jacobi kernel of the approx-D core)."""
    import torch
    ctx = ctx or default_context(mat.device.index or 0)
    n = mat.shape[0]
    assert mat.shape == (n, n) and mat.dtype == torch.float64 and mat.is_cuda
    u = torch.empty((n, n), dtype=torch.float64, device=mat.device)
    v = torch.empty((n, n), dtype=torch.float64, device=mat.device)
    s = torch.empty(n, dtype=torch.float64, device=mat.device)
    conv = C.c_int(0)
    _torch_sync_stream(ctx, mat)
    _check(ctx.lib.coru_svd_f64_dev(ctx.h, mat.data_ptr(), mat.stride(0), n, u.data_ptr(), n, s.data_ptr(),
                                    v.data_ptr(), n, C.byref(conv)))
    return SvdFactors(u, s, v, conv.value > 0)


def tsr_svd(a, ell: int, seed: RngSeed = RngSeed(), ctx: Optional[Context] = None) -> SvdFactors:
    """tsr_svd(a, ell, seed) (baselines.hpp:43-56); numpy (host entry) or CUDA torch (device entry)."""
    ctx = ctx or default_context()
    m, n = a.shape
    conv = C.c_int(0)
    if _is_torch(a):
        import torch
        assert a.dtype == torch.float64
        u = torch.empty((m, ell), dtype=torch.float64, device=a.device)
        v = torch.empty((n, ell), dtype=torch.float64, device=a.device)
        s = torch.empty(ell, dtype=torch.float64, device=a.device)
        _torch_sync_stream(ctx, a)
        _check(ctx.lib.coru_tsr_svd_f64_dev(ctx.h, a.data_ptr(), m, n, a.stride(0), ell, seed.seed, seed.stream,
                                            u.data_ptr(), ell, s.data_ptr(), v.data_ptr(), ell, C.byref(conv)))
        return SvdFactors(u, s, v, bool(conv.value))
    a = np.ascontiguousarray(a, np.float64)
    u = np.empty((m, ell)); s = np.empty(ell); v = np.empty((n, ell))
    _check(ctx.lib.coru_tsr_svd_f64(ctx.h, a.ctypes.data, m, n, ell, seed.seed, seed.stream, u.ctypes.data,
                                    s.ctypes.data, v.ctypes.data, C.byref(conv)))
    return SvdFactors(u, s, v, bool(conv.value))


def sor_svd(a, k: int, ell: int, q: int, seed: RngSeed = RngSeed(), ctx: Optional[Context] = None):
    """sor_svd(a, k, ell, q, seed) (baselines.hpp:61-71) -> the m x n rank-k approximation."""
    ctx = ctx or default_context()
    m, n = a.shape
    if _is_torch(a):
        import torch
        assert a.dtype == torch.float64
        out = torch.empty((m, n), dtype=torch.float64, device=a.device)
        _torch_sync_stream(ctx, a)
        _check(ctx.lib.coru_sor_svd_f64_dev(ctx.h, a.data_ptr(), m, n, a.stride(0), k, ell, q, seed.seed, seed.stream,
                                            out.data_ptr(), n))
        return out
    a = np.ascontiguousarray(a, np.float64)
    out = np.empty((m, n))
    _check(ctx.lib.coru_sor_svd_f64(ctx.h, a.ctypes.data, m, n, k, ell, q, seed.seed, seed.stream, out.ctypes.data))
    return out


# ---- robust PCA: alm_rpca with the CoR-UTV inner step (rpca.hpp:53-169) ------------------------
class RpcaInner(enum.IntEnum):
    svt_exact = 0   # rpca.hpp:53 — not provided (CORU_ENOTSUP)
    corutv = 1


class CorutvThresholding(enum.IntEnum):
    soft = 0        # rpca.hpp:58
    hard = 1


class _RpcaConfig(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("mu0", C.c_double), ("rho", C.c_double), ("mu_bar", C.c_double),
                ("tol", C.c_double), ("max_iter", C.c_int), ("inner", C.c_int), ("corutv_ell", C.c_int64),
                ("corutv_q", C.c_int), ("thresholding", C.c_int)]


class _RpcaResult(C.Structure):
    _fields_ = [("iterations", C.c_int), ("residuals", C.c_void_p), ("rank_l", C.c_int64), ("s_l0", C.c_int64),
                ("converged", C.c_int), ("ell_clamped", C.c_int)]


@dataclass
class RpcaConfig:
    """RpcaConfig (rpca.hpp:60-78): same fields and defaults, except inner defaults to corutv (the one
    inner step this build provides)."""
    lambda_: float = 0.0
    mu0: float = 0.0
    rho: float = 1.5
    mu_bar: float = 0.0
    tol: float = 1e-5
    max_iter: int = 50
    inner: RpcaInner = RpcaInner.corutv
    corutv_ell: int = 0
    corutv_q: int = 1
    corutv_thresholding: CorutvThresholding = CorutvThresholding.soft

    def _c(self) -> _RpcaConfig:
        return _RpcaConfig(float(self.lambda_), float(self.mu0), float(self.rho), float(self.mu_bar),
                           float(self.tol), int(self.max_iter), int(self.inner), int(self.corutv_ell),
                           int(self.corutv_q), int(self.corutv_thresholding))


@dataclass
class RpcaResult:
    """RpcaResult (rpca.hpp:80-88)."""
    l: Any
    s: Any
    iterations: int
    residuals: list
    rank_l: int
    s_l0: int
    converged: bool
    ell_clamped: bool


def alm_rpca(m, config: RpcaConfig = RpcaConfig(), seed: RngSeed = RngSeed(),
             ctx: Optional[Context] = None) -> RpcaResult:
    """alm_rpca(m, config, seed) (rpca.hpp:95-169) with the CoR-UTV inner step on the GPU. ``m`` is a numpy
    array (host entry: copies in and out) or a CUDA float64 tensor (device entry)."""
    ctx = ctx or default_context()
    rows, cols = m.shape
    cfg = config._c()
    resid = np.zeros(max(int(config.max_iter), 1))
    res = _RpcaResult()
    res.residuals = resid.ctypes.data
    if _is_torch(m):
        import torch
        assert m.dtype == torch.float64
        l = torch.empty((rows, cols), dtype=torch.float64, device=m.device)
        s = torch.empty((rows, cols), dtype=torch.float64, device=m.device)
        _torch_sync_stream(ctx, m)
        _check(ctx.lib.coru_alm_rpca_f64_dev(ctx.h, m.data_ptr(), rows, cols, m.stride(0), C.byref(cfg), seed.seed,
                                             seed.stream, l.data_ptr(), cols, s.data_ptr(), cols, C.byref(res)))
    else:
        m = np.ascontiguousarray(m, np.float64)
        l = np.empty((rows, cols))
        s = np.empty((rows, cols))
        _check(ctx.lib.coru_alm_rpca_f64(ctx.h, m.ctypes.data, rows, cols, C.byref(cfg), seed.seed, seed.stream,
                                         l.ctypes.data, s.ctypes.data, C.byref(res)))
    return RpcaResult(l, s, res.iterations, list(resid[:res.iterations]), int(res.rank_l), int(res.s_l0),
                      bool(res.converged), bool(res.ell_clamped))


def corutv_ooc(a: np.ndarray, ell: int, q: int, variant: DVariant = DVariant.exact, seed: RngSeed = RngSeed(),
               chunk_rows: int = 0, ctx: Optional[Context] = None) -> UtvApprox:
    """Out-of-core corutv (§8 f4): ``a`` is a host numpy array streamed to the GPU in row chunks
    (coru_corutv_{f64,f32}_ooc); U, T, V come back as numpy arrays."""
    import torch
    ctx = ctx or default_context()
    assert isinstance(a, np.ndarray) and a.dtype in (np.float64, np.float32) and a.strides[1] == a.itemsize
    m, n = a.shape
    sfx = "f64" if a.dtype == np.float64 else "f32"
    tdt = torch.float64 if sfx == "f64" else torch.float32
    dev = torch.device("cuda", ctx.device)
    u = torch.empty((m, ell), dtype=tdt, device=dev)
    t = torch.empty((ell, ell), dtype=tdt, device=dev)
    v = torch.empty((n, ell), dtype=tdt, device=dev)
    perm = np.zeros(ell, np.int64)
    out = _Utv(u.data_ptr(), ell, t.data_ptr(), ell, v.data_ptr(), ell, perm.ctypes.data, 0, 0)
    torch.cuda.synchronize(dev)
    _check(getattr(ctx.lib, f"coru_corutv_{sfx}_ooc")(ctx.h, a.ctypes.data, m, n, a.strides[0] // a.itemsize, ell, q,
                                                     int(variant), seed.seed, seed.stream, chunk_rows, C.byref(out)))
    torch.cuda.synchronize(dev)
    return UtvApprox(u.cpu().numpy(), t.cpu().numpy(), v.cpu().numpy(), ell, q, variant, seed, bool(out.lower),
                     bool(out.conditioning_warning), perm)


class CoruIoError(IOError):
    """coru::IoError (io.hpp): unreadable or malformed CORU file (CORU_EIO)."""


def write_matrix_bin(path: str, a: np.ndarray) -> None:
    """write_matrix_bin (io.hpp:67-77): "CORU", rows, cols (u64 LE), fp64 LE row-major."""
    import struct
    a = np.ascontiguousarray(a, "<f8")
    with open(path, "wb") as f:
        f.write(b"CORU" + struct.pack("<QQ", a.shape[0], a.shape[1]))
        f.write(a.tobytes())


def read_matrix_bin_header(path: str) -> tuple[int, int]:
    r, c = C.c_int64(), C.c_int64()
    _check(load_library().coru_read_matrix_bin_header(path.encode(), C.byref(r), C.byref(c)))
    return r.value, c.value


def corutv_file(path: str, ell: int, q: int, variant: DVariant = DVariant.exact, seed: RngSeed = RngSeed(),
                chunk_rows: int = 0, ctx: Optional[Context] = None) -> UtvApprox:
    """corutv of a CORU binary matrix file, streamed out of core from the memory-mapped file."""
    import torch
    ctx = ctx or default_context()
    m, n = read_matrix_bin_header(path)
    dev = torch.device("cuda", ctx.device)
    u = torch.empty((m, ell), dtype=torch.float64, device=dev)
    t = torch.empty((ell, ell), dtype=torch.float64, device=dev)
    v = torch.empty((n, ell), dtype=torch.float64, device=dev)
    perm = np.zeros(ell, np.int64)
    out = _Utv(u.data_ptr(), ell, t.data_ptr(), ell, v.data_ptr(), ell, perm.ctypes.data, 0, 0)
    torch.cuda.synchronize(dev)
    _check(ctx.lib.coru_corutv_f64_file(ctx.h, path.encode(), ell, q, int(variant), seed.seed, seed.stream, chunk_rows,
                                        C.byref(out)))
    torch.cuda.synchronize(dev)
    return UtvApprox(u.cpu().numpy(), t.cpu().numpy(), v.cpu().numpy(), ell, q, variant, seed, bool(out.lower),
                     bool(out.conditioning_warning), perm)
