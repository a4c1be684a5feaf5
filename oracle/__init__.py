"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes front-end for the two CPU checkers of the CoR-UTV hot path:

* ``Oracle`` — ``liboracle.so``, the plain-C restatement in ``coru_oracle.c`` (fp64 and
  fp32), each function citing the reference file:line it follows.
* ``Reference`` — ``_ref/libcoru_ref.so``, the unmodified reference headers
  (``/root/reference/proj/include/coru``) compiled by ``oracle/Makefile`` behind a C-ABI.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package, and only as the checker / CPU baseline.
The product package ``paper_1810_07323_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
# the same restatement built with FMA contraction: SURVEY.md §8c protocol 2 (implementation floor)
ORACLE_FMA_SO = os.path.join(HERE, "liboracle_fma.so")
REF_SO = os.path.join(HERE, "_ref", "libcoru_ref.so")

_i64, _u64, _int, _dbl = C.c_int64, C.c_uint64, C.c_int, C.c_double
_p = C.c_void_p


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_p)


def build(quiet: bool = True) -> None:
    """Compile the checkers (oracle/Makefile). The reference part only where /root/reference exists."""
    import subprocess

    subprocess.run(["make", "-C", HERE, "all"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


@dataclass
class Utv:
    u: np.ndarray
    t: np.ndarray
    v: np.ndarray
    lower: bool
    conditioning_warning: bool
    perm: np.ndarray | None = None


class CoruError(ValueError):
    """Mirrors the reference's std::invalid_argument."""


class Oracle:
    """The plain-C restatement (liboracle.so)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = L = C.CDLL(path)
        L.oracle_gaussian.argtypes = [_i64, _i64, _u64, _u64, _p]
        L.oracle_xoshiro_words.argtypes = [_u64, _u64, _i64, _p]
        L.oracle_max_threads.restype = _int
        L.oracle_pinv_f64.argtypes = [_p, _i64, _p]
        L.oracle_svd_square_f64.argtypes = [_p, _i64, _p, _p, _p]
        L.oracle_svd_square_f64.restype = _int
        L.oracle_tsr_svd_f64.argtypes = [_p, _i64, _i64, _i64, _u64, _u64, _int, _p, _p, _p, _p]
        L.oracle_sor_svd_f64.argtypes = [_p, _i64, _i64, _i64, _i64, _int, _u64, _u64, _int, _p]
        L.oracle_jacobi_svd_square.argtypes = [_p, _i64, _p, _p, _p]
        L.oracle_jacobi_svd_square.restype = _int
        for sfx in ("f64", "f32", "f80"):
            getattr(L, f"oracle_matmul_{sfx}").argtypes = [_p, _i64, _i64, _p, _i64, _p, _int]
            getattr(L, f"oracle_matmul_tn_{sfx}").argtypes = [_p, _i64, _i64, _p, _i64, _p, _int]
            getattr(L, f"oracle_householder_qr_{sfx}").argtypes = [_p, _i64, _i64, _p, _p]
            getattr(L, f"oracle_qrcp_{sfx}").argtypes = [_p, _i64, _i64, _p, _p, _p]
            getattr(L, f"oracle_sketch_bases_{sfx}").argtypes = [
                _p, _i64, _i64, _i64, _int, _u64, _u64, _int, _p, _p, _p, _p, _p]
            getattr(L, f"oracle_corutv_{sfx}").argtypes = [
                _p, _i64, _i64, _i64, _int, _int, _u64, _u64, _int, _p, _p, _p, _p, _p]

    @staticmethod
    def _sfx(dtype):
        dt = np.dtype(dtype)
        if dt == np.float64:
            return "f64"
        if dt == np.longdouble and dt.itemsize == 16:
            return "f80"
        return "f32"

    def max_threads(self) -> int:
        return self.lib.oracle_max_threads()

    def gaussian(self, rows: int, cols: int, seed: int, stream: int = 0) -> np.ndarray:
        out = np.empty((rows, cols), np.float64)
        self.lib.oracle_gaussian(rows, cols, seed, stream, _ptr(out))
        return out

    def xoshiro_words(self, seed: int, stream: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        self.lib.oracle_xoshiro_words(seed, stream, count, _ptr(out))
        return out

    def matmul(self, a, b, threads=1):
        a = np.ascontiguousarray(a); b = np.ascontiguousarray(b, a.dtype)
        c = np.empty((a.shape[0], b.shape[1]), a.dtype)
        getattr(self.lib, f"oracle_matmul_{self._sfx(a.dtype)}")(
            _ptr(a), a.shape[0], a.shape[1], _ptr(b), b.shape[1], _ptr(c), threads)
        return c

    def matmul_tn(self, a, y, threads=1):
        """a^T · y in the order of matmul(a.transposed(), y)."""
        a = np.ascontiguousarray(a); y = np.ascontiguousarray(y, a.dtype)
        c = np.empty((a.shape[1], y.shape[1]), a.dtype)
        getattr(self.lib, f"oracle_matmul_tn_{self._sfx(a.dtype)}")(
            _ptr(a), a.shape[0], a.shape[1], _ptr(y), y.shape[1], _ptr(c), threads)
        return c

    def householder_qr(self, a):
        a = np.ascontiguousarray(a); m, n = a.shape
        q = np.empty((m, n), a.dtype); r = np.empty((n, n), a.dtype)
        if getattr(self.lib, f"oracle_householder_qr_{self._sfx(a.dtype)}")(_ptr(a), m, n, _ptr(q), _ptr(r)):
            raise CoruError("householder_qr: requires rows >= cols")
        return q, r

    def qrcp(self, a):
        a = np.ascontiguousarray(a); m, n = a.shape
        q = np.empty((m, n), a.dtype); r = np.empty((n, n), a.dtype); perm = np.empty(n, np.int64)
        if getattr(self.lib, f"oracle_qrcp_{self._sfx(a.dtype)}")(_ptr(a), m, n, _ptr(q), _ptr(r), _ptr(perm)):
            raise CoruError("qrcp: requires rows >= cols")
        return q, r, perm

    def pinv(self, a):
        """pinv of a square matrix (svd.hpp:167-187), fp64 Jacobi SVD."""
        a = np.ascontiguousarray(a, np.float64); n = a.shape[0]
        assert a.shape == (n, n)
        out = np.empty((n, n))
        self.lib.oracle_pinv_f64(_ptr(a), n, _ptr(out))
        return out

    def svd_square(self, a):
        """svd (svd.hpp:141-161) of a square matrix: (u, sigma, v, converged)."""
        a = np.ascontiguousarray(a, np.float64); n = a.shape[0]
        u = np.empty((n, n)); v = np.empty((n, n)); s = np.empty(n)
        conv = self.lib.oracle_svd_square_f64(_ptr(a), n, _ptr(u), _ptr(s), _ptr(v))
        return u, s, v, bool(conv)

    def tsr_svd(self, a, ell, seed, stream=0, threads=1):
        """tsr_svd (baselines.hpp:43-56) -> (u, sigma, v, converged)."""
        a = np.ascontiguousarray(a, np.float64); m, n = a.shape
        u = np.empty((m, ell)); s = np.empty(ell); v = np.empty((n, ell)); conv = np.zeros(1, np.int32)
        if self.lib.oracle_tsr_svd_f64(_ptr(a), m, n, ell, seed, stream, threads, _ptr(u), _ptr(s), _ptr(v), _ptr(conv)):
            raise CoruError("tsr_svd: ell out of range")
        return u, s, v, bool(conv[0])

    def sor_svd(self, a, k, ell, q, seed, stream=0, threads=1):
        """sor_svd (baselines.hpp:61-71) -> m x n."""
        a = np.ascontiguousarray(a, np.float64); m, n = a.shape
        out = np.empty((m, n))
        if self.lib.oracle_sor_svd_f64(_ptr(a), m, n, k, ell, q, seed, stream, threads, _ptr(out)):
            raise CoruError("sor_svd: bad parameters")
        return out

    def jacobi_svd_square(self, a):
        """detail::jacobi_svd_square (svd.hpp:31-134) on a square a: (u, sigma, v, converged)."""
        a = np.ascontiguousarray(a, np.float64); n = a.shape[0]
        acm = np.ascontiguousarray(a.T)
        u = np.empty((n, n)); v = np.empty((n, n)); s = np.empty(n)
        conv = self.lib.oracle_jacobi_svd_square(_ptr(acm), n, _ptr(u), _ptr(s), _ptr(v))
        return u, s, v, bool(conv)

    def sketch_bases(self, a, ell, q, seed, stream=0, threads=1):
        a = np.ascontiguousarray(a); m, n = a.shape; dt = a.dtype
        q1 = np.empty((m, ell), dt); q2 = np.empty((n, ell), dt)
        c1 = np.empty((m, ell), dt); c2p = np.empty((n, ell), dt); w = np.zeros(1, np.int32)
        rc = getattr(self.lib, f"oracle_sketch_bases_{self._sfx(dt)}")(
            _ptr(a), m, n, ell, q, seed, stream, threads, _ptr(q1), _ptr(q2), _ptr(c1), _ptr(c2p), _ptr(w))
        if rc:
            raise CoruError("sketch_bases: bad parameters")
        return q1, q2, c1, c2p, bool(w[0])

    def corutv(self, a, ell, q, variant=0, seed=0, stream=0, threads=1) -> Utv:
        a = np.ascontiguousarray(a); m, n = a.shape; dt = a.dtype
        u = np.empty((m, ell), dt); t = np.empty((ell, ell), dt); v = np.empty((n, ell), dt)
        flags = np.zeros(2, np.int32); perm = np.empty(ell, np.int64)
        if ell < 1 or ell >= min(m, n) or q < 0:
            raise CoruError("corutv: bad parameters")
        rc = getattr(self.lib, f"oracle_corutv_{self._sfx(dt)}")(
            _ptr(a), m, n, ell, q, variant, seed, stream, threads, _ptr(u), _ptr(t), _ptr(v), _ptr(flags), _ptr(perm))
        if rc == 1:
            raise CoruError("corutv: bad parameters")
        return Utv(u, t, v, bool(flags[0]), bool(flags[1]), perm)


    # ---- alm_rpca with the CoR-UTV inner step: a numpy restatement of rpca.hpp:95-169 over the C
    # restatement's sketch_bases / corutv / matmul / Jacobi SVD (bit-exact with the reference, pinned in
    # tests/test_oracle.py against oracle/_ref and tests/golden/rpca_ref_cases.npz).
    @staticmethod
    def frobenius(a):
        """frobenius_norm (matrix.hpp:133-137): serial left-to-right sum of squares (np.cumsum is serial)."""
        a = np.ascontiguousarray(a, np.float64).ravel()
        return float(np.sqrt(np.cumsum(a * a)[-1])) if a.size else 0.0

    def singular_values(self, a):
        """svd(a).sigma (svd.hpp:140-162): the Jacobi SVD of R from householder_qr when rows > cols, of a^T
        when rows < cols."""
        a = np.ascontiguousarray(a, np.float64)
        if a.shape[0] < a.shape[1]:
            a = np.ascontiguousarray(a.T)
        if a.shape[0] > a.shape[1]:
            a = self.householder_qr(a)[1]
        return self.jacobi_svd_square(a)[1]

    def alm_rpca(self, mat, lambda_=0.0, mu0=0.0, rho=1.5, mu_bar=0.0, tol=1e-5, max_iter=50, inner=1,
                 corutv_ell=0, corutv_q=1, thresholding=0, seed=0, stream=0):
        """alm_rpca (rpca.hpp:95-169), inner = corutv (rpca.hpp:121-140)."""
        if rho <= 1.0 or tol <= 0.0 or max_iter < 1 or corutv_q < 0:
            raise CoruError("RpcaConfig: invalid")                       # rpca.hpp:72-77
        if inner != 1:
            raise NotImplementedError("svt_exact inner is not restated")
        mat = np.ascontiguousarray(mat, np.float64)
        rows, cols = mat.shape
        lam = lambda_ if lambda_ > 0.0 else 1.0 / np.sqrt(float(max(rows, cols)))
        m_fro = self.frobenius(mat)
        mu = mu0 if mu0 > 0.0 else 1.25 / float(self.singular_values(mat)[0])
        mub = mu_bar if mu_bar > 0.0 else mu * 1e7
        l = np.zeros_like(mat); s = np.zeros_like(mat); y = np.zeros_like(mat)
        residuals = []; rank_l = 0; converged = False; clamped = False; it = 0
        while it < max_iter:
            it += 1
            inv_mu = 1.0 / mu
            x = mat - s
            x += y * inv_mu                                               # rpca.hpp:114-115
            if corutv_ell:
                ell = corutv_ell
            else:                                                         # predict_rank (rpca.hpp:45-51)
                fro = self.frobenius(x)
                if fro == 0.0:
                    k = 0
                else:
                    sig = self.singular_values(x)
                    nuc = float(np.cumsum(sig)[-1])
                    kk = np.ceil((nuc / fro) * (nuc / fro) - 1e-9)
                    k = 1 if kk < 1.0 else int(kk)
                ell = k + 2
            ell_max = min(rows, cols) - 1
            if ell > ell_max:
                ell = ell_max; clamped = True
            ell = max(ell, 1)
            if thresholding == 1:                                         # cor_threshold (corutv.hpp:124-134)
                f = self.corutv(x, ell, corutv_q, 0, seed, stream + it)
                est = np.abs(np.diag(f.t))
                r = int(np.sum(est > inv_mu))
                if r == 0:
                    l = np.zeros_like(mat)
                elif f.lower:                                             # truncate_rank_k (:106-110)
                    l = self.matmul(self.matmul(f.u, np.ascontiguousarray(f.t[:, :r])), np.ascontiguousarray(f.v[:, :r].T))
                else:
                    l = self.matmul(self.matmul(np.ascontiguousarray(f.u[:, :r]), np.ascontiguousarray(f.t[:r, :])),
                                    np.ascontiguousarray(f.v.T))
            else:                                                         # rpca.hpp:135-139
                q1, q2, _, _, _ = self.sketch_bases(x, ell, corutv_q, seed, stream + it)
                d = self.matmul(self.matmul(np.ascontiguousarray(q1.T), x), q2)
                u, sg, v, _ = self.svd_square(d)                          # svt (rpca.hpp:30-40)
                r = 0
                while r < len(sg) and sg[r] > inv_mu:
                    r += 1
                if r == 0:
                    l = np.zeros_like(mat)
                else:
                    us = u[:, :r] * (sg[:r] - inv_mu)
                    dthr = self.matmul(np.ascontiguousarray(us), np.ascontiguousarray(v[:, :r].T))
                    l = self.matmul(self.matmul(q1, dthr), np.ascontiguousarray(q2.T))
            rank_l = r
            w = mat - l
            w += y * inv_mu                                               # rpca.hpp:143-144
            mag = np.abs(w) - lam * inv_mu                                # shrink (rpca.hpp:17-26)
            s = np.where(mag > 0.0, np.where(w > 0.0, mag, -mag), 0.0)
            resid = mat - l
            resid -= s
            y += mu * resid
            mu = min(rho * mu, mub)
            zeta = self.frobenius(resid) / m_fro
            residuals.append(zeta)
            if zeta < tol:
                converged = True
                break
        return dict(l=l, s=s, iterations=it, residuals=np.array(residuals), rank_l=rank_l,
                    s_l0=int(np.count_nonzero(s)), converged=converged, ell_clamped=clamped)


class Reference:
    """The reference library itself, compiled from /root/reference headers (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build it here with `make -C oracle ref`")
        self.lib = L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_gaussian.argtypes = [_i64, _i64, _u64, _u64, _p]
        L.ref_xoshiro_words.argtypes = [_u64, _u64, _i64, _p]
        L.ref_matmul.argtypes = [_p, _i64, _i64, _p, _i64, _p]
        L.ref_householder_qr.argtypes = [_p, _i64, _i64, _p, _p]
        L.ref_qrcp.argtypes = [_p, _i64, _i64, _p, _p, _p]
        L.ref_svd.argtypes = [_p, _i64, _i64, _p, _p, _p, _p]
        L.ref_pinv.argtypes = [_p, _i64, _i64, _p]
        L.ref_tsr_svd.argtypes = [_p, _i64, _i64, _i64, _u64, _u64, _p, _p, _p, _p]
        L.ref_sor_svd.argtypes = [_p, _i64, _i64, _i64, _i64, _int, _u64, _u64, _p]
        L.ref_corutv.argtypes = [_p, _i64, _i64, _i64, _int, _int, _u64, _u64, _p, _p, _p, _p]
        L.ref_corutv_mt.argtypes = [_p, _i64, _i64, _i64, _int, _u64, _u64, _int, _p, _p, _p, _p]
        L.ref_sketch_bases.argtypes = [_p, _i64, _i64, _i64, _int, _u64, _u64, _p, _p, _p, _p, _p]
        L.ref_gen_fast_decay.argtypes = [_i64, _i64, _u64, _u64, _p]
        L.ref_gen_noisy_lowrank.argtypes = [_i64, _i64, _dbl, _u64, _u64, _p]
        L.ref_corutv_batch.argtypes = [_p, _i64, _i64, _i64, _int, _u64, _u64, _int, _int]
        L.ref_corutv_batch.restype = _dbl
        L.ref_frobenius.argtypes = [_p, _i64, _i64]
        L.ref_frobenius.restype = _dbl
        L.ref_write_matrix_bin.argtypes = [C.c_char_p, _p, _i64, _i64]
        L.ref_read_matrix_bin.argtypes = [C.c_char_p, _p, _p, _p]
        L.ref_alm_rpca.argtypes = [_p, _i64, _i64, _p, _p, _u64, _u64, _p, _p, _p, _p]
        L.ref_gen_rpca_instance.argtypes = [_i64, _i64, _u64, _dbl, _u64, _u64, _p, _p, _p]
        L.ref_spectral_norm.argtypes = [_p, _i64, _i64]
        L.ref_spectral_norm.restype = _dbl

    def _check(self, rc):
        if rc == 1:
            raise CoruError(self.lib.ref_last_error().decode())
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def gaussian(self, rows, cols, seed, stream=0):
        out = np.empty((rows, cols), np.float64)
        self._check(self.lib.ref_gaussian(rows, cols, seed, stream, _ptr(out)))
        return out

    def xoshiro_words(self, seed, stream, count):
        out = np.empty(count, np.uint64)
        self.lib.ref_xoshiro_words(seed, stream, count, _ptr(out))
        return out

    def matmul(self, a, b):
        a = np.ascontiguousarray(a, np.float64); b = np.ascontiguousarray(b, np.float64)
        c = np.empty((a.shape[0], b.shape[1]))
        self._check(self.lib.ref_matmul(_ptr(a), a.shape[0], a.shape[1], _ptr(b), b.shape[1], _ptr(c)))
        return c

    def svd(self, a):
        a = np.ascontiguousarray(a, np.float64); m, n = a.shape; r = min(m, n)
        u = np.empty((m, r)); s = np.empty(r); v = np.empty((n, r)); conv = np.zeros(1, np.int32)
        self._check(self.lib.ref_svd(_ptr(a), m, n, _ptr(u), _ptr(s), _ptr(v), _ptr(conv)))
        return u, s, v, bool(conv[0])

    def tsr_svd(self, a, ell, seed, stream=0):
        a = np.ascontiguousarray(a, np.float64); m, n = a.shape
        u = np.empty((m, ell)); s = np.empty(ell); v = np.empty((n, ell)); conv = np.zeros(1, np.int32)
        self._check(self.lib.ref_tsr_svd(_ptr(a), m, n, ell, seed, stream, _ptr(u), _ptr(s), _ptr(v), _ptr(conv)))
        return u, s, v, bool(conv[0])

    def sor_svd(self, a, k, ell, q, seed, stream=0):
        a = np.ascontiguousarray(a, np.float64); m, n = a.shape
        out = np.empty((m, n))
        self._check(self.lib.ref_sor_svd(_ptr(a), m, n, k, ell, q, seed, stream, _ptr(out)))
        return out

    def pinv(self, a):
        a = np.ascontiguousarray(a, np.float64); m, n = a.shape
        out = np.empty((n, m))
        self._check(self.lib.ref_pinv(_ptr(a), m, n, _ptr(out)))
        return out

    def householder_qr(self, a):
        a = np.ascontiguousarray(a, np.float64); m, n = a.shape
        q = np.empty((m, n)); r = np.empty((n, n))
        self._check(self.lib.ref_householder_qr(_ptr(a), m, n, _ptr(q), _ptr(r)))
        return q, r

    def qrcp(self, a):
        a = np.ascontiguousarray(a, np.float64); m, n = a.shape
        q = np.empty((m, n)); r = np.empty((n, n)); perm = np.empty(n, np.int64)
        self._check(self.lib.ref_qrcp(_ptr(a), m, n, _ptr(q), _ptr(r), _ptr(perm)))
        return q, r, perm

    def corutv(self, a, ell, q, variant=0, seed=0, stream=0, threads=1) -> Utv:
        a = np.ascontiguousarray(a, np.float64); m, n = a.shape
        u = np.empty((m, ell)); t = np.empty((ell, ell)); v = np.empty((n, ell)); flags = np.zeros(2, np.int32)
        if threads > 1 and m >= n and variant == 0:
            self._check(self.lib.ref_corutv_mt(_ptr(a), m, n, ell, q, seed, stream, threads,
                                               _ptr(u), _ptr(t), _ptr(v), _ptr(flags)))
        else:
            self._check(self.lib.ref_corutv(_ptr(a), m, n, ell, q, variant, seed, stream,
                                            _ptr(u), _ptr(t), _ptr(v), _ptr(flags)))
        return Utv(u, t, v, bool(flags[0]), bool(flags[1]))

    def corutv_batch(self, a, ell, q, seed, stream0, count, threads):
        """`count` unchanged corutv calls fanned out over `threads` threads; returns a checksum."""
        a = np.ascontiguousarray(a, np.float64); m, n = a.shape
        return self.lib.ref_corutv_batch(_ptr(a), m, n, ell, q, seed, stream0, count, threads)

    def sketch_bases(self, a, ell, q, seed, stream=0):
        a = np.ascontiguousarray(a, np.float64); m, n = a.shape
        q1 = np.empty((m, ell)); q2 = np.empty((n, ell)); c1 = np.empty((m, ell)); c2p = np.empty((n, ell))
        w = np.zeros(1, np.int32)
        self._check(self.lib.ref_sketch_bases(_ptr(a), m, n, ell, q, seed, stream,
                                              _ptr(q1), _ptr(q2), _ptr(c1), _ptr(c2p), _ptr(w)))
        return q1, q2, c1, c2p, bool(w[0])

    def gen_fast_decay(self, n, k, seed, stream=0):
        out = np.empty((n, n))
        self._check(self.lib.ref_gen_fast_decay(n, k, seed, stream, _ptr(out)))
        return out

    def gen_noisy_lowrank(self, n, k, gap, seed, stream=0):
        out = np.empty((n, n))
        self._check(self.lib.ref_gen_noisy_lowrank(n, k, gap, seed, stream, _ptr(out)))
        return out

    def frobenius(self, a):
        a = np.ascontiguousarray(a, np.float64)
        return self.lib.ref_frobenius(_ptr(a), a.shape[0], a.reshape(a.shape[0], -1).shape[1])


    def alm_rpca(self, mat, lambda_=0.0, mu0=0.0, rho=1.5, mu_bar=0.0, tol=1e-5, max_iter=50, inner=1,
                 corutv_ell=0, corutv_q=1, thresholding=0, seed=0, stream=0):
        """coru::alm_rpca (rpca.hpp:95-169); inner 1 = corutv, thresholding 0 = soft / 1 = hard."""
        mat = np.ascontiguousarray(mat, np.float64)
        m, n = mat.shape
        cfg = np.array([lambda_, mu0, rho, mu_bar, tol], np.float64)
        icfg = np.array([max_iter, inner, corutv_ell, corutv_q, thresholding], np.int64)
        l, s = np.empty((m, n)), np.empty((m, n))
        res = np.zeros(max_iter)
        out = np.zeros(5, np.int64)
        self._check(self.lib.ref_alm_rpca(_ptr(mat), m, n, _ptr(cfg), _ptr(icfg), seed, stream, _ptr(l), _ptr(s),
                                          _ptr(res), _ptr(out)))
        it = int(out[0])
        return dict(l=l, s=s, iterations=it, residuals=res[:it].copy(), rank_l=int(out[1]), s_l0=int(out[2]),
                    converged=bool(out[3]), ell_clamped=bool(out[4]))

    def gen_rpca_instance(self, n, r, s, amplitude, seed, stream=0):
        """coru::gen_rpca_instance (testgen.hpp:86-109) -> (m, l_true, s_true)."""
        m, l, sp = np.empty((n, n)), np.empty((n, n)), np.empty((n, n))
        self._check(self.lib.ref_gen_rpca_instance(n, r, s, amplitude, seed, stream, _ptr(m), _ptr(l), _ptr(sp)))
        return m, l, sp

    def write_matrix_bin(self, path, a):
        a = np.ascontiguousarray(a, np.float64)
        self._check(self.lib.ref_write_matrix_bin(path.encode(), _ptr(a), a.shape[0], a.shape[1]))

    def read_matrix_bin(self, path):
        """read_matrix_bin (io.hpp:79-95); raises on malformed files like the reference (IoError)."""
        mn = np.zeros(2, np.int64)
        self._check(self.lib.ref_read_matrix_bin(path.encode(), _ptr(mn[:1]), _ptr(mn[1:]), None))
        out = np.empty((int(mn[0]), int(mn[1])))
        self._check(self.lib.ref_read_matrix_bin(path.encode(), _ptr(mn[:1]), _ptr(mn[1:]), _ptr(out)))
        return out

    def spectral_norm(self, a):
        a = np.ascontiguousarray(a, np.float64)
        return self.lib.ref_spectral_norm(_ptr(a), a.shape[0], a.shape[1])


def has_reference() -> bool:
    return os.path.exists(REF_SO)
