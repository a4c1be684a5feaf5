"""The C-ABI library without a GPU: it loads, exports every symbol include/coru_gpu.h declares,
host-side logic (sharding, the bit-exact Gaussian test matrix) works, and compute entry points
fail loudly (no CPU fallback) when no sm_100 device is visible."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "coru_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(coru_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_1810_07323_b200 as cg
    lib = C.CDLL(cg.library_path())
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_abi_version():
    import paper_1810_07323_b200 as cg
    assert cg.load_library().coru_abi_version() == 1


def test_shard_rows_partition():
    import paper_1810_07323_b200 as cg
    for m in (1000, 4000, 200000, 32768, 7):
        for world in (1, 2, 4, 8):
            if m < world:
                continue
            spans = [cg.shard_rows(m, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (a0, n0), (a1, _) in zip(spans, spans[1:]):
                assert a0 + n0 == a1
            assert sum(n for _, n in spans) == m
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1


def test_host_gaussian_bitexact_with_reference_fixtures():
    """The product's host Φ generator (rng_host.cpp) against the reference's gaussian()."""
    import paper_1810_07323_b200 as cg
    from golden import kat
    k = kat()
    assert np.array_equal(cg.gaussian(7, 9, cg.RngSeed(42, 3)), k["gaussian_7x9_42_3"])
    assert np.array_equal(cg.gaussian(100, 100, cg.RngSeed(42, 0), threads=8), k["gaussian_100x100_42_0"])
    assert np.array_equal(cg.gaussian(1, 5, cg.RngSeed(7, 0)), k["gaussian_1x5_7_0"])


def test_host_gaussian_threads_bitexact(oracle):
    import paper_1810_07323_b200 as cg
    for thr in (1, 3, 8):
        assert np.array_equal(cg.gaussian(4001, 61, cg.RngSeed(5, 2), threads=thr), oracle.gaussian(4001, 61, 5, 2))


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1810_07323_b200 as cg
    with pytest.raises(cg.CoruError):
        cg.Context(0)


def test_invalid_arguments_before_device():
    """EINVAL for the reference's parameter errors even before any device work."""
    import paper_1810_07323_b200 as cg
    lib = cg.load_library()
    rc = lib.coru_gaussian(0, 3, 1, 0, None, 1)
    assert rc == cg.CORU_EINVAL


def test_rpca_config_validation_before_device():
    """RpcaConfig::validate (rpca.hpp:72-77) and the svt_exact ENOTSUP are reported before device work."""
    import ctypes as C
    import paper_1810_07323_b200 as cg
    lib = cg.load_library()
    cfg = cg.RpcaConfig(corutv_ell=4)
    assert cfg.rho == 1.5 and cfg.tol == 1e-5 and cfg.max_iter == 50 and cfg.corutv_q == 1
    c = cg._RpcaConfig()
    lib.coru_rpca_config_default(C.byref(c))
    assert (c.rho, c.tol, c.max_iter, c.corutv_q, c.inner, c.thresholding) == (1.5, 1e-5, 50, 1, 1, 0)
