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


def test_coru_bin_format_against_reference(tmp_path):
    """write_matrix_bin / read_matrix_bin (io.hpp:67-95): the reference's own files (tests/golden/*.bin)
    parse with the C-ABI header reader and the Python writer produces the reference's bytes."""
    import os
    import paper_1810_07323_b200 as cg
    from golden import HERE
    for name, shape in (("ref_matrix_3x2.bin", (3, 2)), ("ref_gaussian_64x24.bin", (64, 24))):
        path = os.path.join(HERE, name)
        assert cg.read_matrix_bin_header(path) == shape
        raw = open(path, "rb").read()
        a = np.frombuffer(raw[20:], "<f8").reshape(shape)
        mine = tmp_path / name
        cg.write_matrix_bin(str(mine), a)
        assert mine.read_bytes() == raw                       # byte-identical to the reference's writer
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"CORX" + bytes(16) + bytes(8))
    with pytest.raises(cg.CoruIoError):
        cg.read_matrix_bin_header(str(bad))
    trunc = tmp_path / "trunc.bin"
    trunc.write_bytes(open(os.path.join(HERE, "ref_matrix_3x2.bin"), "rb").read()[:-1])
    with pytest.raises(cg.CoruIoError):
        cg.read_matrix_bin_header(str(trunc))
    with pytest.raises(cg.CoruIoError):
        cg.read_matrix_bin_header(str(tmp_path / "missing.bin"))


def test_coru_bin_reference_reader_roundtrip(reference, tmp_path):
    import paper_1810_07323_b200 as cg
    a = np.random.default_rng(1).standard_normal((17, 9))
    p = str(tmp_path / "a.bin")
    cg.write_matrix_bin(p, a)
    assert np.array_equal(reference.read_matrix_bin(p), a)
    a[2, 3] = np.inf
    cg.write_matrix_bin(p, a)
    with pytest.raises(Exception):
        reference.read_matrix_bin(p)                           # IoError: non-finite (io.hpp:90-94)
