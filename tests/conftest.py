"""Shared fixtures. `gpu` tests need a B200 (run through gpurun); everything else runs on CPU."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device (B200)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import Reference, has_reference
    if not has_reference():
        pytest.skip("oracle/_ref/libcoru_ref.so not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1810_07323_b200 as cg
    return cg.Context(0)


def haar(rng, n, k):
    """Haar-random n x k orthonormal factor: Q of QR(N(0,1)) with diag(R) > 0."""
    q, r = np.linalg.qr(rng.standard_normal((n, k)))
    return q * np.sign(np.diag(r))


def rel_recon_error(a, u, t, v):
    """||A - U T V^T||_F / ||A||_F computed explicitly (never through ||A||^2 - ||T||^2)."""
    return np.linalg.norm(a - (u @ t) @ v.T) / np.linalg.norm(a)


def orth_residual(q):
    """||Q^T Q - I||_F (tests/oracles.hpp:133-137)."""
    g = q.T @ q
    return np.linalg.norm(g - np.eye(g.shape[0]))
