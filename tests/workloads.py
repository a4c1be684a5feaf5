"""Synthetic BASELINE workloads, shared by tests and bench.py.

No public dataset is involved; each config is regenerated from a fixed seed:
X, Y are Haar factors (Q of the QR of seeded N(0,1) matrices with diag(R) > 0), A = X·diag(σ)·Y^T + E.
Small configs (C1, C2, scaled variants) are generated with numpy PCG64 on the host so the GPU path
and the CPU oracle see identical bytes; full-size C3-C5 are generated on the GPU with torch
(seeded CUDA generator) and only ever checked through size-independent properties.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    d: int
    q: int
    k: int
    dtype: str  # "f64" | "f32"
    desc: str


CONFIGS = {
    "C1": Config("C1", 1000, 1000, 25, 0, 20, "f64", "rank-20 Haar, sigma=1, E ~ N(0,1)*1e-3/sqrt(1000)"),
    "C2q1": Config("C2q1", 4000, 4000, 60, 1, 50, "f64", "sigma_i = i^-2, full Haar"),
    "C2q2": Config("C2q2", 4000, 4000, 60, 2, 50, "f64", "sigma_i = i^-2, full Haar"),
    "C3": Config("C3", 200000, 2000, 110, 1, 100, "f64", "sigma_i = 10^(-i/20), full rank, Haar"),
    "C4": Config("C4", 32768, 32768, 220, 2, 200, "f64",
                 "rank-200 Haar, sigma 100->1 linear, E iid N(0, var 1e-4)"),
    "C5": Config("C5", 65536, 65536, 520, 2, 500, "f32",
                 "sigma_i = 1/(1+i/50) i<=2000, Haar, E iid N(0, var 1e-6)"),
}


def haar_np(rng, n, k):
    q, r = np.linalg.qr(rng.standard_normal((n, k)))
    return q * np.sign(np.diag(r))


def spectrum(name: str, count: int) -> np.ndarray:
    i = np.arange(1, count + 1, dtype=np.float64)
    if name == "C1":
        return np.ones(count)
    if name.startswith("C2"):
        return i ** -2.0
    if name.startswith("C3"):
        return 10.0 ** (-i / 20.0)
    if name.startswith("C4"):
        return np.linspace(100.0, 1.0, count)
    if name.startswith("C5"):
        return 1.0 / (1.0 + i / 50.0)
    raise KeyError(name)


def make_host(name: str, m: int | None = None, n: int | None = None, seed: int = 0) -> np.ndarray:
    """Host (numpy) generator; m, n override the size for shape-scaled variants."""
    c = CONFIGS[name]
    m = m or c.m
    n = n or c.n
    rng = np.random.default_rng(1000 + seed + sum(map(ord, name)))
    if name == "C1":
        r = 20
        x, y = haar_np(rng, m, r), haar_np(rng, n, r)
        a = (x * spectrum(name, r)) @ y.T
        a += rng.standard_normal((m, n)) * (1e-3 / np.sqrt(1000.0))
        return a
    if name.startswith("C4"):
        r = 200
        x, y = haar_np(rng, m, r), haar_np(rng, n, r)
        return (x * spectrum(name, r)) @ y.T + rng.standard_normal((m, n)) * 1e-2
    if name.startswith("C5"):
        r = min(2000, min(m, n))
        x, y = haar_np(rng, m, r), haar_np(rng, n, r)
        a = (x * spectrum(name, r)) @ y.T + rng.standard_normal((m, n)) * 1e-3
        return a.astype(np.float32)
    r = min(m, n)
    x, y = haar_np(rng, m, r), haar_np(rng, n, r)
    return (x * spectrum(name, r)) @ y.T


def make_device(name: str, device="cuda", seed: int = 0, m: int | None = None, n: int | None = None):
    """GPU (torch) generator for full-size configs; deterministic for a given GPU type."""
    import torch
    c = CONFIGS[name]
    m = m or c.m
    n = n or c.n
    g = torch.Generator(device=device)
    g.manual_seed(1000 + seed + sum(map(ord, name)))

    def haar(rows, k):
        z = torch.randn(rows, k, dtype=torch.float64, device=device, generator=g)
        q, r = torch.linalg.qr(z)
        return q * torch.sign(torch.diagonal(r))

    if name == "C1":
        r = 20
        sig = torch.ones(r, dtype=torch.float64, device=device)
        noise = 1e-3 / np.sqrt(1000.0)
    elif name.startswith("C4"):
        r = 200
        sig = torch.linspace(100.0, 1.0, r, dtype=torch.float64, device=device)
        noise = 1e-2
    elif name.startswith("C5"):
        r = min(2000, m, n)
        sig = torch.from_numpy(spectrum(name, r)).to(device)
        noise = 1e-3
    else:
        r = min(m, n)
        sig = torch.from_numpy(spectrum(name, r)).to(device)
        noise = 0.0
    x = haar(m, r)
    y = haar(n, r)
    a = (x * sig) @ y.T
    del x, y
    if noise:
        a.add_(torch.randn(m, n, dtype=torch.float64, device=device, generator=g), alpha=noise)
    if c.dtype == "f32":
        a = a.float()
    return a


def sha256(a) -> str:
    if type(a).__module__.startswith("torch"):
        a = a.detach().cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
