"""Seeded synthetic instances for the five BASELINE.json configs.

CPU generator (numpy PCG64) for parity tests — the same bits go to the GPU and
to the CPU checkers — and a GPU generator (torch, cuSOLVER QR) for the
n = 32768 benchmark instance, which numpy cannot factor in reasonable time.
Q is always the Q factor of a QR of an N(0,1) matrix with diag(R) > 0
(proj/src/core.cpp:58-60), so A = Q diag(lambda) Q^T with Q Haar-orthogonal.
"""
from __future__ import annotations

import math

import numpy as np

CONFIGS = {
    0: dict(n=512, k=2, signs=(1, 1), name="cfg0 rank-2 n=512"),
    1: dict(n=4096, k=2, signs=(1, -1), name="cfg1 rank-2 indefinite e_j a^T + a e_j^T n=4096"),
    2: dict(n=8192, k=4, signs=(1, 1, -1, -1), name="cfg2 rank-4 n=8192"),
    3: dict(n=16384, k=8, signs=(1,) * 8, name="cfg3 deflation stress rank-8 n=16384"),
    4: dict(n=32768, k=16, signs=tuple(1 if r % 2 == 0 else -1 for r in range(16)),
            name="cfg4 rank-16 n=32768"),
}
SEED_BASE = 1706_00773


def default_seed(cfg: int) -> int:
    return SEED_BASE + cfg


def _haar_q(rng, n):
    g = rng.standard_normal((n, n))
    q, r = np.linalg.qr(g)
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s[None, :]


def _spectrum(rng, cfg, n):
    if cfg == 0:
        lam = np.sort(rng.uniform(-1.0, 1.0, n))
        assert np.all(np.diff(lam) > 0)
        return lam
    if cfg == 1:
        return np.sort(rng.uniform(-10.0, 10.0, n))
    if cfg == 2:
        return np.sort(rng.standard_normal(n))
    if cfg == 3:
        return _cluster_spectrum(rng, n)
    if cfg == 4:
        return np.sort(rng.uniform(-100.0, 100.0, n))
    raise ValueError(cfg)


def _cluster_spectrum(rng, n):
    """20% of the values in tight clusters c + m*1e-12 (~51 per cluster, 64
    clusters at n=16384, proportionally fewer below), rest U[-1,1]."""
    ncl_vals = int(round(0.2 * n))
    nclusters = max(1, int(round(64 * n / 16384)))
    per = [ncl_vals // nclusters + (1 if c < ncl_vals % nclusters else 0) for c in range(nclusters)]
    centers = rng.uniform(-1.0, 1.0, nclusters)
    vals = [centers[c] + np.arange(per[c]) * 1e-12 for c in range(nclusters)]
    rest = rng.uniform(-1.0, 1.0, n - ncl_vals)
    return np.sort(np.concatenate(vals + [rest]))


def make_instance(cfg: int, n: int | None = None, seed: int | None = None):
    """Returns (Q, lambda, K, signs) as float64/int32 numpy arrays."""
    c = CONFIGS[cfg]
    n = c["n"] if n is None else int(n)
    k = c["k"]
    signs = np.array(c["signs"], dtype=np.int32)
    rng = np.random.default_rng(default_seed(cfg) if seed is None else seed)
    q = _haar_q(rng, n)
    lam = _spectrum(rng, cfg, n)
    if cfg == 1:
        j = int(rng.integers(0, n))
        a = rng.normal(0.0, 1.0 / math.sqrt(n), n)
        e = np.zeros(n)
        e[j] = 1.0
        kmat = np.stack([(e + a) / math.sqrt(2.0), (e - a) / math.sqrt(2.0)], axis=1)
    else:
        kmat = rng.normal(0.0, 1.0 / math.sqrt(n), (n, k))
    if cfg == 3:
        u = q.T @ kmat
        rows = rng.choice(n, size=int(round(0.05 * n)), replace=False)
        u[rows] *= 1e-14
        kmat = q @ u
    return q, lam, np.ascontiguousarray(kmat), signs


def make_instance_torch(cfg: int, n: int | None = None, seed: int | None = None,
                        device="cuda"):
    """GPU generator (same distributions, different bits): Q from a cuSOLVER QR
    of a Philox N(0,1) matrix. Used for the n=32768 benchmark instance."""
    import torch

    c = CONFIGS[cfg]
    n = c["n"] if n is None else int(n)
    k = c["k"]
    gen = torch.Generator(device=device)
    gen.manual_seed(default_seed(cfg) if seed is None else seed)
    g = torch.randn((n, n), generator=gen, device=device, dtype=torch.float64)
    q, r = torch.linalg.qr(g)
    del g
    s = torch.sign(torch.diagonal(r))
    s[s == 0] = 1.0
    del r
    q.mul_(s[None, :])
    rng = np.random.default_rng((default_seed(cfg) if seed is None else seed) + 99)
    lam = torch.from_numpy(_spectrum(rng, cfg, n)).to(device)
    signs = torch.tensor(c["signs"], dtype=torch.int32)
    if cfg == 1:
        j = int(rng.integers(0, n))
        a = torch.from_numpy(rng.normal(0.0, 1.0 / math.sqrt(n), n)).to(device)
        e = torch.zeros(n, dtype=torch.float64, device=device)
        e[j] = 1.0
        kmat = torch.stack([(e + a) / math.sqrt(2.0), (e - a) / math.sqrt(2.0)], dim=1)
    else:
        kmat = torch.randn((n, k), generator=gen, device=device, dtype=torch.float64) / math.sqrt(n)
    if cfg == 3:
        u = q.T @ kmat
        rows = torch.from_numpy(rng.choice(n, size=int(round(0.05 * n)), replace=False)).to(device)
        u[rows] *= 1e-14
        kmat = q @ u
    return q.contiguous(), lam.contiguous(), kmat.contiguous(), signs
