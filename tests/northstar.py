"""North-star acceptance measures (BASELINE.json north_star), shared by the
tests and smoke():

  eigenvalues    |lambda' - lambda'_ref| <= 1e-10 ||A'||_2 per eigenvalue
  residual       max_j ||A' x_j - lambda'_j x_j||_2 / ||A'||_2 <= 1e-10
                 (per-column 2-norm, not the max-abs entry)
  orthogonality  ||Q'^T Q' - I||_max <= 1e-9
"""
from __future__ import annotations

import numpy as np

EIG_TOL = 1e-10
RESID_TOL = 1e-10
ORTHO_TOL = 1e-9


def aprime(q, lam, kmat, signs):
    """A' = Q diag(lambda) Q^T + K J K^T, symmetrized."""
    q = np.asarray(q, float)
    a = (q * np.asarray(lam, float)[None, :]) @ q.T
    a += (np.asarray(kmat, float) * np.asarray(signs, float)[None, :]) @ np.asarray(kmat, float).T
    return 0.5 * (a + a.T)


def norm2(ev) -> float:
    """||A'||_2 from its eigenvalues (floored at the smallest normal)."""
    return max(float(np.abs(np.asarray(ev)).max()), np.finfo(float).tiny)


def residual(a, q, lam, nrm) -> float:
    """max_j ||A' q_j - lambda_j q_j||_2 / ||A'||_2."""
    r = a @ q - q * np.asarray(lam)[None, :]
    return float(np.sqrt((r * r).sum(axis=0)).max()) / nrm


def ortho(q) -> float:
    return float(np.abs(q.T @ q - np.eye(q.shape[1])).max())
