"""ctypes binding of the C restatement (oracle/eigmod_oracle.c).

TEST INFRASTRUCTURE ONLY — the checker for the CUDA path and the "port"
CPU baseline. Built by ``make -C oracle oracle`` (also done by
``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libeigmod_oracle.so")
_lib = None

PARITY_RUN_REL = 1e-12   # secular.hpp:66 kPoleMergeRelGap
EXACT_RUN_REL = 1e-10    # exact mode


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE, "oracle"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.eo_drop_zero_columns.restype = C.c_int64
        _lib.eo_count_below.restype = C.c_int64
    return _lib


_D = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
_I = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
_L = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def transform(q, kmat):
    q, kmat = _f64(q), _f64(kmat)
    n, k = kmat.shape
    u = np.empty((n, k))
    lib().eo_transform(_D(q), _D(kmat), C.c_int64(n), C.c_int64(k), _D(u))
    return u


def drop_zero_columns(u):
    u = _f64(u)
    n, k = u.shape
    keep = np.empty(k, np.int64)
    m = lib().eo_drop_zero_columns(_D(u), C.c_int64(n), C.c_int64(k), _L(keep))
    return keep[:m].copy()


def secular_weights(lam, u, signs):
    lam, u, signs = _f64(lam), _f64(u), _i32(signs)
    n, k = u.shape
    out = np.empty(n)
    if lib().eo_secular_weights(_D(lam), _D(u), _I(signs), C.c_int64(n), C.c_int64(k), _D(out)):
        raise ValueError("secular_weights: bad input")
    return out


def deflate(lam, u, signs, merge_rel=PARITY_RUN_REL):
    lam, u, signs = _f64(lam), _f64(u), _i32(signs)
    n, k = u.shape
    poles = np.empty(n); w = np.empty(n)
    po = np.empty(n, np.int64); un = np.empty(n, np.int64); co = np.empty(n, np.int64)
    cnt = np.zeros(3, np.int64)
    if lib().eo_deflate(_D(lam), _D(u), _I(signs), C.c_int64(n), C.c_int64(k),
                        C.c_double(merge_rel), _D(poles), _D(w), _L(po), _L(un), _L(co),
                        _L(cnt)):
        raise ValueError("deflate: bad input")
    m, nu, nc = (int(x) for x in cnt)
    return dict(poles=poles[:m].copy(), weights=w[:m].copy(), pole_origin=po[:m].copy(),
                unchanged=un[:nu].copy(), collided=co[:nc].copy())


def update(q, lam, kmat, signs, run_rel=EXACT_RUN_REL, vectors=True):
    """Full update → (lambda', Q' or None, info dict)."""
    q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
    n, k = kmat.shape
    lo = np.empty(n)
    qo = np.empty((n, n)) if vectors else None
    info = np.zeros(4, np.int64)
    rc = lib().eo_update(_D(q), _D(lam), _D(kmat), _I(signs), C.c_int64(n), C.c_int64(k),
                         C.c_double(run_rel), _D(lo), _D(qo) if vectors else None, _L(info))
    if rc == 1:
        raise ValueError("eo_update: invalid argument")
    if rc == 2:
        raise RuntimeError("eo_update: eigenvalue accounting failed")
    return lo, qo, dict(roots=int(info[0]), decoupled=int(info[1]), collided=int(info[2]),
                        evals=int(info[3]))


def solve_roots(d, ut, signs, j0=0, j1=None):
    d, ut, signs = _f64(d), _f64(ut), _i32(signs)
    n, k = ut.shape
    j1 = n if j1 is None else j1
    m = j1 - j0
    roots = np.empty(m); orig = np.empty(m, np.int64); dl = np.empty(m); ev = np.zeros(1, np.int64)
    if lib().eo_solve_roots(_D(d), _D(ut), _I(signs), C.c_int64(n), C.c_int64(k), C.c_int64(j0),
                            C.c_int64(j1), _D(roots), _L(orig), _D(dl), _L(ev)):
        raise ValueError("solve_roots: bad input")
    return roots, orig, dl, int(ev[0])


def count_below(d, ut, signs, x):
    d, ut, signs = _f64(d), _f64(ut), _i32(signs)
    n, k = ut.shape
    return int(lib().eo_count_below(_D(d), _D(ut), _I(signs), C.c_int64(n), C.c_int64(k),
                                    C.c_double(x)))


def gemm_nt(a, b):
    a, b = _f64(a), _f64(b)
    m, l = a.shape
    nn = b.shape[0]
    c = np.empty((m, nn))
    lib().eo_gemm_nt(_D(a), _D(b), C.c_int64(m), C.c_int64(nn), C.c_int64(l), _D(c))
    return c


class LocateUnsupported(Exception):
    """eo_locate does not restate merged multi-row runs (k >= 2)."""


def locate_from_u(lam, u, signs):
    """Location vector over the reference deflation record's poles (oracle)."""
    lam, u, signs = _f64(lam), _f64(u), _i32(signs)
    n, k = u.shape
    out = np.zeros(n + 1, np.int64)
    cnt = np.zeros(1, np.int64)
    rc = lib().eo_locate(_D(lam), _D(u), _I(signs), C.c_int64(n), C.c_int64(k), _L(out),
                         _L(cnt))
    if rc == 1:
        raise ValueError("eo_locate: invalid argument")
    if rc == 3:
        raise LocateUnsupported("merged multi-row run")
    return [int(v) for v in out[: int(cnt[0])]]
