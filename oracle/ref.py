"""ctypes binding of the UNMODIFIED reference library (oracle/_ref).

TEST INFRASTRUCTURE ONLY. ``oracle/Makefile`` compiles the reference's own
sources (/root/reference/proj/src) together with ``ref_capi.cpp`` into
``oracle/_ref/libeigmod_ref.so``; this module calls its entry points with
numpy buffers. Errors are re-raised with the reference's semantics:
``ValueError`` for std::invalid_argument, ``RefNumericalError`` (carrying the
stage) for eigmod::NumericalError.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libeigmod_ref.so")
_lib = None


class RefNumericalError(RuntimeError):
    def __init__(self, msg: str):
        super().__init__(msg)
        m = re.match(r"\[(\w+)\]", msg)
        self.stage = m.group(1) if m else ""


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (run `make -C oracle ref`)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_default_tolerance.restype = C.c_double
    return _lib


_D = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
_I = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
_L = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _check(rc: int, buf) -> None:
    if rc == 0:
        return
    msg = buf.value.decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise RefNumericalError(msg)
    raise RuntimeError(msg)


def set_parallel(on: bool) -> None:
    lib().ref_set_parallel(1 if on else 0)


def set_threads(n: int) -> None:
    """omp_set_num_threads for the reference's OpenMP paths."""
    lib().ref_set_threads(int(n))


def worker_count() -> int:
    return lib().ref_worker_count()


def random_instance(n: int, k: int, norm: float, seed: int):
    """core.hpp:17-20 — the reference's own seeded instance (signs all +1)."""
    q = np.empty((n, n)); lam = np.empty(n); km = np.empty((n, k))
    buf = C.create_string_buffer(512)
    _check(lib().ref_random_instance(C.c_int64(n), C.c_int64(k), C.c_double(norm),
                                     C.c_uint64(seed), _D(q), _D(lam), _D(km), buf, 512), buf)
    return q, lam, km


def transform_update(q, lam, kmat, signs):
    q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
    n, k = kmat.shape
    u = np.empty((n, k))
    buf = C.create_string_buffer(512)
    _check(lib().ref_transform_update(_D(q), _D(lam), _D(kmat), _I(signs), C.c_int64(n),
                                      C.c_int64(k), _D(u), buf, 512), buf)
    return u


def secular_weights(lam, u, signs):
    lam, u, signs = _f64(lam), _f64(u), _i32(signs)
    n, k = u.shape
    out = np.empty(n)
    buf = C.create_string_buffer(512)
    _check(lib().ref_secular_weights(_D(lam), _D(u), _I(signs), C.c_int64(n), C.c_int64(k),
                                     _D(out), buf, 512), buf)
    return out


def deflate_problem(lam, u, signs):
    """secular.cpp:278-340 → dict(poles, weights, pole_origin, unchanged, collided)."""
    lam, u, signs = _f64(lam), _f64(u), _i32(signs)
    n, k = u.shape
    poles = np.empty(n); w = np.empty(n)
    po = np.empty(n, np.int64); un = np.empty(n, np.int64); co = np.empty(n, np.int64)
    cnt = np.zeros(3, np.int64)
    buf = C.create_string_buffer(512)
    _check(lib().ref_deflate_problem(_D(lam), _D(u), _I(signs), C.c_int64(n), C.c_int64(k),
                                     _D(poles), _D(w), _L(po), _L(un), _L(co), _L(cnt), buf,
                                     512), buf)
    m, nu, nc = (int(x) for x in cnt)
    return dict(poles=poles[:m].copy(), weights=w[:m].copy(), pole_origin=po[:m].copy(),
                unchanged=un[:nu].copy(), collided=co[:nc].copy())


def default_tolerance(lam, kmat, signs):
    lam, kmat, signs = _f64(lam), _f64(kmat), _i32(signs)
    n, k = kmat.shape
    return lib().ref_default_tolerance(_D(lam), _D(kmat), _I(signs), C.c_int64(n), C.c_int64(k))


def update_eigenvalues_full(q, lam, kmat, signs, tol, sturm=False):
    """rootfind.hpp:51-53 → (values, roots, seconds)."""
    q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
    n, k = kmat.shape
    vals = np.empty(n); roots = np.empty(n); nr = np.zeros(1, np.int64); sec = np.zeros(1)
    buf = C.create_string_buffer(1024)
    _check(lib().ref_update_eigenvalues_full(_D(q), _D(lam), _D(kmat), _I(signs), C.c_int64(n),
                                             C.c_int64(k), C.c_double(tol), C.c_int(1 if sturm else 0),
                                             _D(vals), _D(roots), _L(nr), _D(sec), buf, 1024), buf)
    return vals, roots[: int(nr[0])].copy(), float(sec[0])


def update_pairs(q, lam, kmat, signs, tol, reorthogonalize=False):
    """update_eigenvalues_full + assemble_eigenvectors → (lambda', Q', (t_eig, t_vec))."""
    q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
    n, k = kmat.shape
    lo = np.empty(n); qo = np.empty((n, n)); sec = np.zeros(2)
    buf = C.create_string_buffer(1024)
    _check(lib().ref_update_pairs(_D(q), _D(lam), _D(kmat), _I(signs), C.c_int64(n), C.c_int64(k),
                                  C.c_double(tol), C.c_int(1 if reorthogonalize else 0), _D(lo),
                                  _D(qo), _D(sec), buf, 1024), buf)
    return lo, qo, (float(sec[0]), float(sec[1]))


def timed_pairs(q, lam, kmat, signs, tol, vectors=True):
    """Both stages timed separately, failures recorded:
    dict(t_eig, t_vec, failed_stage ("" / "eigenvalues" / "eigenvectors"),
    error, values, q_out). A failing stage's time is its time to failure."""
    q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
    n, k = kmat.shape
    lo = np.empty(n)
    qo = np.empty((n, n)) if vectors else None
    out3 = np.zeros(3)
    buf = C.create_string_buffer(1024)
    L = lib()
    rc = L.ref_timed_pairs(_D(q), _D(lam), _D(kmat), _I(signs), C.c_int64(n), C.c_int64(k),
                           C.c_double(tol), _D(lo), _D(qo) if vectors else None, _D(out3), buf,
                           1024)
    failed = {0: "", 1: "eigenvalues", 2: "eigenvectors"}[int(out3[2])]
    return dict(t_eig=float(out3[0]), t_vec=float(out3[1]) if vectors else None,
                failed_stage=failed, error=buf.value.decode(errors="replace") if rc else "",
                values=lo if rc == 0 or failed == "eigenvectors" else None,
                q_out=qo if rc == 0 else None)


def update_decomposition(q, lam, kmat, signs, tol, reorthogonalize=False):
    """eigvec.hpp:35-36 → (lambda', Q', residual_fro, ortho_err, wall_time)."""
    q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
    n, k = kmat.shape
    lo = np.empty(n); qo = np.empty((n, n)); met = np.zeros(3)
    buf = C.create_string_buffer(1024)
    _check(lib().ref_update_decomposition(_D(q), _D(lam), _D(kmat), _I(signs), C.c_int64(n),
                                          C.c_int64(k), C.c_double(tol),
                                          C.c_int(1 if reorthogonalize else 0), _D(lo), _D(qo),
                                          _D(met), buf, 1024), buf)
    return lo, qo, float(met[0]), float(met[1]), float(met[2])


def jacobi_eigenvalues(a):
    a = _f64(a)
    n = a.shape[0]
    out = np.empty(n)
    buf = C.create_string_buffer(512)
    _check(lib().ref_jacobi_eigenvalues(_D(a), C.c_int64(n), _D(out), buf, 512), buf)
    return out


def eval_secular(poles, weights, x, leading=1.0):
    poles, weights = _f64(poles), _f64(weights)
    f = np.zeros(1)
    buf = C.create_string_buffer(512)
    _check(lib().ref_eval_secular(_D(poles), _D(weights), C.c_int64(len(poles)),
                                  C.c_double(leading), C.c_double(x), _D(f), buf, 512), buf)
    return float(f[0])


# ---- per-eigenpair sampling of the reference at full size ----------------
class _Handle:
    def __init__(self, ptr, free):
        self.ptr, self._free = ptr, free

    def __del__(self):
        try:
            self._free(self.ptr)
        except Exception:
            pass


def matrix(a):
    """Persistent eigmod::Matrix copy of a (for repeated ref_gemm_nn calls)."""
    a = _f64(a)
    L = lib()
    L.ref_matrix_new.restype = C.c_void_p
    L.ref_matrix_free.argtypes = [C.c_void_p]
    p = L.ref_matrix_new(_D(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]))
    return _Handle(p, L.ref_matrix_free)


def matrix_const(rows, cols, value):
    """Persistent rows x cols eigmod::Matrix filled with value."""
    L = lib()
    L.ref_matrix_const.restype = C.c_void_p
    L.ref_matrix_const.argtypes = [C.c_int64, C.c_int64, C.c_double]
    L.ref_matrix_free.argtypes = [C.c_void_p]
    return _Handle(L.ref_matrix_const(rows, cols, value), L.ref_matrix_free)


def gemm_nn(h, b):
    """kernels::gemm_nn (the reference's Q X, kernels.cpp:32-48) on a handle."""
    b = _f64(b)
    rows = None
    L = lib()
    L.ref_gemm_nn.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int64,
                              C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
    out = np.empty((b.shape[0] if rows is None else rows, b.shape[1]))
    buf = C.create_string_buffer(512)
    _check(L.ref_gemm_nn(h.ptr, _D(b), C.c_int64(b.shape[1]), _D(out), buf, 512), buf)
    return out


def gemm_nn_hh(ha, hb, rows, cols):
    """kernels::gemm_nn on two persistent handles (rows x cols result)."""
    L = lib()
    L.ref_gemm_nn_hh.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_double), C.c_char_p,
                                 C.c_size_t]
    out = np.empty((rows, cols))
    buf = C.create_string_buffer(512)
    _check(L.ref_gemm_nn_hh(ha.ptr, hb.ptr, _D(out), buf, 512), buf)
    return out


def transformed(u, signs):
    u, signs = _f64(u), _i32(signs)
    L = lib()
    L.ref_tu_new.restype = C.c_void_p
    L.ref_tu_free.argtypes = [C.c_void_p]
    p = L.ref_tu_new(_D(u), _I(signs), C.c_int64(u.shape[0]), C.c_int64(u.shape[1]))
    return _Handle(p, L.ref_tu_free)


def basis_vector(tu, lam, root):
    """eigvec.cpp:133-153: null_problem + null_direction + resolvent."""
    lam = _f64(lam)
    n = lam.shape[0]
    L = lib()
    L.ref_basis_vector.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.c_double,
                                   C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_char_p,
                                   C.c_size_t]
    w = np.empty(n)
    res = np.zeros(1)
    buf = C.create_string_buffer(512)
    _check(L.ref_basis_vector(tu.ptr, _D(lam), C.c_int64(n), C.c_double(root), _D(w), _D(res),
                              buf, 512), buf)
    return w, float(res[0])


def dnc_solve(poles, weights, lo, hi, expected, tol):
    """rootfind.cpp:89-229 on the bracket (lo, hi) holding `expected` roots."""
    poles, weights = _f64(poles), _f64(weights)
    L = lib()
    out = np.empty(max(1, int(expected)))
    nr = np.zeros(1, np.int64)
    buf = C.create_string_buffer(1024)
    _check(L.ref_dnc_solve(_D(poles), _D(weights), C.c_int64(len(poles)), C.c_double(lo),
                           C.c_double(hi), C.c_int64(expected), C.c_double(tol), _D(out), _L(nr),
                           buf, 1024), buf)
    return out[: int(nr[0])].copy()


def locate_from_u(lam, u, signs):
    """tools/eigmod.cpp:143-161 (cmd_locate) after transform_update: the
    reference's deflate_problem + locate_rank2 / locate_rank_k counts."""
    lam, u, signs = _f64(lam), _f64(u), _i32(signs)
    n, k = u.shape
    out = np.zeros(n + 1, np.int64)
    cnt = np.zeros(1, np.int64)
    buf = C.create_string_buffer(512)
    _check(lib().ref_locate_from_u(_D(lam), _D(u), _I(signs), C.c_int64(n), C.c_int64(k),
                                   _L(out), _L(cnt), buf, C.c_size_t(512)), buf)
    return [int(v) for v in out[: int(cnt[0])]]


def reconstruct(q, lam):
    """core.hpp:11 — Q diag(lambda) Q^T, symmetrized (kernels.cpp:98-109)."""
    q, lam = _f64(q), _f64(lam)
    n = lam.shape[0]
    out = np.empty((n, n))
    buf = C.create_string_buffer(512)
    _check(lib().ref_reconstruct(_D(q), _D(lam), C.c_int64(n), _D(out), buf, C.c_size_t(512)), buf)
    return out


def apply_update(a, kmat, signs):
    """core.hpp:14 — a + sum_r s_r k_r k_r^T, symmetrized (core.cpp:105-115)."""
    a, kmat, signs = _f64(a), _f64(kmat), _i32(signs)
    n, k = kmat.shape
    out = np.empty((n, n))
    buf = C.create_string_buffer(512)
    _check(lib().ref_apply_update(_D(a), _D(kmat), _I(signs), C.c_int64(n), C.c_int64(k),
                                  _D(out), buf, C.c_size_t(512)), buf)
    return out


def ortho_error(a):
    """kernels.hpp:36 — max |A^T A - I| (kernels.cpp:150-154)."""
    a = _f64(a)
    f = lib().ref_ortho_error
    f.restype = C.c_double
    return float(f(_D(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1])))


class RefFormatError(RuntimeError):
    pass


def _io_check(rc, buf):
    if rc == 0:
        return
    msg = buf.value.decode(errors="replace")
    if rc == 3:
        raise RefFormatError(msg)
    raise RuntimeError(msg)


def write_csv(path, m, signs=None):
    """io.cpp:176-194 write_csv_matrix."""
    m = _f64(m)
    if m.ndim == 1:
        m = m[:, None]
    s = None if signs is None else _i32(signs)
    buf = C.create_string_buffer(1024)
    _io_check(lib().ref_write_csv(str(path).encode(), _D(m), C.c_int64(m.shape[0]),
                                  C.c_int64(m.shape[1]), _I(s) if s is not None else None,
                                  C.c_int64(0 if s is None else s.shape[0]), buf,
                                  C.c_size_t(1024)), buf)


def read_csv(path):
    """io.cpp:145-174 read_csv_matrix -> (values, signs or None)."""
    shape = np.zeros(3, np.int64)
    buf = C.create_string_buffer(1024)
    _io_check(lib().ref_read_csv(str(path).encode(), _L(shape), None, None, buf,
                                 C.c_size_t(1024)), buf)
    vals = np.empty((int(shape[0]), int(shape[1])))
    signs = np.empty(max(0, int(shape[2])), np.int32)
    _io_check(lib().ref_read_csv(str(path).encode(), _L(shape), _D(vals), _I(signs), buf,
                                 C.c_size_t(1024)), buf)
    return vals, (signs if shape[2] >= 0 else None)


def write_matrix_market(path, a):
    """io.cpp:119-131."""
    a = _f64(a)
    buf = C.create_string_buffer(1024)
    _io_check(lib().ref_write_mm(str(path).encode(), _D(a), C.c_int64(a.shape[0]), buf,
                                 C.c_size_t(1024)), buf)


def read_matrix_market(path):
    """io.cpp:59-117."""
    n = np.zeros(1, np.int64)
    buf = C.create_string_buffer(1024)
    _io_check(lib().ref_read_mm(str(path).encode(), _L(n), None, buf, C.c_size_t(1024)), buf)
    a = np.empty((int(n[0]), int(n[0])))
    _io_check(lib().ref_read_mm(str(path).encode(), _L(n), _D(a), buf, C.c_size_t(1024)), buf)
    return a


def locate_coeffs(poles, weights, signs):
    """locate_rank2 (two signs) / locate_rank_k on given coefficients."""
    poles, weights, signs = _f64(poles), _f64(weights), _i32(signs)
    out = np.zeros(len(poles) + 1, np.int64)
    buf = C.create_string_buffer(1024)
    _check(lib().ref_locate_coeffs(_D(poles), _D(weights), C.c_int64(len(poles)), _I(signs),
                                   C.c_int64(len(signs)), _L(out), buf, 1024), buf)
    return [int(x) for x in out]


def crossing_count(poles, weights, lo, hi, samples):
    poles, weights = _f64(poles), _f64(weights)
    out = np.zeros(1, np.int64)
    buf = C.create_string_buffer(512)
    _check(lib().ref_crossing_count(_D(poles), _D(weights), C.c_int64(len(poles)), C.c_double(lo),
                                    C.c_double(hi), C.c_int(samples), _L(out), buf, 512), buf)
    return int(out[0])


def solve_rank1(poles, zeta, sigma, tol):
    poles, zeta = _f64(poles), _f64(zeta)
    out = np.empty(len(poles))
    buf = C.create_string_buffer(512)
    _check(lib().ref_solve_rank1(_D(poles), _D(zeta), C.c_int64(len(poles)), C.c_double(sigma),
                                 C.c_double(tol), _D(out), buf, 512), buf)
    return out


def null_problem(u, signs, lam, lam_new):
    u, signs, lam = _f64(u), _i32(signs), _f64(lam)
    n, k = u.shape
    m = np.empty((k, k))
    buf = C.create_string_buffer(512)
    _check(lib().ref_null_problem(_D(u), _I(signs), _D(lam), C.c_int64(n), C.c_int64(k),
                                  C.c_double(lam_new), _D(m), buf, 512), buf)
    return m


def null_direction(m):
    m = _f64(m)
    k = m.shape[0]
    d, r = np.empty(k), np.zeros(1)
    buf = C.create_string_buffer(512)
    _check(lib().ref_null_direction(_D(m), C.c_int64(k), _D(d), _D(r), buf, 512), buf)
    return d, float(r[0])


def update_eigenvector(q, lam, kmat, signs, lam_new):
    q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
    n, k = kmat.shape
    v = np.empty(n)
    buf = C.create_string_buffer(512)
    _check(lib().ref_update_eigenvector(_D(q), _D(lam), _D(kmat), _I(signs), C.c_int64(n),
                                        C.c_int64(k), C.c_double(lam_new), _D(v), buf, 512), buf)
    return v
