"""Matrix Market / CSV ingest and egest (include/eigmod_b200_io.h, host C++
in lib/libeigmod_b200_cxx.so): the reference's io.hpp:17-33 for Python
callers. FormatError mirrors eigmod::FormatError."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libeigmod_b200_cxx.so")
_lib = None


class FormatError(RuntimeError):
    """eigmod::FormatError (proj/include/eigmod/io.hpp:10-14)."""


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise FileNotFoundError(f"{_LIB} missing: run __graft_entry__.build()")
        _lib = C.CDLL(_LIB)
        _lib.eigmod_b200_io_last_error.restype = C.c_char_p
    return _lib


_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_L = C.POINTER(C.c_int64)


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = (lib().eigmod_b200_io_last_error() or b"").decode()
    if rc == 3:
        raise FormatError(msg)
    raise RuntimeError(msg)


def write_csv(path, m, signs=None) -> None:
    m = np.ascontiguousarray(m, dtype=np.float64)
    if m.ndim == 1:
        m = m[:, None]
    s = None if signs is None else np.ascontiguousarray(signs, dtype=np.int32)
    _check(lib().eigmod_b200_io_write_csv(str(path).encode(), m.ctypes.data_as(_D),
                                          C.c_int64(m.shape[0]), C.c_int64(m.shape[1]),
                                          s.ctypes.data_as(_I) if s is not None else None,
                                          C.c_int64(0 if s is None else s.shape[0])))


def read_csv(path):
    """-> (values (rows x cols), signs or None)."""
    shape = np.zeros(3, np.int64)
    _check(lib().eigmod_b200_io_read_csv(str(path).encode(), shape.ctypes.data_as(_L)))
    vals = np.empty((int(shape[0]), int(shape[1])))
    signs = np.empty(max(0, int(shape[2])), np.int32)
    _check(lib().eigmod_b200_io_take_csv(vals.ctypes.data_as(_D), signs.ctypes.data_as(_I)))
    return vals, (signs if shape[2] >= 0 else None)


def write_matrix_market(path, a) -> None:
    a = np.ascontiguousarray(a, dtype=np.float64)
    _check(lib().eigmod_b200_io_write_matrix_market(str(path).encode(), a.ctypes.data_as(_D),
                                                    C.c_int64(a.shape[0])))


def read_matrix_market(path) -> np.ndarray:
    n = np.zeros(1, np.int64)
    _check(lib().eigmod_b200_io_read_matrix_market(str(path).encode(), n.ctypes.data_as(_L)))
    a = np.empty((int(n[0]), int(n[0])))
    _check(lib().eigmod_b200_io_take_matrix_market(a.ctypes.data_as(_D)))
    return a
