"""ctypes binding of the C ABI in include/eigmod_b200.h (lib/libeigmod_b200.so).

This is the Python host side of the drop-in boundary. It mirrors the
reference's entry points (proj/include/eigmod/*.hpp) with the same names,
argument meaning and error behaviour:

  transform_update         secular.hpp:28        U = Q^T K
  secular_weights          secular.hpp:34        per-pole weights alpha
  deflate_problem          secular.hpp:69        deflation record
  update_eigenvalues_full  rootfind.hpp:51-53    eigenvalue stage (rank-2 and rank-k)
  update_eigenvalues       rootfind.hpp:58
  update_decomposition     eigvec.hpp:35-36      eigenvalues + eigenvectors

std::invalid_argument -> ValueError; eigmod::NumericalError -> NumericalError
(with .stage); device failures -> DeviceError. There is no CPU fallback: if
the shared library or a B200 is missing, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EIGMOD_B200_LIB") or os.path.join(_PKG, "lib", "libeigmod_b200.so")

_lib = None
_lock = threading.Lock()


class NumericalError(RuntimeError):
    """eigmod::NumericalError (proj/include/eigmod/types.hpp:79-87)."""

    def __init__(self, stage: str, msg: str):
        super().__init__(msg)
        self.stage = stage


class DeviceError(RuntimeError):
    """CUDA / device failure (no CPU fallback exists)."""


_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int)
_I64 = C.POINTER(C.c_int64)
_VP = C.c_void_p


def _declare(lib):
    sig = {
        "eigmod_b200_ctx_create": (C.c_int, [C.c_int, C.POINTER(_VP)]),
        "eigmod_b200_ctx_destroy": (None, [_VP]),
        "eigmod_b200_ctx_set_stream": (C.c_int, [_VP, _VP]),
        "eigmod_b200_ctx_use_own_stream": (C.c_int, [_VP]),
        "eigmod_b200_set_option": (C.c_int, [_VP, C.c_char_p, C.c_double]),
        "eigmod_b200_last_error": (C.c_char_p, [_VP]),
        "eigmod_b200_last_stage": (C.c_char_p, [_VP]),
        "eigmod_b200_stats": (C.c_int, [_VP, _D]),
        "eigmod_b200_workspace_bytes": (C.c_int64, [_VP]),
        "eigmod_b200_solver_profile": (C.c_int, [_VP, _D]),
        "eigmod_b200_solver_trace": (C.c_int, [_VP, _D]),
        "eigmod_b200_presolve_profile": (C.c_int, [_VP, _D]),
        "eigmod_b200_stage_times": (C.c_int, [_VP, _D, C.c_int]),
        "eigmod_b200_launch_count": (C.c_int64, []),
        "eigmod_b200_fp64_peaks": (C.c_int, [_VP, _D]),
        "eigmod_b200_transform_update": (C.c_int, [_VP, _D, _D, C.c_int64, C.c_int64, _D]),
        "eigmod_b200_secular_weights": (C.c_int, [_VP, _D, _D, _I32, C.c_int64, C.c_int64, _D]),
        "eigmod_b200_deflate_problem": (C.c_int, [_VP, _D, _D, _I32, C.c_int64, C.c_int64, _D, _D,
                                                  _I64, _I64, _I64, _I64]),
        "eigmod_b200_locate": (C.c_int, [_VP, _D, _D, _D, _I32, C.c_int64, C.c_int64, _I64,
                                         _I64]),
        "eigmod_b200_locate_from_u": (C.c_int, [_VP, _D, _D, _I32, C.c_int64, C.c_int64, _I64,
                                                _I64]),
        "eigmod_b200_reconstruct": (C.c_int, [_VP, _D, _D, C.c_int64, _D]),
        "eigmod_b200_reconstruct_device": (C.c_int, [_VP, _VP, _VP, C.c_int64, _VP]),
        "eigmod_b200_apply_update": (C.c_int, [_VP, _D, _D, _I32, C.c_int64, C.c_int64, _D]),
        "eigmod_b200_apply_update_device": (C.c_int, [_VP, _VP, _VP, _I32, C.c_int64, C.c_int64,
                                                      _VP]),
        "eigmod_b200_ortho_error": (C.c_int, [_VP, _D, C.c_int64, C.c_int64, _D]),
        "eigmod_b200_ortho_error_device": (C.c_int, [_VP, _VP, C.c_int64, C.c_int64, _D]),
        "eigmod_b200_update_eigenvalues": (C.c_int, [_VP, _D, _D, _D, _I32, C.c_int64, C.c_int64,
                                                     C.c_double, _D, _D, _I64, _D, _I64, _I64]),
        "eigmod_b200_update_decomposition": (C.c_int, [_VP, _D, _D, _D, _I32, C.c_int64,
                                                       C.c_int64, C.c_double, _D, _D, _D]),
        "eigmod_b200_assemble_from_u": (C.c_int, [_VP, _D, _D, _D, _I32, C.c_int64, C.c_int64, _D,
                                                  _D]),
        "eigmod_b200_update_metrics": (C.c_int, [_VP, _D, _D, _D, _I32, C.c_int64, C.c_int64, _D,
                                                 _D, _D, _D]),
        "eigmod_b200_gemm_nt": (C.c_int, [_VP, _D, _D, C.c_int64, C.c_int64, C.c_int64, _D]),
        "eigmod_b200_update_decomposition_device": (C.c_int, [_VP, _VP, _VP, _VP, _I32, C.c_int64,
                                                              C.c_int64, _VP, _VP]),
        "eigmod_b200_padded_rank": (C.c_int, [C.c_int64]),
        "eigmod_b200_record_width": (C.c_int, [C.c_int]),
        "eigmod_b200_project_device": (C.c_int, [_VP, _VP, _VP, C.c_int64, C.c_int64, C.c_int64,
                                                 C.c_int64, _VP]),
        "eigmod_b200_plan_device": (C.c_int, [_VP, _VP, _VP, _I32, C.c_int64, C.c_int64, _I64]),
        "eigmod_b200_plan_groups_device": (C.c_int, [_VP, _VP, _VP, _I32, C.c_int64, C.c_int64,
                                                     _I64]),
        "eigmod_b200_plan_weights_device": (C.c_int, [_VP, C.c_int64, C.c_int64, _VP]),
        "eigmod_b200_plan_finish_device": (C.c_int, [_VP, _VP, _I64]),
        "eigmod_b200_solve_device": (C.c_int, [_VP, C.c_int64, C.c_int64, _VP]),
        "eigmod_b200_finish_device": (C.c_int, [_VP, _VP, _VP, C.c_int64, C.c_int64, _VP, _VP,
                                                C.c_int64]),
        "eigmod_b200_gemm_nt_device": (C.c_int, [_VP, _VP, _VP, C.c_int64, C.c_int64, C.c_int64,
                                                 _VP, C.c_int64]),
        "eigmod_b200_assemble": (C.c_int, [_VP, _D, _D, _D, _I32, C.c_int64, C.c_int64, _D,
                                           C.c_int64, _I64, C.c_int64, _I64, C.c_int64, _D, _D,
                                           _I32]),
        "eigmod_b200_stage_calls": (C.c_int, [_VP, _I64]),
        "eigmod_b200_null_problem": (C.c_int, [_VP, _D, _I32, _D, C.c_int64, C.c_int64,
                                               C.c_double, _D]),
        "eigmod_b200_null_direction": (C.c_int, [_D, C.c_int64, _D, _D]),
        "eigmod_b200_update_eigenvector": (C.c_int, [_VP, _D, _D, _D, _I32, C.c_int64, C.c_int64,
                                                     C.c_double, _D]),
        "eigmod_b200_secular_eval": (C.c_int, [_VP, _D, _D, C.c_int64, C.c_double, _D, C.c_int64,
                                               _D, _D, _I32]),
        "eigmod_b200_crossing_count": (C.c_int, [_VP, _D, _D, C.c_int64, C.c_double, C.c_double,
                                                 C.c_double, C.c_int, _I64]),
        "eigmod_b200_dnc_solve": (C.c_int, [_VP, _D, _D, C.c_int64, C.c_double, C.c_double,
                                            C.c_double, C.c_int64, C.c_double, _D, _I64, _I64,
                                            _I64]),
        "eigmod_b200_solve_rank1": (C.c_int, [_VP, _D, _D, C.c_int64, C.c_double, C.c_double,
                                              _D]),
        "eigmod_b200_locate_coeffs": (C.c_int, [_VP, _D, _D, C.c_int64, C.c_double, _I64]),
        "eigmod_b200_gemm": (C.c_int, [_VP, C.c_int, C.c_int, _D, _D, C.c_int64, C.c_int64,
                                       C.c_int64, _D]),
        "eigmod_b200_multi_create": (C.c_int, [_I32, C.c_int, C.POINTER(_VP)]),
        "eigmod_b200_multi_destroy": (None, [_VP]),
        "eigmod_b200_multi_size": (C.c_int, [_VP]),
        "eigmod_b200_multi_last_error": (C.c_char_p, [_VP]),
        "eigmod_b200_multi_last_stage": (C.c_char_p, [_VP]),
        "eigmod_b200_multi_set_option": (C.c_int, [_VP, C.c_char_p, C.c_double]),
        "eigmod_b200_multi_update_decomposition": (C.c_int, [_VP, _D, _D, _D, _I32, C.c_int64,
                                                             C.c_int64, C.c_double, _D, _D, _D]),
        "eigmod_b200_multi_update_eigenvalues": (C.c_int, [_VP, _D, _D, _D, _I32, C.c_int64,
                                                           C.c_int64, C.c_double, _D]),
        "eigmod_b200_split": (C.c_int, [C.c_int64, C.c_int, C.c_int, _I64, _I64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return sig


EXPORTED = None


def lib():
    """Loads lib/libeigmod_b200.so; raises if it was not built."""
    global _lib, EXPORTED
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                                  "(python -m paper_1706_00773_b200.build)")
            _lib = C.CDLL(LIB_PATH)
            EXPORTED = sorted(_declare(_lib))
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _dp(a):
    return a.ctypes.data_as(_D)


class Context:
    """One device context (stream + workspaces); not thread-safe."""

    def __init__(self, device: int = 0):
        self._l = lib()
        h = _VP()
        rc = self._l.eigmod_b200_ctx_create(int(device), C.byref(h))
        if rc != 0:
            raise DeviceError(f"eigmod_b200_ctx_create(device={device}) failed (rc={rc}): "
                              "no usable sm_100 GPU")
        self.h = h
        self.device = device
        # diagnostics: solver options for every new context, "key=value,..."
        for kv in os.environ.get("EIGMOD_B200_OPTS", "").split(","):
            if kv.strip():
                key, val = kv.split("=")
                self.set_option(key.strip(), float(val))

    def close(self):
        if getattr(self, "h", None):
            self._l.eigmod_b200_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int):
        if rc == 0:
            return
        msg = (self._l.eigmod_b200_last_error(self.h) or b"").decode()
        stage = (self._l.eigmod_b200_last_stage(self.h) or b"").decode()
        if rc == 1:
            raise ValueError(msg)
        if rc == 2:
            raise NumericalError(stage, msg)
        raise DeviceError(msg)

    def set_stream(self, stream_ptr: int | None):
        """Run on this cudaStream_t handle (0 = legacy default stream);
        None returns to the context's own stream."""
        if stream_ptr is None:
            self.check(self._l.eigmod_b200_ctx_use_own_stream(self.h))
        else:
            self.check(self._l.eigmod_b200_ctx_set_stream(self.h, _VP(int(stream_ptr))))

    def set_option(self, key: str, value: float):
        self.check(self._l.eigmod_b200_set_option(self.h, key.encode(), C.c_double(value)))

    def stats(self) -> dict:
        s = np.zeros(8)
        self.check(self._l.eigmod_b200_stats(self.h, _dp(s)))
        keys = ["roots", "decoupled", "collided", "evals", "max_evals", "kp", "k_eff", "groups"]
        return {k: float(v) for k, v in zip(keys, s)}

    def stage_times(self, reset: bool = False) -> dict:
        """Cumulative per-stage device ms (option "timing" must be on)."""
        s = np.zeros(8)
        self.check(self._l.eigmod_b200_stage_times(self.h, _dp(s), 1 if reset else 0))
        keys = ["k1_project", "k2_plan", "k3_solve", "k4_columns", "k5_gemm", "sign_rule"]
        out = {k: float(v) for k, v in zip(keys, s)}
        out["calls"] = int(s[7])
        return out

    def fp64_peaks(self) -> dict:
        """Live FP64 ceilings (TFLOP/s) of this device: DMMA and DFMA loops."""
        out = np.zeros(2)
        self.check(self._l.eigmod_b200_fp64_peaks(self.h, _dp(out)))
        return {"dmma_tflops": float(out[0]), "dfma_tflops": float(out[1])}

    def solver_profile(self) -> dict:
        o = np.zeros(10)
        self.check(self._l.eigmod_b200_solver_profile(self.h, o.ctypes.data_as(_D)))
        cyc = max(1.0, o[3] + o[4] + o[5] + o[6])
        return {"passes": o[0], "active_slot_passes": o[1], "batches": o[2],
                "slot_util": o[1] / max(1.0, 32.0 * o[0]),
                "cycles": {"refill": o[3], "pass": o[4], "reduce": o[5], "step": o[6]},
                "share": {"refill": o[3] / cyc, "pass": o[4] / cyc, "reduce": o[5] / cyc,
                          "step": o[6] / cyc, "step_load": o[7] / cyc, "step_factor": o[8] / cyc,
                          "step_solve": o[9] / cyc}}

    def presolve_profile(self) -> dict:
        o = np.zeros(4)
        self.check(self._l.eigmod_b200_presolve_profile(self.h, o.ctypes.data_as(_D)))
        return {"converged": o[0], "unconverged": o[1], "evals": o[2], "max_evals": o[3]}

    def solver_trace(self) -> np.ndarray:
        o = np.zeros((200, 12))
        self.check(self._l.eigmod_b200_solver_trace(self.h, o.ctypes.data_as(_D)))
        return o[o[:, 0] > 0]

    def workspace_bytes(self) -> int:
        return int(self._l.eigmod_b200_workspace_bytes(self.h))


_default: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    ctx = _default.get(device)
    if ctx is None:
        ctx = _default[device] = Context(device)
    return ctx


# --------------------------------------------------------------- host API
@dataclass
class DeflatedProblem:
    """secular.hpp:59-64."""

    poles: np.ndarray
    weights: np.ndarray
    pole_origin: np.ndarray
    unchanged: np.ndarray
    collided: np.ndarray
    leading: float = 1.0


@dataclass
class EigenvalueUpdate:
    """rootfind.hpp:40-45."""

    values: np.ndarray
    roots: np.ndarray
    problem: DeflatedProblem | None
    u: np.ndarray                      # transformed U (zero columns dropped)
    signs: np.ndarray
    keep: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))


@dataclass
class UpdateResult:
    """types.hpp:71-76 (residual_fro / ortho_err filled on request)."""

    lam: np.ndarray
    q: np.ndarray
    residual_fro: float = float("nan")
    ortho_err: float = float("nan")
    wall_time: float = 0.0


def transform_update(q, kmat, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    q, kmat = _f64(q), _f64(kmat)
    if kmat.ndim != 2 or q.shape != (kmat.shape[0], kmat.shape[0]):
        raise ValueError("transform_update: dimension mismatch")
    n, k = kmat.shape
    u = np.empty((n, k))
    ctx.check(ctx._l.eigmod_b200_transform_update(ctx.h, _dp(q), _dp(kmat), n, k, _dp(u)))
    return u


def secular_weights(lam, u, signs, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    lam, u, signs = _f64(lam), _f64(u), _i32(signs)
    n, k = u.shape
    if k == 0:
        raise ValueError("secular_weights: k = 0")
    if lam.shape[0] != n or signs.shape[0] != k:
        raise ValueError("secular_weights: dimension mismatch")
    out = np.empty(n)
    ctx.check(ctx._l.eigmod_b200_secular_weights(ctx.h, _dp(lam), _dp(u),
                                                  signs.ctypes.data_as(_I32), n, k, _dp(out)))
    return out


def deflate_problem(lam, u, signs, ctx: Context | None = None) -> DeflatedProblem:
    ctx = ctx or default_context()
    lam, u, signs = _f64(lam), _f64(u), _i32(signs)
    n, k = u.shape
    if lam.shape[0] != n:
        raise ValueError("deflate_problem: dimension mismatch")
    poles, w = np.empty(n), np.empty(n)
    po, un, co = (np.empty(n, np.int64) for _ in range(3))
    cnt = np.zeros(3, np.int64)
    ctx.check(ctx._l.eigmod_b200_deflate_problem(
        ctx.h, _dp(lam), _dp(u), signs.ctypes.data_as(_I32), n, k, _dp(poles), _dp(w),
        po.ctypes.data_as(_I64), un.ctypes.data_as(_I64), co.ctypes.data_as(_I64),
        cnt.ctypes.data_as(_I64)))
    m, nu, nc = (int(x) for x in cnt)
    return DeflatedProblem(poles[:m].copy(), w[:m].copy(), po[:m].copy(), un[:nu].copy(),
                           co[:nc].copy())


def locate(q, lam, kmat, signs, ctx: Context | None = None) -> list[int]:
    """Location vector of the CLI locate path (tools/eigmod.cpp:143-161):
    transform -> deflate -> per-interval root counts over the deflated poles
    (locate.hpp:13-50). Returns N + 1 counts ([0] when every pole deflates)."""
    ctx = ctx or default_context()
    q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
    _check_update(q, lam, kmat, signs)
    n, k = kmat.shape
    out = np.zeros(n + 1, np.int64)
    cnt = np.zeros(1, np.int64)
    ctx.check(ctx._l.eigmod_b200_locate(ctx.h, _dp(q), _dp(lam), _dp(kmat),
                                        signs.ctypes.data_as(_I32), n, k,
                                        out.ctypes.data_as(_I64), cnt.ctypes.data_as(_I64)))
    return [int(v) for v in out[: int(cnt[0])]]


def locate_from_u(lam, u, signs, ctx: Context | None = None) -> list[int]:
    """locate() from U = Q^T K."""
    ctx = ctx or default_context()
    lam, u, signs = _f64(lam), _f64(u), _i32(signs)
    if u.ndim != 2 or lam.shape[0] != u.shape[0] or signs.shape[0] != u.shape[1]:
        raise ValueError("locate: dimension mismatch")
    n, k = u.shape
    out = np.zeros(n + 1, np.int64)
    cnt = np.zeros(1, np.int64)
    ctx.check(ctx._l.eigmod_b200_locate_from_u(ctx.h, _dp(lam), _dp(u),
                                               signs.ctypes.data_as(_I32), n, k,
                                               out.ctypes.data_as(_I64),
                                               cnt.ctypes.data_as(_I64)))
    return [int(v) for v in out[: int(cnt[0])]]


def reconstruct(q, lam, ctx: Context | None = None) -> np.ndarray:
    """core.hpp:11 — Q diag(lambda) Q^T, symmetrized (K5 DMMA GEMM)."""
    ctx = ctx or default_context()
    q, lam = _f64(q), _f64(lam)
    n = lam.shape[0]
    if q.shape != (n, n):
        raise ValueError("reconstruct: dimension mismatch")
    out = np.empty((n, n))
    ctx.check(ctx._l.eigmod_b200_reconstruct(ctx.h, _dp(q), _dp(lam), n, _dp(out)))
    return out


def apply_update(a, kmat, signs, ctx: Context | None = None) -> np.ndarray:
    """core.hpp:14 — a + sum_r s_r k_r k_r^T, symmetrized (bit-identical)."""
    ctx = ctx or default_context()
    a, kmat, signs = _f64(a), _f64(kmat), _i32(signs)
    n, k = kmat.shape
    if a.shape != (n, n):
        raise ValueError("apply_update: dimension mismatch")
    if signs.shape[0] != k:
        raise ValueError("apply_update: signs size")
    out = np.empty((n, n))
    ctx.check(ctx._l.eigmod_b200_apply_update(ctx.h, _dp(a), _dp(kmat),
                                              signs.ctypes.data_as(_I32), n, k, _dp(out)))
    return out


def ortho_error(a, ctx: Context | None = None) -> float:
    """kernels.hpp:36 — max |A^T A - I| (K5 DMMA GEMM)."""
    ctx = ctx or default_context()
    a = _f64(a)
    if a.ndim != 2:
        raise ValueError("ortho_error: matrix expected")
    out = np.zeros(1)
    ctx.check(ctx._l.eigmod_b200_ortho_error(ctx.h, _dp(a), a.shape[0], a.shape[1], _dp(out)))
    return float(out[0])


def _check_update(q, lam, kmat, signs):
    if kmat.ndim != 2 or lam.ndim != 1 or q.shape != (lam.shape[0], lam.shape[0]):
        raise ValueError("LowRankUpdate: dimension mismatch")
    if kmat.shape[0] != lam.shape[0]:
        raise ValueError("LowRankUpdate: dimension mismatch")
    if signs.shape[0] != kmat.shape[1]:
        raise ValueError("LowRankUpdate: signs size")


def update_eigenvalues_full(q, lam, kmat, signs, tol, with_problem=True,
                            ctx: Context | None = None) -> EigenvalueUpdate:
    ctx = ctx or default_context()
    q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
    _check_update(q, lam, kmat, signs)
    n, k = kmat.shape
    vals, roots = np.empty(n), np.empty(n)
    nr, keff = np.zeros(1, np.int64), np.zeros(1, np.int64)
    u = np.empty(n * k)
    keep = np.zeros(k, np.int64)
    ctx.check(ctx._l.eigmod_b200_update_eigenvalues(
        ctx.h, _dp(q), _dp(lam), _dp(kmat), signs.ctypes.data_as(_I32), n, k, C.c_double(tol),
        _dp(vals), _dp(roots), nr.ctypes.data_as(_I64), _dp(u), keff.ctypes.data_as(_I64),
        keep.ctypes.data_as(_I64)))
    ke = int(keff[0])
    uk = u[: n * ke].reshape(n, ke).copy()
    sg = signs[keep[:ke]].copy()
    prob = None
    if with_problem and ke > 0:
        prob = deflate_problem(lam, uk, sg, ctx=ctx)
    elif with_problem:
        prob = DeflatedProblem(np.zeros(0), np.zeros(0), np.zeros(0, np.int64),
                               np.arange(n, dtype=np.int64), np.zeros(0, np.int64))
    return EigenvalueUpdate(vals, roots[: int(nr[0])].copy(), prob, uk, sg, keep[:ke].copy())


def update_eigenvalues(q, lam, kmat, signs, tol, ctx: Context | None = None) -> np.ndarray:
    return update_eigenvalues_full(q, lam, kmat, signs, tol, with_problem=False, ctx=ctx).values


def update_decomposition(q, lam, kmat, signs, tol, metrics=False,
                         ctx: Context | None = None) -> UpdateResult:
    ctx = ctx or default_context()
    q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
    _check_update(q, lam, kmat, signs)
    n, k = kmat.shape
    lo = np.empty(n)
    qo = np.empty((n, n))
    wt = np.zeros(1)
    ctx.check(ctx._l.eigmod_b200_update_decomposition(
        ctx.h, _dp(q), _dp(lam), _dp(kmat), signs.ctypes.data_as(_I32), n, k, C.c_double(tol),
        _dp(lo), _dp(qo), _dp(wt)))
    res = UpdateResult(lo, qo, wall_time=float(wt[0]))
    if metrics:  # eigvec.cpp:384-393 (validation only, outside the timed update), on the GPU
        rf, oe = np.zeros(1), np.zeros(1)
        ctx.check(ctx._l.eigmod_b200_update_metrics(
            ctx.h, _dp(q), _dp(lam), _dp(kmat), signs.ctypes.data_as(_I32), n, k, _dp(qo),
            _dp(lo), _dp(rf), _dp(oe)))
        res.residual_fro, res.ortho_err = float(rf[0]), float(oe[0])
    return res


def assemble_eigenvectors(q, lam, plan: EigenvalueUpdate, ctx: Context | None = None,
                          return_path=False):
    """eigvec.hpp:29-31 — Q' and lambda' from a finished eigenvalue stage. The
    plan of the last update_eigenvalues_full on the same context is reused on
    the device (K4 + K5 only); any other plan is checked against the secular
    equation of plan.u first (NumericalError "assemble" if its eigenvalues are
    not those)."""
    ctx = ctx or default_context()
    q, lam = _f64(q), _f64(lam)
    n = lam.shape[0]
    u, sg = _f64(plan.u), _i32(plan.signs)
    k = u.shape[1] if u.ndim == 2 else 0
    if q.shape != (n, n) or (k and u.shape[0] != n):
        raise ValueError("assemble_eigenvectors: plan does not match the decomposition")
    roots = _f64(plan.roots)
    prob = plan.problem
    un = np.ascontiguousarray(prob.unchanged if prob is not None else [], dtype=np.int64)
    co = np.ascontiguousarray(prob.collided if prob is not None else [], dtype=np.int64)
    lo = np.empty(n)
    qo = np.empty((n, n))
    path = np.zeros(1, np.int32)
    ctx.check(ctx._l.eigmod_b200_assemble(
        ctx.h, _dp(q), _dp(lam), _dp(u), sg.ctypes.data_as(_I32), n, k, _dp(roots), len(roots),
        un.ctypes.data_as(_I64), len(un), co.ctypes.data_as(_I64), len(co), _dp(lo), _dp(qo),
        path.ctypes.data_as(_I32)))
    return (lo, qo, int(path[0])) if return_path else (lo, qo)


def stage_calls(ctx: Context | None = None) -> dict:
    """Stage launches on a context: K1 projections, K2 plans, K3 solves, K4+K5 builds."""
    ctx = ctx or default_context()
    out = np.zeros(4, np.int64)
    ctx.check(ctx._l.eigmod_b200_stage_calls(ctx.h, out.ctypes.data_as(_I64)))
    return dict(zip(("project", "plan", "solve", "columns"), (int(x) for x in out)))


# ------------------------------------------- single eigenpairs, secular function
def null_problem(u, signs, lam, lam_new, ctx: Context | None = None) -> np.ndarray:
    """eigvec.hpp:19 — I + J U^T (Lambda - lambda' I)^{-1} U (k x k)."""
    ctx = ctx or default_context()
    u, signs, lam = _f64(u), _i32(signs), _f64(lam)
    n, k = u.shape
    if lam.shape[0] != n:
        raise ValueError("null_problem: dimension mismatch")
    m = np.empty((k, k))
    ctx.check(ctx._l.eigmod_b200_null_problem(ctx.h, _dp(u), signs.ctypes.data_as(_I32),
                                              _dp(lam), n, k, C.c_double(lam_new), _dp(m)))
    return m


def null_direction(m) -> tuple[np.ndarray, float]:
    """eigvec.hpp:15 — smallest singular direction of a k x k matrix."""
    m = _f64(m)
    k = m.shape[0]
    if m.shape != (k, k) or k == 0:
        raise ValueError("null_direction: square matrix required")
    d, r = np.empty(k), np.zeros(1)
    rc = lib().eigmod_b200_null_direction(_dp(m), k, _dp(d), _dp(r))
    if rc:
        raise ValueError("null_direction: square matrix required")
    return d, float(r[0])


def update_eigenvector(q, lam, kmat, signs, lam_new, ctx: Context | None = None) -> np.ndarray:
    """eigvec.hpp:25 — one updated eigenvector."""
    ctx = ctx or default_context()
    q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
    _check_update(q, lam, kmat, signs)
    n, k = kmat.shape
    v = np.empty(n)
    ctx.check(ctx._l.eigmod_b200_update_eigenvector(ctx.h, _dp(q), _dp(lam), _dp(kmat),
                                                    signs.ctypes.data_as(_I32), n, k,
                                                    C.c_double(lam_new), _dp(v)))
    return v


def secular_eval(poles, weights, xs, leading=1.0, derivative=False, ctx: Context | None = None):
    """eval_secular (+ eval_secular_derivative) at many points on the device;
    returns (f, f' or None, hit)."""
    ctx = ctx or default_context()
    poles, weights, xs = _f64(poles), _f64(weights), _f64(np.atleast_1d(xs))
    f, hit = np.empty(len(xs)), np.zeros(len(xs), np.int32)
    fp = np.empty(len(xs)) if derivative else None
    ctx.check(ctx._l.eigmod_b200_secular_eval(ctx.h, _dp(poles), _dp(weights), len(poles),
                                              C.c_double(leading), _dp(xs), len(xs), _dp(f),
                                              _dp(fp) if derivative else None,
                                              hit.ctypes.data_as(_I32)))
    return f, fp, hit


def crossing_count(poles, weights, lo, hi, samples, leading=1.0, ctx: Context | None = None):
    """secular.hpp:48."""
    ctx = ctx or default_context()
    poles, weights = _f64(poles), _f64(weights)
    out = np.zeros(1, np.int64)
    ctx.check(ctx._l.eigmod_b200_crossing_count(ctx.h, _dp(poles), _dp(weights), len(poles),
                                                C.c_double(leading), C.c_double(lo),
                                                C.c_double(hi), int(samples),
                                                out.ctypes.data_as(_I64)))
    return int(out[0])


def dnc_solve(poles, weights, lo, hi, expected, tol, leading=1.0, ctx: Context | None = None,
              stats=False):
    """rootfind.hpp:28 — the `expected` roots in (lo, hi), ascending."""
    ctx = ctx or default_context()
    poles, weights = _f64(poles), _f64(weights)
    out = np.empty(max(1, int(expected)))
    nr, ev, rd = (np.zeros(1, np.int64) for _ in range(3))
    ctx.check(ctx._l.eigmod_b200_dnc_solve(ctx.h, _dp(poles), _dp(weights), len(poles),
                                           C.c_double(leading), C.c_double(lo), C.c_double(hi),
                                           int(expected), C.c_double(tol), _dp(out),
                                           nr.ctypes.data_as(_I64), ev.ctypes.data_as(_I64),
                                           rd.ctypes.data_as(_I64)))
    r = out[: int(nr[0])].copy()
    return (r, {"evaluations": int(ev[0]), "rounds": int(rd[0])}) if stats else r


def solve_rank1(poles, zeta, sigma, tol, ctx: Context | None = None) -> np.ndarray:
    """rootfind.hpp:33 — eigenvalues of diag(poles) + sigma zeta zeta^T."""
    ctx = ctx or default_context()
    poles, zeta = _f64(poles), _f64(zeta)
    if zeta.shape != poles.shape or len(poles) == 0:
        raise ValueError("solve_rank1: bad inputs")
    out = np.empty(len(poles))
    ctx.check(ctx._l.eigmod_b200_solve_rank1(ctx.h, _dp(poles), _dp(zeta), len(poles),
                                             C.c_double(sigma), C.c_double(tol), _dp(out)))
    return out


def locate_coeffs(poles, weights, leading=1.0, ctx: Context | None = None) -> list[int]:
    """locate.hpp:31,50 — root counts per pole interval from the coefficients."""
    ctx = ctx or default_context()
    poles, weights = _f64(poles), _f64(weights)
    out = np.zeros(len(poles) + 1, np.int64)
    ctx.check(ctx._l.eigmod_b200_locate_coeffs(ctx.h, _dp(poles), _dp(weights), len(poles),
                                               C.c_double(leading), out.ctypes.data_as(_I64)))
    return [int(x) for x in out]


def gemm(a, b, trans_a=False, trans_b=False, ctx: Context | None = None) -> np.ndarray:
    """kernels.hpp:19-21 — op(A) op(B) on the DMMA GEMM."""
    ctx = ctx or default_context()
    a, b = _f64(a), _f64(b)
    m, kk = (a.shape[1], a.shape[0]) if trans_a else a.shape
    kb, nn = (b.shape[1], b.shape[0]) if trans_b else b.shape
    if kb != kk:
        raise ValueError("gemm: dimension mismatch")
    c = np.empty((m, nn))
    ctx.check(ctx._l.eigmod_b200_gemm(ctx.h, int(trans_a), int(trans_b), _dp(a), _dp(b), m, nn,
                                      kk, _dp(c)))
    return c


def split(n: int, world: int, rank: int) -> tuple[int, int]:
    """The C ABI's partition of [0, n) across `world` ranks."""
    lo, hi = np.zeros(1, np.int64), np.zeros(1, np.int64)
    rc = lib().eigmod_b200_split(int(n), int(world), int(rank), lo.ctypes.data_as(_I64),
                                 hi.ctypes.data_as(_I64))
    if rc:
        raise ValueError("split: bad arguments")
    return int(lo[0]), int(hi[0])


class MultiContext:
    """Single-process multi-GPU context (one device per rank, NCCL)."""

    def __init__(self, devices):
        self._l = lib()
        dv = np.ascontiguousarray(devices, dtype=np.int32)
        h = _VP()
        rc = self._l.eigmod_b200_multi_create(dv.ctypes.data_as(_I32), len(dv), C.byref(h))
        if rc == 1:
            raise ValueError(f"multi_create: bad device list {list(devices)}")
        if rc != 0:
            raise DeviceError(f"eigmod_b200_multi_create({list(devices)}) failed (rc={rc})")
        self.h = h
        self.devices = [int(d) for d in dv]

    def close(self):
        if getattr(self, "h", None):
            self._l.eigmod_b200_multi_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc):
        if rc == 0:
            return
        msg = (self._l.eigmod_b200_multi_last_error(self.h) or b"").decode()
        stage = (self._l.eigmod_b200_multi_last_stage(self.h) or b"").decode()
        if rc == 1:
            raise ValueError(msg)
        if rc == 2:
            raise NumericalError(stage, msg)
        raise DeviceError(msg)

    def set_option(self, key, value):
        self.check(self._l.eigmod_b200_multi_set_option(self.h, key.encode(), C.c_double(value)))

    def update_decomposition(self, q, lam, kmat, signs, tol) -> UpdateResult:
        q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
        _check_update(q, lam, kmat, signs)
        n, k = kmat.shape
        lo, qo, wt = np.empty(n), np.empty((n, n)), np.zeros(1)
        self.check(self._l.eigmod_b200_multi_update_decomposition(
            self.h, _dp(q), _dp(lam), _dp(kmat), signs.ctypes.data_as(_I32), n, k,
            C.c_double(tol), _dp(lo), _dp(qo), _dp(wt)))
        return UpdateResult(lo, qo, wall_time=float(wt[0]))

    def update_eigenvalues(self, q, lam, kmat, signs, tol) -> np.ndarray:
        q, lam, kmat, signs = _f64(q), _f64(lam), _f64(kmat), _i32(signs)
        _check_update(q, lam, kmat, signs)
        n, k = kmat.shape
        vals = np.empty(n)
        self.check(self._l.eigmod_b200_multi_update_eigenvalues(
            self.h, _dp(q), _dp(lam), _dp(kmat), signs.ctypes.data_as(_I32), n, k,
            C.c_double(tol), _dp(vals)))
        return vals


def default_tolerance(lam, kmat) -> float:
    """rootfind.cpp:306-312."""
    scale = max(1.0, float(np.max(np.abs(lam))) if len(lam) else 1.0)
    kn = float(np.linalg.norm(kmat))
    return 1e-12 * max(scale, kn * kn)


# --------------------------------------------------------- device (torch) API
def _ptr(t):
    return _VP(t.data_ptr())


def launch_count() -> int:
    """Kernels launched by libeigmod_b200.so in this process."""
    return int(lib().eigmod_b200_launch_count())


def padded_rank(k: int) -> int:
    return int(lib().eigmod_b200_padded_rank(int(k)))


def record_width(kp: int) -> int:
    return int(lib().eigmod_b200_record_width(int(kp)))


def check_device_operands(ctx, ops):
    """The C ABI takes raw device pointers to dense row-major float64 with
    leading dimension = the column count: reject anything else before the
    call (a float32, strided or wrongly sized tensor would otherwise be read
    out of bounds or silently misinterpreted)."""
    import torch

    for name, (t, shape) in ops.items():
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name}: expected a torch CUDA tensor")
        if t.dtype != torch.float64:
            raise TypeError(f"{name}: expected float64, got {t.dtype}")
        if t.device.type != "cuda" or (t.device.index or 0) != ctx.device:
            raise ValueError(f"{name}: expected a tensor on cuda:{ctx.device}, got {t.device}")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
        if not t.is_contiguous():
            raise ValueError(f"{name}: expected a contiguous (row-major) tensor")


def update_decomposition_device(q, lam, kmat, signs, lam_out, q_out, ctx: Context | None = None):
    """All-device update on torch CUDA float64 tensors (runs on torch's
    current stream)."""
    import torch

    ctx = ctx or default_context(q.device.index or 0)
    n, k = kmat.shape
    check_device_operands(ctx, {"q": (q, (n, n)), "lam": (lam, (n,)), "kmat": (kmat, (n, k)),
                                "lam_out": (lam_out, (n,)), "q_out": (q_out, (n, n))})
    ctx.set_stream(torch.cuda.current_stream(q.device).cuda_stream)
    sg = _i32(np.asarray(signs))
    if sg.shape != (k,):
        raise ValueError(f"signs: expected {k} entries, got {sg.shape}")
    ctx.check(ctx._l.eigmod_b200_update_decomposition_device(
        ctx.h, _ptr(q), _ptr(lam), _ptr(kmat), sg.ctypes.data_as(_I32), n, k, _ptr(lam_out),
        _ptr(q_out)))


def gemm_nt_device(a, b, c, ctx: Context | None = None):
    import torch

    ctx = ctx or default_context(a.device.index or 0)
    m, kk = a.shape
    nn = b.shape[0]
    check_device_operands(ctx, {"a": (a, (m, kk)), "b": (b, (nn, kk))})
    if c.dtype != torch.float64 or tuple(c.shape) != (m, nn) or c.stride(1) != 1:
        raise ValueError("c: expected a float64 (m, nn) tensor with unit column stride")
    ctx.set_stream(torch.cuda.current_stream(a.device).cuda_stream)
    ctx.check(ctx._l.eigmod_b200_gemm_nt_device(ctx.h, _ptr(a), _ptr(b), m, nn, kk, _ptr(c),
                                                 c.stride(0)))
