"""Root/column-partitioned update across GPUs (one process per GPU).

SURVEY.md §8(e): every rank holds Lambda, U and Q (Q replicated). The only
exchanges are
  1. all-gather of U: rank r projects U rows [r*C, (r+1)*C) (Q columns),
  1b. all-gather of the K2 pole weights: rank r computes its group slice,
  2. all-gather of the root records: rank r solves root indices of its slice,
then rank r writes the column block [c0, c1) of Q' = Q X locally. The plan
(deflation, reduced problem) is computed redundantly on every rank from the
same bits, so every rank sees the same roots and the same column order.

The driver is backend-agnostic: ``CudaBackend`` calls the C ABI staged entry
points (eigmod_b200_project/plan/solve/finish_device); tests drive the same
code with a CPU stand-in over gloo (tests/test_sharded.py).
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def split(n: int, world: int, rank: int) -> tuple[int, int, int]:
    """Equal chunks of ceil(n/world); returns (lo, hi, chunk)."""
    c = -(-n // world) if n > 0 else 0
    lo = min(n, rank * c)
    hi = min(n, lo + c)
    return lo, hi, c


class CudaBackend:
    """Staged C-ABI calls on torch CUDA tensors (current stream)."""

    def __init__(self, ctx, n, k, signs):
        from . import capi

        self.capi = capi
        self.ctx = ctx
        self.n, self.k = n, k
        self.signs = np.ascontiguousarray(signs, dtype=np.int32)
        self.kp = capi.padded_rank(k)
        self.width = capi.record_width(self.kp)

    @staticmethod
    def capi_f64():
        import torch

        return torch.float64

    def project(self, q, kmat, lo, hi, u_out):
        c = self.ctx
        self.capi.check_device_operands(c, {"q": (q, (self.n, self.n)),
                                            "kmat": (kmat, (self.n, self.k))})
        c.check(c._l.eigmod_b200_project_device(c.h, C.c_void_p(q.data_ptr()),
                                                C.c_void_p(kmat.data_ptr()), self.n, self.k, lo,
                                                hi, C.c_void_p(u_out.data_ptr())))

    def plan(self, lam, u_full) -> int:
        c = self.ctx
        nr = np.zeros(1, np.int64)
        c.check(c._l.eigmod_b200_plan_device(
            c.h, C.c_void_p(lam.data_ptr()), C.c_void_p(u_full.data_ptr()),
            self.signs.ctypes.data_as(C.POINTER(C.c_int)), self.n, self.k,
            nr.ctypes.data_as(C.POINTER(C.c_int64))))
        return int(nr[0])

    def plan_groups(self, lam, u_full) -> int:
        c = self.ctx
        ng = np.zeros(1, np.int64)
        c.check(c._l.eigmod_b200_plan_groups_device(
            c.h, C.c_void_p(lam.data_ptr()), C.c_void_p(u_full.data_ptr()),
            self.signs.ctypes.data_as(C.POINTER(C.c_int)), self.n, self.k,
            ng.ctypes.data_as(C.POINTER(C.c_int64))))
        return int(ng[0])

    def plan_weights(self, g0, g1, alpha_out):
        c = self.ctx
        c.check(c._l.eigmod_b200_plan_weights_device(c.h, g0, g1,
                                                     C.c_void_p(alpha_out.data_ptr())))

    def plan_finish(self, alpha_all) -> int:
        c = self.ctx
        nr = np.zeros(1, np.int64)
        c.check(c._l.eigmod_b200_plan_finish_device(c.h, C.c_void_p(alpha_all.data_ptr()),
                                                    nr.ctypes.data_as(C.POINTER(C.c_int64))))
        return int(nr[0])

    def solve(self, j0, j1, rec_out):
        c = self.ctx
        c.check(c._l.eigmod_b200_solve_device(c.h, j0, j1, C.c_void_p(rec_out.data_ptr())))

    def finish(self, q, rec_all, c0, c1, lam_out, q_out):
        c = self.ctx
        self.capi.check_device_operands(c, {"q": (q, (self.n, self.n)),
                                            "lam_out": (lam_out, (self.n,))})
        if q_out.dtype != self.capi_f64() or q_out.shape[0] != self.n or q_out.stride(1) != 1 \
                or q_out.shape[1] < c1 - c0:
            raise ValueError("q_out: expected float64 (n, >= c1 - c0) with unit column stride")
        c.check(c._l.eigmod_b200_finish_device(
            c.h, C.c_void_p(q.data_ptr()), C.c_void_p(rec_all.data_ptr()), c0, c1,
            C.c_void_p(lam_out.data_ptr()), C.c_void_p(q_out.data_ptr()), q_out.stride(0)))


class ShardedUpdate:
    """One rank's share of a root/column-partitioned update."""

    def __init__(self, ctx_or_backend, n, k, signs, rank, world, device, group=None):
        import torch

        self.torch = torch
        if hasattr(ctx_or_backend, "project"):
            self.be = ctx_or_backend
        else:
            self.be = CudaBackend(ctx_or_backend, n, k, signs)
        self.n, self.k = n, k
        self.rank, self.world = rank, world
        self.device = device
        self.group = group
        self.kp = self.be.kp
        self.width = self.be.width
        self.u_lo, self.u_hi, self.u_chunk = split(n, world, rank)
        self.c0, self.c1, _ = split(n, world, rank)
        self.ncols_local = self.c1 - self.c0
        f64 = torch.float64
        self.u_part = torch.zeros((self.u_chunk, self.kp), dtype=f64, device=device)
        self.u_all = torch.zeros((self.u_chunk * world, self.kp), dtype=f64, device=device)

    def alloc_output(self):
        return self.torch.empty((self.n, max(self.ncols_local, 1)), dtype=self.torch.float64,
                                device=self.device)

    def run(self, q, lam, kmat, lam_out, q_out):
        import torch.distributed as dist

        torch = self.torch
        # 1. U slice + all-gather
        if self.u_hi > self.u_lo:
            self.be.project(q, kmat, self.u_lo, self.u_hi, self.u_part)
        dist.all_gather_into_tensor(self.u_all, self.u_part, group=self.group)
        u_full = self.u_all[: self.n]
        # 2. plan: groups on every rank, the K2 weights shared out by group
        #    slices and all-gathered, then the (redundant, cheap) reduction
        ng = self.be.plan_groups(lam, u_full)
        g0, g1, gc = split(ng, self.world, self.rank)
        gc = max(gc, 1)
        a_part = torch.zeros(gc, dtype=torch.float64, device=self.device)
        a_all = torch.zeros(gc * self.world, dtype=torch.float64, device=self.device)
        if g1 > g0:
            self.be.plan_weights(g0, g1, a_part)
        dist.all_gather_into_tensor(a_all, a_part, group=self.group)
        nred = self.be.plan_finish(a_all[: max(ng, 1)])
        # 3. roots of this rank + all-gather of the records
        j0, j1, jc = split(nred, self.world, self.rank)
        jc = max(jc, 1)
        rec_part = torch.zeros((jc, self.width), dtype=torch.float64, device=self.device)
        rec_all = torch.zeros((jc * self.world, self.width), dtype=torch.float64,
                              device=self.device)
        if j1 > j0:
            self.be.solve(j0, j1, rec_part)
        dist.all_gather_into_tensor(rec_all, rec_part, group=self.group)
        # 4. this rank's column block of Q' (+ all eigenvalues)
        self.be.finish(q, rec_all[: max(nred, 1)], self.c0, self.c1, lam_out, q_out)
