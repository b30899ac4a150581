"""Evaluations per root and accuracy for solver rule variants (dev tool)."""
import sys

sys.path.insert(0, '.')
import numpy as np
import torch

from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch

dev = torch.device('cuda', 0)
variants = [
    dict(floor_ulps=0.0, stall_ratio=1.0),   # previous rules
    dict(floor_ulps=4.0, stall_ratio=1.0),
    dict(floor_ulps=4.0, stall_ratio=0.5),
    dict(floor_ulps=16.0, stall_ratio=0.5),
]
for cfg, n in [(4, 16384), (2, 8192), (3, 16384), (1, 4096), (0, 512)]:
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    sg = signs.to(dev, torch.float64)
    lo = torch.empty(n, dtype=torch.float64, device=dev)
    qo = torch.empty((n, n), dtype=torch.float64, device=dev)
    a = q @ (lam[:, None] * q.T) + kmat @ (sg[:, None] * kmat.T)
    ev = torch.linalg.eigvalsh(0.5 * (a + a.T))
    del a
    for v in variants:
        ctx = capi.Context(0)
        ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
        ctx.set_option('timing', 1)
        for kk, vv in v.items():
            ctx.set_option(kk, vv)
        for _ in range(2):
            ctx.stage_times(reset=True)
            capi.update_decomposition_device(q, lam, kmat, signs.numpy(), lo, qo, ctx=ctx)
            torch.cuda.synchronize()
        st = ctx.stats()
        t = ctx.stage_times()
        nrm = float(lo.abs().max())
        r = q @ (lam[:, None] * (q.T @ qo)) + kmat @ (sg[:, None] * (kmat.T @ qo)) - qo * lo[None, :]
        resid = float(r.abs().max()) / nrm
        del r
        orth = float((qo.T @ qo - torch.eye(n, dtype=torch.float64, device=dev)).abs().max())
        everr = float((lo - ev).abs().max()) / nrm
        print(f"cfg{cfg} n={n} {v}: evals/root {st['evals'] / max(1, st['roots']):.3f} max {st['max_evals']:.0f} "
              f"solve {t['k3_solve']:.2f} ms resid {resid:.2e} orth {orth:.2e} eig {everr:.2e}", flush=True)
