"""Solver slot utilisation and per-pass time (dev tool)."""
import os
import sys

sys.path.insert(0, '.')
import torch

from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
from paper_1706_00773_b200.sharded import CudaBackend, split

dev = torch.device('cuda', 0)
cases = [(4, 32768), (2, 8192), (4, 8192)][: int(os.environ.get('EXP_NCASES', '3'))]
for cfg, n in cases:
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    k = kmat.shape[1]
    ctx = capi.Context(0)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    import os
    for kv in os.environ.get("EIGMOD_OPTS", "").split(","):
        if kv:
            kk, vv = kv.split("=")
            ctx.set_option(kk, float(vv))
    be = CudaBackend(ctx, n, k, signs.numpy())
    u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
    be.project(q, kmat, 0, n, u)
    nred = be.plan(lam, u)
    for world in (1, 8):
        j0, j1, _ = split(nred, world, world // 2)
        rec = torch.zeros((j1 - j0, be.width), dtype=torch.float64, device=dev)
        for sweep in (1, 0):
            ctx.set_option('sweep', sweep)
            for _ in range(2):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record()
                be.solve(j0, j1, rec)
                b.record()
                torch.cuda.synchronize()
            t = a.elapsed_time(b)
            pr = ctx.solver_profile()
            ev = float(rec[:, 4].sum())
            per_batch = pr['passes'] / max(1, pr['batches'])
            print(f"cfg{cfg} n={n} roots={j1 - j0} sweep={sweep}: {t:8.2f} ms evals {ev:.0f} "
                  f"({ev / (j1 - j0):.2f}/root) batches {pr['batches']:.0f} passes/batch {per_batch:.1f} "
                  f"slot util {pr['slot_util']:.3f}  ms/pass {t / max(1, per_batch):.3f}", flush=True)
        ctx.set_option('sweep', 1)
