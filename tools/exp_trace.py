"""Iterate trace of the most expensive roots (dev tool)."""
import sys

sys.path.insert(0, '.')
import numpy as np
import torch

from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
from paper_1706_00773_b200.sharded import CudaBackend

np.set_printoptions(linewidth=220, precision=6)
dev = torch.device('cuda', 0)
cfg, n = int(sys.argv[1]), int(sys.argv[2])
q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
k = kmat.shape[1]
ctx = capi.Context(0)
ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
be = CudaBackend(ctx, n, k, signs.numpy())
u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
be.project(q, kmat, 0, n, u)
nred = be.plan(lam, u)
rec = torch.zeros((nred, be.width), dtype=torch.float64, device=dev)
be.solve(0, nred, rec)
r = rec.cpu().numpy()
ev = r[:, 4].astype(int)
order = np.argsort(-ev)
picks = [order[0], order[5], order[50], order[200]]
for j in picks:
    ctx.set_option('trace_root', int(j))
    be.solve(0, nred, rec)
    tr = ctx.solver_trace()
    print(f"root {j}: evals {ev[j]} value {r[j, 0]!r} origin {int(r[j, 1])} delta {r[j, 2]:.6e}")
    print("   it ph fm/cnt        delta           lo             hi              f            f'        sigma          g          step")
    for row in tr:
        print(f"  {int(row[0]):3d} {int(row[1])} {int(row[2]):4d} {row[3]: .8e} {row[4]: .6e} {row[5]: .6e} "
              f"{row[6]: .4e} {row[7]: .4e} {row[8]: .4e} {row[9]: .4e} {row[10]: .4e} o={int(row[11])}")
ctx.set_option('trace_root', -1)
