"""Iterate trace of given roots of config 4 (dev tool): python tools/exp_trace_root.py n j [j ...]"""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
from paper_1706_00773_b200.sharded import CudaBackend
n = int(sys.argv[1])
dev = torch.device('cuda', 0)
q, lam, kmat, signs = make_instance_torch(4, n=n, device=dev)
ctx = capi.Context(0)
ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
be = CudaBackend(ctx, n, 16, signs.numpy())
u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
be.project(q, kmat, 0, n, u)
nred = be.plan(lam, u)
rec = torch.zeros((nred, be.width), dtype=torch.float64, device=dev)
for j in [int(a) for a in sys.argv[2:]]:
    ctx.set_option('trace_root', j)
    be.solve(0, nred, rec)
    tr = ctx.solver_trace()
    r = rec[j].cpu().numpy()
    print(f"root {j}: evals {int(r[4])} value {r[0]!r} origin {int(r[1])} delta {r[2]:.6e}")
    print("   it ph fm/cnt        delta           lo             hi              f            f'        sigma          g          step")
    for row in tr:
        print(f"  {int(row[0]):3d} {int(row[1])} {int(row[2]):4d} {row[3]: .16e} {row[4]: .6e} {row[5]: .6e} "
              f"{row[6]: .4e} {row[7]: .4e} {row[8]: .4e} {row[9]: .4e} {row[10]: .4e} o={int(row[11])}")
ctx.set_option('trace_root', -1)
