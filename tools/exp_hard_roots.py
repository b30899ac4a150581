"""Evaluation counts of one rank's roots (dev tool): which roots set the tail."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
from paper_1706_00773_b200.sharded import CudaBackend, split
world, r = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device('cuda', 0)
q, lam, kmat, signs = make_instance_torch(4, n=32768, device=dev)
ctx = capi.Context(0)
ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
be = CudaBackend(ctx, 32768, 16, signs.numpy())
u = torch.zeros((32768, be.kp), dtype=torch.float64, device=dev)
be.project(q, kmat, 0, 32768, u)
nred = be.plan(lam, u)
j0, j1, _ = split(nred, world, r)
rec = torch.zeros((j1 - j0, be.width), dtype=torch.float64, device=dev)
be.solve(j0, j1, rec)
torch.cuda.synchronize()
R = rec.cpu().numpy()
ev = R[:, 4].astype(int)
fl = R[:, 3].astype(int)
itA = (fl >> 8) & 255
print(f"world {world} rank {r}: roots {j1 - j0} evals mean {ev.mean():.2f} max {ev.max()}")
print("  hist", np.bincount(ev)[:40].tolist())
top = np.argsort(-ev)[:12]
for t in top:
    print(f"   root {j0 + t}: evals {ev[t]} phaseA {itA[t]} flags {fl[t] & 255}")
