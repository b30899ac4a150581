import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance
from paper_1706_00773_b200.sharded import CudaBackend, split
ctx = capi.default_context(0)
q, lam, kmat, s = make_instance(2, n=700, seed=5)
dev = torch.device("cuda", 0)
tq, tl, tk = (torch.from_numpy(x).to(dev) for x in (q, lam, kmat))
n, k = kmat.shape
ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
be = CudaBackend(ctx, n, k, s)
u_full = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
be.project(tq, tk, 0, n, u_full)
nred = be.plan(tl, u_full)
print("nred", nred, "width", be.width)
recA = torch.zeros((nred, be.width), dtype=torch.float64, device=dev)
be.solve(0, nred, recA)
recB = torch.zeros((nred, be.width), dtype=torch.float64, device=dev)
be.solve(0, 350, recB[:350]); be.solve(350, nred, recB[350:])
torch.cuda.synchronize()
print("rec diff", (recA-recB).abs().max().item(), recA[348:352,:5])
for (c0,c1) in [(0,350),(350,700),(0,700)]:
    blk = torch.zeros((n, c1-c0), dtype=torch.float64, device=dev)
    lo = torch.empty(n, dtype=torch.float64, device=dev)
    be.finish(tq, recA, c0, c1, lo, blk)
    torch.cuda.synchronize()
    print(c0, c1, blk.abs().max().item(), blk.abs().sum(0)[:3].tolist(), blk.abs().sum(0)[-3:].tolist())
