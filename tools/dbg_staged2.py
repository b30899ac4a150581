import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance
from paper_1706_00773_b200.sharded import CudaBackend, split
api = capi; ctx = capi.default_context(0)
q, lam, kmat, s = make_instance(2, n=700, seed=5)
dev = torch.device("cuda", 0)
tq, tl, tk = (torch.from_numpy(x).to(dev) for x in (q, lam, kmat))
n, k = kmat.shape
lo1 = torch.empty(n, dtype=torch.float64, device=dev)
qo1 = torch.empty((n, n), dtype=torch.float64, device=dev)
api.update_decomposition_device(tq, tl, tk, s, lo1, qo1, ctx=ctx)
ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
be = CudaBackend(ctx, n, k, s)
world = 2
u_all = torch.zeros((split(n, world, 0)[2] * world, be.kp), dtype=torch.float64, device=dev)
for r in range(world):
    a, b, ch = split(n, world, r)
    part = torch.zeros((ch, be.kp), dtype=torch.float64, device=dev)
    be.project(tq, tk, a, b, part)
    u_all[r * ch: r * ch + (b - a)] = part[: b - a]
nred = be.plan(tl, u_all[:n])
recs = []
for r in range(world):
    j0, j1, jc = split(nred, world, r)
    part = torch.zeros((jc, be.width), dtype=torch.float64, device=dev)
    be.solve(j0, j1, part)
    recs.append(part[: j1 - j0])
rec_all = torch.cat(recs)
lo2 = torch.empty(n, dtype=torch.float64, device=dev)
qo2 = torch.zeros((n, n), dtype=torch.float64, device=dev)
for r in range(world):
    c0, c1, _ = split(n, world, r)
    blk = torch.empty((n, c1 - c0), dtype=torch.float64, device=dev)
    be.finish(tq, rec_all, c0, c1, lo2, blk)
    torch.cuda.synchronize()
    print(r, c0, c1, blk.shape, blk.stride(), (blk - qo1[:, c0:c1]).abs().max().item(), flush=True)
    qo2[:, c0:c1] = blk
torch.cuda.synchronize()
d = (qo1 - qo2).abs().max(0).values
print("cols differing:", torch.nonzero(d).flatten().tolist()[:20], d.max().item())
