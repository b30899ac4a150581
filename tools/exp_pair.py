import sys; sys.path.insert(0,'.')
import torch, numpy as np
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
from paper_1706_00773_b200.sharded import CudaBackend
import oracle.port as port
dev = torch.device("cuda", 0)
cfg, n = 2, 8192
q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
ctx = capi.Context(0); ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
be = CudaBackend(ctx, n, 4, signs.numpy())
u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
be.project(q, kmat, 0, n, u)
nred = be.plan(lam, u)
rec = torch.zeros((nred, be.width), dtype=torch.float64, device=dev)
be.solve(0, nred, rec)
lo = torch.empty(n, dtype=torch.float64, device=dev); qo = torch.empty((n, n), dtype=torch.float64, device=dev)
be.finish(q, rec, 0, n, lo, qo)
torch.cuda.synchronize()
R = rec.cpu().numpy()
flags = R[:, 3].astype(int)
print("flags histogram", np.bincount(flags), "evals mean", R[:, 4].mean())
g = qo.T @ qo - torch.eye(n, dtype=torch.float64, device=dev)
col = g.abs().max(0).values.cpu().numpy()
worst = np.argsort(-col)[:8]
print("worst cols", worst, col[worst])
lh = lam.cpu().numpy(); uh = u[:, :4].cpu().numpy(); sg = signs.numpy()
for j in worst[:6]:
    o = int(R[j, 1]); d = R[j, 2]
    roots, orig, dl, ev = port.solve_roots(lh, uh, sg, int(j), int(j) + 1)
    gaps = np.sort(np.abs(lh - R[j, 0]))[:2]
    print(f"col {j}: root {R[j,0]:.17g} o {o} delta {d:.6e} flags {flags[j]} evals {R[j,4]:.0f} | oracle root {roots[0]:.17g} origin {orig[0]} delta {dl[0]:.6e} | diff {R[j,0]-roots[0]:.3e} pole gaps {gaps}")
    print("   y", R[j, 5:9])
