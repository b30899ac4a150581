import sys; sys.path.insert(0,'.')
import torch, numpy as np
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch, CONFIGS
from paper_1706_00773_b200.sharded import CudaBackend
dev = torch.device("cuda", 0)
for cfg, n in [(0, 512), (1, 4096), (2, 8192), (4, 8192), (3, 4096)]:
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    ctx = capi.Context(0); ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    be = CudaBackend(ctx, n, CONFIGS[cfg]["k"], signs.numpy())
    u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
    be.project(q, kmat, 0, n, u); nred = be.plan(lam, u)
    rec = torch.zeros((nred, be.width), dtype=torch.float64, device=dev)
    be.solve(0, nred, rec); torch.cuda.synchronize()
    R = rec.cpu().numpy(); fl = R[:, 3].astype(int); ev = R[:, 4]
    A = fl >> 8; B = ev - A
    print(f"cfg{cfg} n={n}: evals mean {ev.mean():.2f} max {ev.max():.0f} | phaseA mean {A.mean():.2f} p50 {np.median(A):.0f} p99 {np.percentile(A,99):.0f} | phaseB mean {B.mean():.2f} p99 {np.percentile(B,99):.0f} | flags {np.bincount(fl & 3)}", flush=True)
    ctx.close()
