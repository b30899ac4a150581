"""Solve-stage time vs thread-block cluster size and root-range size (dev tool)."""
import sys

sys.path.insert(0, '.')
import torch

from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
from paper_1706_00773_b200.sharded import CudaBackend, split

dev = torch.device('cuda', 0)
for cfg, n in [(4, 32768), (2, 8192), (4, 8192)]:
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    k = kmat.shape[1]
    ctx = capi.Context(0)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    be = CudaBackend(ctx, n, k, signs.numpy())
    u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
    be.project(q, kmat, 0, n, u)
    nred = be.plan(lam, u)
    print(f"cfg{cfg} n={n} nred={nred}", flush=True)
    for world in (1, 2, 4, 8):
        j0, j1, _ = split(nred, world, world // 2)
        rec = torch.zeros((j1 - j0, be.width), dtype=torch.float64, device=dev)
        row = []
        for cl in (1, 2, 4, 8):
            ctx.set_option('cluster', cl)
            best = 1e30
            for _ in range(2):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record()
                be.solve(j0, j1, rec)
                b.record()
                torch.cuda.synchronize()
                best = min(best, a.elapsed_time(b))
            row.append(best)
        print(f"  roots {j1 - j0:6d}: " + "  ".join(f"CL{c}={t:7.2f}" for c, t in zip((1, 2, 4, 8), row)),
              flush=True)
    ctx.set_option('sweep', 0)
    ctx.set_option('cluster', 4)
    rec = torch.zeros((nred, be.width), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    be.solve(0, nred, rec)
    b.record()
    torch.cuda.synchronize()
    print(f"  no-sweep full CL4: {a.elapsed_time(b):.2f}", flush=True)
