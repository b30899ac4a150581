"""Solve time and evaluations with and without the pole-limit split (dev tool)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
from paper_1706_00773_b200.sharded import CudaBackend
dev = torch.device('cuda', 0)
for cfg, n in [(4, 32768), (3, 16384), (2, 8192)]:
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    ctx = capi.Context(0)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    be = CudaBackend(ctx, n, kmat.shape[1], signs.numpy())
    u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
    be.project(q, kmat, 0, n, u)
    nred = be.plan(lam, u)
    rec = torch.zeros((nred, be.width), dtype=torch.float64, device=dev)
    for ps in (0, 1, 0, 1):
        ctx.set_option('pole_split', ps)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); be.solve(0, nred, rec); b.record(); torch.cuda.synchronize()
        ev = rec[:, 4]
        print(f"cfg{cfg} n={n} pole_split={ps}: {a.elapsed_time(b):.2f} ms evals/root {float(ev.mean()):.3f} max {int(ev.max())}", flush=True)
