"""Kernel-level breakdown of one rank's root solve at N ranks (dev tool)."""
import sys
sys.path.insert(0, '.')
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
from paper_1706_00773_b200.sharded import CudaBackend, split
world, r = int(sys.argv[1]) if len(sys.argv) > 1 else 8, int(sys.argv[2]) if len(sys.argv) > 2 else 4
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
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); be.solve(j0, j1, rec); b.record(); torch.cuda.synchronize()
print(f"world {world} rank {r}: solve {a.elapsed_time(b):.2f} ms")
for ev in prof.key_averages():
    if ev.device_time_total > 50:
        print(f"   {ev.key[:70]}: {ev.device_time_total / 1000:.2f} ms x{ev.count}")
