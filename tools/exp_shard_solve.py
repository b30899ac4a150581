"""Per-rank solve stage time for a root-partitioned update (dev tool).

Runs the staged C ABI on one GPU, one virtual rank after another (no
cross-rank waits), and prints the solve time of each rank's root range next
to the one-rank solve, i.e. the solver's weak-scaling share.
"""
import sys

sys.path.insert(0, '.')
import torch

from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
from paper_1706_00773_b200.sharded import CudaBackend, split

dev = torch.device('cuda', 0)
cfg, n = int(sys.argv[1]) if len(sys.argv) > 1 else 4, int(sys.argv[2]) if len(sys.argv) > 2 else 32768
q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
k = kmat.shape[1]
ctx = capi.Context(0)
ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
be = CudaBackend(ctx, n, k, signs.numpy())
u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
be.project(q, kmat, 0, n, u)
nred = be.plan(lam, u)


def timed(j0, j1, reps=2):
    rec = torch.zeros((max(j1 - j0, 1), be.width), dtype=torch.float64, device=dev)
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        be.solve(j0, j1, rec)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best, rec


full, rec_full = timed(0, nred)
print(f"cfg{cfg} n={n} nred={nred} one-rank solve {full:.2f} ms")
for world in (2, 4, 8):
    ts = []
    same = True
    for r in range(world):
        j0, j1, _ = split(nred, world, r)
        t, rec = timed(j0, j1)
        ts.append(t)
        same &= bool(torch.equal(rec[: j1 - j0], rec_full[j0:j1]))
    print(f"world {world}: max {max(ts):.2f} ms  ideal {full / world:.2f} ms  "
          f"eff {full / world / max(ts):.3f}  bit-identical {same}  per-rank "
          + " ".join(f"{t:.1f}" for t in ts))
