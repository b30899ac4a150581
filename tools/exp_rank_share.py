"""Per-rank device time of the root/column-partitioned update (dev tool).

Runs one rank's share of each stage on one GPU (no collectives; every rank's
inputs are the single-GPU intermediate results) and prints the stage times
of the slowest rank next to the one-GPU step: the compute side of the weak /
strong scaling estimate. Usage: python tools/exp_rank_share.py [cfg] [n]
"""
import sys

sys.path.insert(0, '.')
import torch

from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
from paper_1706_00773_b200.sharded import CudaBackend, split

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
dev = torch.device('cuda', 0)
q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
k = kmat.shape[1]
ctx = capi.Context(0)
ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
be = CudaBackend(ctx, n, k, signs.numpy())


def t(fn, reps=2):
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
be.project(q, kmat, 0, n, u)
nred = be.plan(lam, u)
rec_all = torch.zeros((max(nred, 1), be.width), dtype=torch.float64, device=dev)
be.solve(0, nred, rec_all)
lo = torch.empty(n, dtype=torch.float64, device=dev)
for world in (1, 2, 4, 8):
    worst = None
    for r in range(world):
        a, b, ch = split(n, world, r)
        part = torch.zeros((ch, be.kp), dtype=torch.float64, device=dev)
        tp = t(lambda: be.project(q, kmat, a, b, part))
        ng = be.plan_groups(lam, u)
        g0, g1, gc = split(ng, world, r)
        ap = torch.zeros(max(gc, 1), dtype=torch.float64, device=dev)
        tg = t(lambda: be.plan_groups(lam, u))
        tw = t(lambda: be.plan_weights(g0, g1, ap))
        alpha = torch.zeros(ng, dtype=torch.float64, device=dev)
        be.plan_weights(0, ng, alpha)
        tf = t(lambda: be.plan_finish(alpha))
        j0, j1, jc = split(nred, world, r)
        rp = torch.zeros((max(jc, 1), be.width), dtype=torch.float64, device=dev)
        ts = t(lambda: be.solve(j0, j1, rp)) if j1 > j0 else 0.0
        c0, c1, _ = split(n, world, r)
        blk = torch.empty((n, max(c1 - c0, 1)), dtype=torch.float64, device=dev)
        tq = t(lambda: be.finish(q, rec_all, c0, c1, lo, blk), reps=2)
        del blk
        row = dict(project=tp, groups=tg, weights=tw, finish_plan=tf, solve=ts, finish=tq)
        row['total'] = sum(row.values())
        if worst is None or row['total'] > worst['total']:
            worst = row
    if world == 1:
        one = worst['total']
    print(f"world {world}: slowest rank {worst['total']:.1f} ms (ideal {one / world:.1f}, "
          f"eff {one / world / worst['total']:.3f}) " +
          " ".join(f"{kk}={v:.1f}" for kk, v in worst.items() if kk != 'total'), flush=True)
