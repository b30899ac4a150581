"""Histogram of S evaluations per root and where the expensive roots sit (dev tool)."""
import sys

sys.path.insert(0, '.')
import numpy as np
import torch

from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
from paper_1706_00773_b200.sharded import CudaBackend

dev = torch.device('cuda', 0)
for cfg, n in [(4, 32768), (2, 8192), (3, 16384)]:
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    k = kmat.shape[1]
    ctx = capi.Context(0)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    be = CudaBackend(ctx, n, k, signs.numpy())
    u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
    be.project(q, kmat, 0, n, u)
    nred = be.plan(lam, u)
    rec = torch.zeros((nred, be.width), dtype=torch.float64, device=dev)
    be.solve(0, nred, rec)
    r = rec.cpu().numpy()
    ev = r[:, 4].astype(int)
    flr = r[:, 3].astype(int)
    fl = flr & 255
    ia = flr >> 8
    h = np.bincount(ev)
    print(f"cfg{cfg} n={n} nred={nred} mean {ev.mean():.2f} max {ev.max()} flags {np.bincount(fl)}")
    print("  evals histogram:", {i: int(c) for i, c in enumerate(h) if c})
    hard = np.nonzero(ev >= 12)[0]
    print("  roots with >= 12 evals:", len(hard), "first idx", hard[:20])
    # relative gap of the root to its origin pole, for hard vs easy roots
    val, dl = r[:, 0], r[:, 2]
    for lo_, hi_ in [(0, 8), (8, 12), (12, 20), (20, 100)]:
        m = (ev >= lo_) & (ev < hi_)
        if m.any():
            print(f"  evals [{lo_},{hi_}): phase-A iters mean {ia[m].mean():.2f}, B iters mean {(ev[m] - ia[m]).mean():.2f}")
    lamh = lam.cpu().numpy()
    rel = np.abs(dl) / np.maximum(np.abs(val), 1e-300)
    for lo_, hi_ in [(0, 8), (8, 12), (12, 20), (20, 100)]:
        m = (ev >= lo_) & (ev < hi_)
        if m.any():
            print(f"  evals [{lo_},{hi_}): {m.sum():6d} roots, median |delta| {np.median(np.abs(dl[m])):.3e}")
