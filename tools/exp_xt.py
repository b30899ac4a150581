"""K4 (Xt columns) stage time, v1 vs tile64 kernel (dev tool): run twice with
EIGMOD_B200_XT unset / =v1."""
import os
import sys

sys.path.insert(0, '.')
import torch

from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch

dev = torch.device('cuda', 0)
for cfg, n in [(4, 32768), (3, 16384), (2, 8192)]:
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    ctx = capi.Context(0)
    ctx.set_option('timing', 1)
    lo = torch.empty(n, dtype=torch.float64, device=dev)
    qo = torch.empty((n, n), dtype=torch.float64, device=dev)
    for rep in range(2):
        ctx.stage_times(reset=True)
        capi.update_decomposition_device(q, lam, kmat, signs.numpy(), lo, qo, ctx=ctx)
        torch.cuda.synchronize()
    st = ctx.stage_times()
    sg = signs.to(dev, torch.float64)
    orth = float((qo[:, :2048].T @ qo[:, :2048] - torch.eye(2048, dtype=torch.float64, device=dev)).abs().max())
    print(f"XT={os.environ.get('EIGMOD_B200_XT', 'v3')} cfg{cfg} n={n}: k4 {st['k4_columns']:.2f} ms "
          f"gemm {st['k5_gemm']:.1f} ms orth(2048 cols) {orth:.2e} sum(lo) {float(lo.sum()):.15e} "
          f"qsum {float(qo.abs().sum()):.15e}", flush=True)
    del q, qo
    torch.cuda.empty_cache()
