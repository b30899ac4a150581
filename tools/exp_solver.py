"""Solver stage time and accuracy for option variants (dev tool)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch, CONFIGS
dev = torch.device('cuda', 0)
for cfg, n in [(4, 8192), (2, 8192), (4, 32768)]:
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    sg = signs.to(dev, torch.float64)
    for opts in ({'cluster': 0}, {'cluster': 1}):
        ctx = capi.Context(0)
        ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
        ctx.set_option('timing', 1)
        for kk, v in opts.items():
            ctx.set_option(kk, v)
        lo = torch.empty(n, dtype=torch.float64, device=dev)
        qo = torch.empty((n, n), dtype=torch.float64, device=dev)
        for rep in range(2):
            ctx.stage_times(reset=True)
            capi.update_decomposition_device(q, lam, kmat, signs.numpy(), lo, qo, ctx=ctx)
            torch.cuda.synchronize()
        st = ctx.stage_times()
        if n <= 8192:
            nrm = float(lo.abs().max())
            r = q @ (lam[:, None] * (q.T @ qo)) + kmat @ (sg[:, None] * (kmat.T @ qo)) - qo * lo[None, :]
            resid = float(r.abs().max()) / nrm
            del r
            orth = float((qo.T @ qo - torch.eye(n, dtype=torch.float64, device=dev)).abs().max())
        else:
            resid = orth = float('nan')
        print(f"cfg{cfg} n={n} {opts}: solve {st['k3_solve']:.1f} ms plan {st['k2_plan']:.1f} cols {st['k4_columns']:.1f} resid {resid:.1e} ortho {orth:.1e}", flush=True)
        ctx.close()
    del q, lam, kmat
    torch.cuda.empty_cache()
