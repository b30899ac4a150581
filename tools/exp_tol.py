import sys; sys.path.insert(0,'.')
import torch, numpy as np
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
dev = torch.device("cuda", 0)
for cfg, n in [(2, 8192), (4, 8192), (0, 512), (1, 4096)]:
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    sg = signs.to(dev, torch.float64)
    for tol in [2.0, 0.5, 0.1]:
        ctx = capi.Context(0)
        ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
        ctx.set_option("step_tol", tol)
        lo = torch.empty(n, dtype=torch.float64, device=dev); qo = torch.empty((n, n), dtype=torch.float64, device=dev)
        capi.update_decomposition_device(q, lam, kmat, signs.numpy(), lo, qo, ctx=ctx)
        torch.cuda.synchronize()
        st = ctx.stats()
        nrm = float(lo.abs().max())
        r = q @ (lam[:, None] * (q.T @ qo)) + kmat @ (sg[:, None] * (kmat.T @ qo)) - qo * lo[None, :]
        resid = float(r.abs().max()) / nrm; del r
        g = qo.T @ qo - torch.eye(n, dtype=torch.float64, device=dev)
        orth = float(g.abs().max())
        i, j = divmod(int(g.abs().argmax()), n)
        print(f"cfg{cfg} n={n} tol={tol}: resid {resid:.2e} ortho {orth:.2e} at ({i},{j}) lam {lo[i].item():.6f} {lo[j].item():.6f} evals/root {st['evals']/st['roots']:.2f} max {st['max_evals']}", flush=True)
        ctx.close()
