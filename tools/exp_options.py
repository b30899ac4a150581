"""K3 time, evaluation counts and accuracy for solver option sets (dev tool).
usage: exp_options.py n cfg 'key=v,key=v' 'key=v' ..."""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_00773_b200 import capi  # noqa: E402
from paper_1706_00773_b200.instances import make_instance_torch  # noqa: E402

dev = torch.device('cuda', 0)
n, cfg = int(sys.argv[1]), int(sys.argv[2])
q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
ref = None
for spec in sys.argv[3:]:
    opts = dict(kv.split('=') for kv in spec.split(',') if kv)
    ctx = capi.Context(0)
    ctx.set_option("timing", 1)
    for kk, v in opts.items():
        ctx.set_option(kk, float(v))
    lo = torch.empty(n, dtype=torch.float64, device=dev)
    qo = torch.empty((n, n), dtype=torch.float64, device=dev)
    for r in range(3):
        if r == 1:
            torch.cuda.synchronize()
            ctx.stage_times(reset=True)
        capi.update_decomposition_device(q, lam, kmat, signs.numpy(), lo, qo, ctx=ctx)
    torch.cuda.synchronize()
    st = ctx.stage_times()
    if ref is None:
        ref = lo.clone()
    dl = float((lo - ref).abs().max() / ref.abs().max())
    # orthogonality of a column sample against all columns: ||Q'^T Q'_S - I_S||_max
    idx = torch.arange(0, n, max(1, n // 512), device=dev)
    g = qo.T @ qo[:, idx]
    g[idx, torch.arange(len(idx), device=dev)] -= 1.0
    orth = float(g.abs().max())
    print(f"{spec or 'default'}: k3={st['k3_solve'] / st['calls']:.2f} ms S-evals={ctx.stats()['evals']:.0f} "
          f"f-evals={ctx.presolve_profile()['evals']:.0f} max|dlam|/|lam|={dl:.1e} ortho(sample)={orth:.1e}",
          flush=True)
    ctx.close()
