"""Iterates of a few roots of the config-4 solve, and the distribution of S evaluations per
root (dev tool). usage: exp_trace.py n root root ..."""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_00773_b200 import capi  # noqa: E402
from paper_1706_00773_b200.instances import make_instance_torch  # noqa: E402

dev = torch.device('cuda', 0)
n = int(sys.argv[1])
q, lam, kmat, signs = make_instance_torch(4, n=n, device=dev)
qn, ln, kn = q.cpu().numpy(), lam.cpu().numpy(), kmat.cpu().numpy()
for j in [int(x) for x in sys.argv[2:]]:
    ctx = capi.Context(0)
    ctx.set_option("trace_root", j)
    lo = torch.empty(n, dtype=torch.float64, device=dev)
    qo = torch.empty((n, n), dtype=torch.float64, device=dev)
    capi.update_decomposition_device(q, lam, kmat, signs.numpy(), lo, qo, ctx=ctx)
    torch.cuda.synchronize()
    tr = ctx.solver_trace()
    print(f"root {j}: {len(tr)} evaluations")
    for r in tr:
        print("  it=%d ph=%d fm=%d delta=%.17e lo=%.3e hi=%.3e sigma=%.3e g=%.3e step=%.3e" %
              (r[0], r[1], r[2], r[3], r[4], r[5], r[8], r[9], r[10]))
    ctx.close()
