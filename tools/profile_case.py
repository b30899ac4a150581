"""One device update of a config-4-shaped instance (for ncu captures)."""
import argparse
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_00773_b200 import capi  # noqa: E402
from paper_1706_00773_b200.instances import CONFIGS, make_instance_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
dev = torch.device("cuda", 0)
q, lam, kmat, signs = make_instance_torch(a.cfg, n=a.n, device=dev)
ctx = capi.Context(0)
ctx.set_option("timing", 1)
lo = torch.empty(a.n, dtype=torch.float64, device=dev)
qo = torch.empty((a.n, a.n), dtype=torch.float64, device=dev)
for r in range(a.reps):
    if r == 1:  # the first call pays the one-time setup (workspaces, attributes)
        torch.cuda.synchronize()
        ctx.stage_times(reset=True)
    capi.update_decomposition_device(q, lam, kmat, signs.numpy(), lo, qo, ctx=ctx)
torch.cuda.synchronize()
st = ctx.stage_times()
print({k: (v / max(1, st["calls"]) if k != "calls" else v) for k, v in st.items()}, ctx.stats())
print("solver_profile", ctx.solver_profile())
print("presolve_profile", ctx.presolve_profile())
