"""K3 time and evaluation counts vs the presolve's stopping tolerance (dev tool)."""
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_1706_00773_b200 import capi  # noqa: E402
from paper_1706_00773_b200.instances import make_instance_torch  # noqa: E402

dev = torch.device('cuda', 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q, lam, kmat, signs = make_instance_torch(4, n=n, device=dev)
ref = None
for rel in [float(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1e-12", "1e-10", "1e-8", "1e-6"])]:
    ctx = capi.Context(0)
    ctx.set_option("timing", 1)
    ctx.set_option("fpre_rel", rel)
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
    print(f"fpre_rel={rel:g} k3={st['k3_solve'] / st['calls']:.2f} ms S-evals={ctx.stats()['evals']:.0f} "
          f"f-evals={ctx.presolve_profile()['evals']:.0f} max|dlam|/|lam|={dl:.1e}", flush=True)
    ctx.close()
