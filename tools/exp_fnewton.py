"""Stage times with and without the f-Newton phase (dev tool)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
dev = torch.device('cuda', 0)
for cfg, n in [(4, 32768), (2, 16384), (1, 16384)]:
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    lo = torch.empty(n, dtype=torch.float64, device=dev)
    qo = torch.empty((n, n), dtype=torch.float64, device=dev)
    for fn in (1, 0):
        ctx = capi.Context(0)
        ctx.set_option('timing', 1)
        ctx.set_option('fnewton', fn)
        for rep in range(2):
            ctx.stage_times(reset=True)
            capi.update_decomposition_device(q, lam, kmat, signs.numpy(), lo, qo, ctx=ctx)
            torch.cuda.synchronize()
        st = ctx.stage_times(); s2 = ctx.stats()
        print(f"cfg{cfg} n={n} fnewton={fn}: plan {st['k2_plan']:.1f} solve {st['k3_solve']:.1f} ms evals/root {s2['evals']/s2['roots']:.2f}", flush=True)
        ctx.close()
    del q, qo; torch.cuda.empty_cache()
