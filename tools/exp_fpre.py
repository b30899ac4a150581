"""Solver stage with and without the scalar f presolve (dev tool): time,
S evaluations per root, max evaluations, and the eigenvalue / orthogonality
agreement of the two variants."""
import os
import sys
sys.path.insert(0, '.')
import torch
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
dev = torch.device('cuda', 0)
cases = [(4, 32768), (2, 16384), (1, 16384), (3, 8192), (4, 4096)]
for cfg, n in cases:
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    lo = torch.empty(n, dtype=torch.float64, device=dev)
    qo = torch.empty((n, n), dtype=torch.float64, device=dev)
    res = {}
    for fp in (0, 1):
        ctx = capi.Context(0)
        ctx.set_option('timing', 1)
        ctx.set_option('fpre', fp)
        if 'EIGMOD_FPRE_ITERS' in os.environ:
            ctx.set_option('fpre_iters', float(os.environ['EIGMOD_FPRE_ITERS']))
        for rep in range(2):
            ctx.stage_times(reset=True)
            capi.update_decomposition_device(q, lam, kmat, signs.numpy(), lo, qo, ctx=ctx)
            torch.cuda.synchronize()
        st = ctx.stage_times(); s2 = ctx.stats()
        pp = ctx.presolve_profile()
        if fp:
            from torch.profiler import profile, ProfilerActivity
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                capi.update_decomposition_device(q, lam, kmat, signs.numpy(), lo, qo, ctx=ctx)
                torch.cuda.synchronize()
            for ev in prof.key_averages():
                if 'fpresolve' in ev.key or 'solve_roots' in ev.key or 'count_sweep' in ev.key:
                    print(f"     {ev.key[:60]}: {ev.device_time_total / 1000:.2f} ms", flush=True)
            print(f"     presolve: {pp}", flush=True)
        import ctypes, numpy as np
        ob = np.zeros(1)
        ctx.check(ctx._l.eigmod_b200_ortho_error_device(ctx.h, capi._ptr(qo), n, n,
                                                        ob.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        orth = float(ob[0])
        res[fp] = lo.clone()
        print(f"cfg{cfg} n={n} fpre={fp}: solve {st['k3_solve']:.1f} ms evals/root "
              f"{s2['evals']/s2['roots']:.2f} max {s2['max_evals']:.0f} ortho {orth:.2e}", flush=True)
        ctx.close()
    d = (res[0] - res[1]).abs().max().item() / res[0].abs().max().item()
    print(f"   max |lam(fpre=0) - lam(fpre=1)| / |lam| = {d:.2e}", flush=True)
    del q, qo; torch.cuda.empty_cache()
