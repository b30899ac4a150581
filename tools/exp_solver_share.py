"""Where the solver kernel's time goes (dev tool): SM cycles of slot refills,
pole passes, cluster reductions and per-slot steps, per case and root share."""
import os
import sys
sys.path.insert(0, '.')
import torch
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
from paper_1706_00773_b200.sharded import CudaBackend, split
dev = torch.device('cuda', 0)
for cfg, n in [(4, 32768)] + ([(4, 16384), (2, 16384), (1, 16384)] if os.environ.get('EXP_ALL') else []):
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    ctx = capi.Context(0)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    for kv in os.environ.get("EIGMOD_OPTS", "").split(","):
        if kv:
            kk, vv = kv.split("=")
            ctx.set_option(kk, float(vv))
    be = CudaBackend(ctx, n, kmat.shape[1], signs.numpy())
    u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
    be.project(q, kmat, 0, n, u)
    nred = be.plan(lam, u)
    for world, r in ((1, 0), (8, 0), (8, 3), (8, 4), (8, 7)):
        j0, j1, _ = split(nred, world, r)
        rec = torch.zeros((j1 - j0, be.width), dtype=torch.float64, device=dev)
        for _ in range(2):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a.record(); be.solve(j0, j1, rec); b.record(); torch.cuda.synchronize()
        pr = ctx.solver_profile()
        sh = pr['share']
        print(f"cfg{cfg} n={n} roots={j1 - j0}: {a.elapsed_time(b):7.2f} ms evals/root "
              f"{float(rec[:, 4].sum()) / (j1 - j0):.2f} util {pr['slot_util']:.3f} share refill "
              f"{sh['refill']:.3f} pass {sh['pass']:.3f} reduce {sh['reduce']:.3f} step {sh['step']:.3f} "
              f"(load {sh['step_load']:.3f} factor {sh['step_factor']:.3f} solve {sh['step_solve']:.3f})", flush=True)
        cyc = pr['cycles']
        tot = sum(cyc.values())
        print(f"    batches {pr['batches']:.0f} passes/batch {pr['passes'] / max(1, pr['batches']):.1f} "
              f"us/pass {tot / max(1, pr['passes']) / 1965.0:.1f}", flush=True)
    ctx.close()
    del q; torch.cuda.empty_cache()
