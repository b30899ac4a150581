import sys, torch
sys.path.insert(0, '.')
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance_torch
dev = torch.device('cuda', 0)
for cfg, n in [(4, 32768), (3, 16384), (2, 8192)]:
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    res = {}
    for comp in (0, 1):
        ctx = capi.Context(0)
        ctx.set_option("timing", 1)
        ctx.set_option("compact", comp)
        lo = torch.empty(n, dtype=torch.float64, device=dev)
        qo = torch.empty((n, n), dtype=torch.float64, device=dev)
        for r in range(3):
            if r == 1:
                torch.cuda.synchronize(); ctx.stage_times(reset=True)
            capi.update_decomposition_device(q, lam, kmat, signs.numpy(), lo, qo, ctx=ctx)
        torch.cuda.synchronize()
        st = ctx.stage_times()
        res[comp] = (lo.clone(), qo[:, :64].clone())
        print(cfg, n, 'compact', comp, 'k3 %.2f' % (st['k3_solve'] / st['calls']), 'slot_util %.3f' % ctx.solver_profile()['slot_util'], flush=True)
        ctx.close()
    print('  identical:', torch.equal(res[0][0], res[1][0]), torch.equal(res[0][1], res[1][1]), flush=True)
    del q, lo, qo, res
    torch.cuda.empty_cache()
