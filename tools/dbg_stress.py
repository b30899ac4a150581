"""Run the stress cases and print failures with details (dev tool)."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from test_stress import _case
from paper_1706_00773_b200 import capi
seeds = [int(a) for a in sys.argv[1:]] or list(range(60))
for seed in seeds:
    q, lam, kmat, signs, kind = _case(1000 + seed)
    n = len(lam)
    try:
        ctx = capi.default_context()
        import os
        for kv in os.environ.get("EIGMOD_OPTS", "").split(","):
            if kv:
                kk, vv = kv.split("=")
                ctx.set_option(kk, float(vv))
        res = capi.update_decomposition(q, lam, kmat, signs, 1e-12, ctx=ctx)
    except Exception as e:
        print(seed, kind, n, kmat.shape[1], 'EXC', type(e).__name__, getattr(e, 'stage', ''), str(e)[:200])
        continue
    a = (q * lam) @ q.T + (kmat * signs) @ kmat.T
    a = 0.5 * (a + a.T)
    ev = np.linalg.eigvalsh(a)
    nrm = np.abs(ev).max()
    e = np.abs(res.lam - ev).max() / nrm
    r = np.abs(a @ res.q - res.q * res.lam).max() / nrm
    o = np.abs(res.q.T @ res.q - np.eye(n)).max()
    if not (e <= 1e-10 and r <= 1e-10 and o <= 1e-9):
        print(seed, kind, n, kmat.shape[1], 'eig', e, 'res', r, 'orth', o)
