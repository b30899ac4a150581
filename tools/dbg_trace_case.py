"""Solver iterate traces of one stress case, with and without the f presolve
(dev tool). Usage: python tools/dbg_trace_case.py seed [root ...]"""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from test_stress import _case
from oracle import port
from paper_1706_00773_b200 import capi
np.set_printoptions(precision=17, linewidth=200)
seed = int(sys.argv[1])
q, lam, kmat, signs, kind = _case(1000 + seed)
n = len(lam)
lo_ref, _, _ = port.update(q, lam, kmat, signs, vectors=False)
roots = [int(a) for a in sys.argv[2:]] or list(range(min(n, 4)))
print('kind', kind, 'n', n, 'k', kmat.shape[1], 'signs', signs)
for fp in (0, 1):
    for j in roots:
        ctx = capi.Context(0)
        ctx.set_option('fpre', fp)
        ctx.set_option('trace_root', j)
        res = capi.update_decomposition(q, lam, kmat, signs, 1e-12, ctx=ctx)
        tr = ctx.solver_trace()
        print(f"fpre={fp} root {j}: lam diff vs oracle {np.abs(res.lam - lo_ref).max():.3e}")
        for row in tr:
            print(f"  {int(row[0]):3d} {int(row[1])} {int(row[2]):4d} {row[3]: .16e} {row[4]: .6e} {row[5]: .6e} "
                  f"{row[6]: .4e} {row[7]: .4e} {row[8]: .4e} {row[9]: .4e} {row[10]: .4e} o={int(row[11])}")
        ctx.close()
