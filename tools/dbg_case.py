"""Compare GPU and oracle on one stress case column by column (dev tool)."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from test_stress import _case
from oracle import port
from paper_1706_00773_b200 import capi
np.set_printoptions(precision=4, linewidth=200)
seed = int(sys.argv[1])
q, lam, kmat, signs, kind = _case(1000 + seed)
n = len(lam)
ctx = capi.Context(0)
res = capi.update_decomposition(q, lam, kmat, signs, 1e-12, ctx=ctx)
st = ctx.stats()
lo, qo, info = port.update(q, lam, kmat, signs)
a = (q * lam) @ q.T + (kmat * signs) @ kmat.T
nrm = np.abs(np.linalg.eigvalsh(0.5 * (a + a.T))).max()
G = res.q.T @ res.q - np.eye(n)
bad = np.nonzero(np.abs(G).max(axis=0) > 1e-9)[0]
print('gpu stats', st, 'oracle info', info)
print('bad cols', bad[:20])
for c in bad[:6]:
    x = q.T @ res.q[:, c]; xo = q.T @ qo[:, c]
    top = np.argsort(-np.abs(x))[:4]
    print(c, 'val gpu', res.lam[c], 'orc', lo[c], 'top', top, x[top], 'orc', xo[top])
    near = np.nonzero(np.abs(lam - res.lam[c]) < 1e-9 * nrm)[0]
    print('   poles near', near, lam[near] - res.lam[c])
