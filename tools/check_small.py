"""Quick GPU-vs-oracle check over small instances of every config (dev tool)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle.port as port  # noqa: E402
from paper_1706_00773_b200 import capi  # noqa: E402
from paper_1706_00773_b200.instances import make_instance  # noqa: E402


def check(cfg, n, seed=None, run_rel=None):
    q, lam, kmat, signs = make_instance(cfg, n=n, seed=seed)
    ctx = capi.default_context()
    if run_rel:
        ctx.set_option("run_rel", run_rel)
    t = time.time()
    res = capi.update_decomposition(q, lam, kmat, signs, 1e-12)
    tg = time.time() - t
    st = ctx.stats()
    lo, qo, info = port.update(q, lam, kmat, signs, run_rel=run_rel or port.EXACT_RUN_REL)
    a = q @ np.diag(lam) @ q.T + kmat @ np.diag(signs.astype(float)) @ kmat.T
    a = 0.5 * (a + a.T)
    ev = np.linalg.eigvalsh(a)
    nrm = float(np.abs(ev).max())
    print(f"cfg{cfg} n={n}: dlam(gpu-oracle)={np.abs(res.lam-lo).max()/nrm:.2e} "
          f"dlam(gpu-lapack)={np.abs(res.lam-ev).max()/nrm:.2e} "
          f"resid={np.abs(a@res.q-res.q*res.lam[None,:]).max()/nrm:.2e} "
          f"ortho={np.abs(res.q.T@res.q-np.eye(n)).max():.2e} "
          f"dQ={np.abs(res.q-qo).max():.2e} t={tg:.2f}s stats={st} oracle={info}", flush=True)


if __name__ == "__main__":
    check(0, 64)
    check(0, 512)
    check(1, 512)
    check(2, 512)
    check(3, 512)
    check(4, 512)
    check(4, 1024)
