import sys, time; sys.path.insert(0,'.')
import torch, numpy as np
from paper_1706_00773_b200 import capi
from paper_1706_00773_b200.instances import make_instance
import oracle.port as port
dev = torch.device("cuda", 0)
for cfg, n in [(2, 2048), (2, 4096)]:
    q, lam, kmat, s = make_instance(cfg, n=n)
    res = capi.update_decomposition(q, lam, kmat, s, 1e-12)
    t = time.time(); lo, qo, info = port.update(q, lam, kmat, s); t = time.time() - t
    for name, Q in (("gpu", res.q), ("oracle", qo)):
        Qt = torch.from_numpy(Q).to(dev)
        g = Qt.T @ Qt - torch.eye(n, dtype=torch.float64, device=dev)
        i, j = divmod(int(g.abs().argmax()), n)
        X = torch.from_numpy(q).to(dev).T @ Qt
        gx = (X.T @ X - torch.eye(n, dtype=torch.float64, device=dev)).abs().max().item()
        print(f"cfg{cfg} n={n} {name}: ortho {g.abs().max().item():.2e} at ({i},{j}) in-basis {gx:.2e}", flush=True)
    print("  dQ gpu-oracle", np.abs(res.q - qo).max(), "oracle time", t, flush=True)
