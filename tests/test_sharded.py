"""The multi-GPU driver (paper_1706_00773_b200/sharded.py) on CPU: world_size 2
over gloo, with a numpy/oracle stand-in for the device stages, must reproduce
the single-process result (same eigenvalues, same column blocks). This covers
the partitioning, the two all-gathers and the column-block assembly that the
NCCL run uses; the CUDA stages themselves are covered by
tests/test_gpu.py::test_staged_path_equals_one_shot."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port


class CpuBackend:
    """Oracle-backed stand-in for CudaBackend (tests only). Records are
    (value, origin, delta) rows; no deflation (generic instances)."""

    def __init__(self, n, k, signs):
        self.n, self.k = n, k
        self.signs = np.asarray(signs, np.int32)
        self.kp = k
        self.width = 3

    def project(self, q, kmat, lo, hi, u_out):
        u_out[: hi - lo] = torch.from_numpy(q.numpy()[:, lo:hi].T @ kmat.numpy())

    def plan(self, lam, u_full):
        self.lam = lam.numpy().copy()
        self.u = u_full.numpy()[:, : self.k].copy()
        return self.n

    def plan_groups(self, lam, u_full):
        self.plan(lam, u_full)
        self.alpha_full = port.secular_weights(self.lam, self.u, self.signs)
        return self.n  # generic instances: every pole its own group

    def plan_weights(self, g0, g1, alpha_out):
        alpha_out[: g1 - g0] = torch.from_numpy(self.alpha_full[g0:g1].copy())

    def plan_finish(self, alpha_all):
        # the gathered slices must reassemble the weights of every group
        assert np.array_equal(alpha_all.numpy(), self.alpha_full)
        return self.n

    def solve(self, j0, j1, rec_out):
        roots, orig, dl, _ = port.solve_roots(self.lam, self.u, self.signs, j0, j1)
        rec_out[: j1 - j0, 0] = torch.from_numpy(roots)
        rec_out[: j1 - j0, 1] = torch.from_numpy(orig.astype(np.float64))
        rec_out[: j1 - j0, 2] = torch.from_numpy(dl)

    def finish(self, q, rec_all, c0, c1, lam_out, q_out):
        rec = rec_all.numpy()
        lam_out[:] = torch.from_numpy(rec[:, 0].copy())
        d, u, J = self.lam, self.u, self.signs.astype(float)
        cols = []
        for j in range(c0, c1):
            o, dl = int(rec[j, 1]), rec[j, 2]
            diff = (d - d[o]) - dl
            s = (u / diff[:, None]).T @ u + np.diag(J)
            w, v = np.linalg.eigh(s)
            y = v[:, np.argmin(np.abs(w))]
            x = (u @ y) / diff
            cols.append(x / np.linalg.norm(x))
        qb = q.numpy() @ np.stack(cols, axis=1)
        for c in range(qb.shape[1]):  # eigvec.cpp:340-347
            i = int(np.argmax(np.abs(qb[:, c])))
            if qb[i, c] < 0:
                qb[:, c] = -qb[:, c]
        q_out[:, : c1 - c0] = torch.from_numpy(qb)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port_, inst, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1706_00773_b200.sharded import ShardedUpdate

    q, lam, kmat = (torch.from_numpy(x) for x in inst[:3])
    signs = inst[3]
    n, k = kmat.shape
    be = CpuBackend(n, k, signs)
    sh = ShardedUpdate(be, n, k, signs, rank, world, torch.device("cpu"))
    lam_out = torch.empty(n, dtype=torch.float64)
    q_out = sh.alloc_output()
    sh.run(q, lam, kmat, lam_out, q_out)
    np.savez(f"{out_path}_{rank}.npz", lam=lam_out.numpy(), q=q_out.numpy()[:, : sh.ncols_local],
             c0=sh.c0, c1=sh.c1)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_driver_matches_single_process(tmp_path, world):
    from paper_1706_00773_b200.instances import make_instance

    q, lam, kmat, signs = make_instance(4, n=96, seed=5)
    out = str(tmp_path / "res")
    mp.spawn(_rank, args=(world, _free_port(), (q, lam, kmat, signs), out), nprocs=world, join=True)
    lo, qo, _ = port.update(q, lam, kmat, signs)
    n = len(lam)
    full = np.zeros((n, n))
    for r in range(world):
        z = np.load(f"{out}_{r}.npz")
        # every rank holds all eigenvalues (U here comes from numpy, not the
        # reference loop order, hence ulp-level differences)
        assert np.abs(z["lam"] - lo).max() <= 1e-13 * np.abs(lo).max()
        full[:, int(z["c0"]): int(z["c1"])] = z["q"]
    assert np.abs(full - qo).max() <= 1e-10
    assert np.abs(full.T @ full - np.eye(n)).max() <= 1e-10


def test_split_covers_range():
    from paper_1706_00773_b200.sharded import split

    for n in (0, 1, 7, 96, 1001):
        for world in (1, 2, 3, 8):
            parts = [split(n, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b, c), (a2, _, _) in zip(parts, parts[1:]):
                assert b == a2 and b - a <= c
