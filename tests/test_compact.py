"""Compact back-transform (capi.cu finish_compact): plans with decoupled
columns multiply only the reduced rows, Q'[:, roots] = Q~_red X_red, and copy
or rotate Q's columns for the decoupled ones. Checked against the dense
back-transform (option compact_gemm 0, the reference's n x n product,
proj/src/eigvec.cpp:285-339), the north-star tolerances, the host-buffer
path and the staged (column-partitioned) path. Every test needs a B200."""
import numpy as np
import pytest

from northstar import residual

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api(ctx):
    from paper_1706_00773_b200 import capi

    return capi


def _aprime(q, lam, kmat, signs):
    a = q @ np.diag(lam) @ q.T + kmat @ np.diag(np.asarray(signs, float)) @ kmat.T
    return 0.5 * (a + a.T)


def _signed_diff(a, b):
    """max over columns of min(|a - b|, |a + b|) and the number of columns
    whose sign differs."""
    dp = np.abs(a - b).max(axis=0)
    dm = np.abs(a + b).max(axis=0)
    return float(np.minimum(dp, dm).max()), int((dm < dp).sum())


def _stress(n, seed):
    """Runs of equal and near-equal poles (compressed groups), unchanged rows
    (zero coupling) and a rank-4 indefinite update."""
    rng = np.random.default_rng(seed)
    lam = np.sort(rng.uniform(-1, 1, n))
    for c in rng.choice(n - 40, 12, replace=False):
        m = int(rng.integers(3, 30))
        lam[c:c + m] = lam[c] + 1e-13 * np.arange(m)
    lam = np.sort(lam)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    kmat = rng.standard_normal((n, 4)) / np.sqrt(n)
    u = q.T @ kmat
    dead = rng.choice(n, n // 10, replace=False)
    u[dead] *= 1e-15
    kmat = q @ u
    return q, lam, kmat, np.array([1, -1, 1, -1], np.int32)


CASES = [("cfg3_n2048_s0", 3, 2048, 0), ("cfg3_n3000_s4", 3, 3000, 4),
         ("cfg3_n4096_s1", 3, 4096, 1), ("stress_n1500", None, 1500, 7),
         ("stress_n2500", None, 2500, 11)]


def _instance(cfg, n, seed):
    from paper_1706_00773_b200.instances import make_instance

    if cfg is None:
        return _stress(n, seed)
    return make_instance(cfg, n=n, seed=seed)


@pytest.mark.parametrize("name,cfg,n,seed", CASES, ids=[c[0] for c in CASES])
def test_compact_matches_dense_back_transform(api, name, cfg, n, seed):
    q, lam, kmat, s = _instance(cfg, n, seed)
    c1 = api.Context(0)
    c0 = api.Context(0)
    c0.set_option("compact_gemm", 0)
    try:
        r1 = api.update_decomposition(q, lam, kmat, s, 1e-12, ctx=c1)
        st = c1.stats()
        r0 = api.update_decomposition(q, lam, kmat, s, 1e-12, ctx=c0)
    finally:
        c0.close()
        c1.close()
    assert st["decoupled"] >= 64, st  # the compact path ran
    assert np.array_equal(r1.lam, r0.lam)  # eigenvalues do not depend on K5
    d, flips = _signed_diff(r1.q, r0.q)
    assert d <= 1e-12, d
    assert flips == 0
    a = _aprime(q, lam, kmat, s)
    nrm = float(np.abs(r1.lam).max())
    assert residual(a, r1.q, r1.lam, nrm) <= 1e-10
    assert float(np.abs(r1.q.T @ r1.q - np.eye(n)).max()) <= 1e-9


def test_compact_host_path_equals_device_path(api):
    """Host buffers (GEMM in column blocks, D2H overlapped) give the same
    bits as the all-device call."""
    import torch

    q, lam, kmat, s = _instance(3, 4096, 2)
    n = len(lam)
    ctx = api.Context(0)
    try:
        rh = api.update_decomposition(q, lam, kmat, s, 1e-12, ctx=ctx)
        assert ctx.stats()["decoupled"] >= 64
        dev = torch.device("cuda", 0)
        tq, tl, tk = (torch.from_numpy(x).to(dev) for x in (q, lam, kmat))
        lo = torch.empty(n, dtype=torch.float64, device=dev)
        qo = torch.empty((n, n), dtype=torch.float64, device=dev)
        api.update_decomposition_device(tq, tl, tk, s, lo, qo, ctx=ctx)
        torch.cuda.synchronize()
    finally:
        ctx.close()
    assert np.array_equal(rh.lam, lo.cpu().numpy())
    assert np.array_equal(rh.q, qo.cpu().numpy())


@pytest.mark.parametrize("world", [2, 3])
def test_compact_staged_columns_equal_one_shot(api, world):
    """Column blocks [c0, c1) of the staged (multi-GPU) path, finished one
    after the other on one GPU, reassemble the one-shot Q' bit for bit (each
    block gathers its own decoupled columns and multiplies its own roots)."""
    import torch

    from paper_1706_00773_b200.sharded import CudaBackend, split

    q, lam, kmat, s = _instance(3, 2600, 3)
    dev = torch.device("cuda", 0)
    tq, tl, tk = (torch.from_numpy(x).to(dev) for x in (q, lam, kmat))
    n, k = kmat.shape
    ctx = api.Context(0)
    try:
        ctx.set_option("fuse_alpha", 0)
        lo1 = torch.empty(n, dtype=torch.float64, device=dev)
        qo1 = torch.empty((n, n), dtype=torch.float64, device=dev)
        api.update_decomposition_device(tq, tl, tk, s, lo1, qo1, ctx=ctx)
        assert ctx.stats()["decoupled"] >= 64
        ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
        be = CudaBackend(ctx, n, k, s)
        u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
        be.project(tq, tk, 0, n, u)
        ng = be.plan_groups(tl, u)
        alpha = torch.zeros(ng, dtype=torch.float64, device=dev)
        be.plan_weights(0, ng, alpha)
        nred = be.plan_finish(alpha)
        rec = torch.zeros((nred, be.width), dtype=torch.float64, device=dev)
        be.solve(0, nred, rec)
        lo2 = torch.empty(n, dtype=torch.float64, device=dev)
        qo2 = torch.empty((n, n), dtype=torch.float64, device=dev)
        for r in range(world):
            c0, c1, _ = split(n, world, r)
            blk = torch.empty((n, c1 - c0), dtype=torch.float64, device=dev)
            be.finish(tq, rec, c0, c1, lo2, blk)
            qo2[:, c0:c1] = blk
        torch.cuda.synchronize()
    finally:
        ctx.close()
    assert torch.equal(lo1, lo2)
    assert torch.equal(qo1, qo2)
