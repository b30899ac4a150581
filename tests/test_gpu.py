"""Parity of the sm_100a path (through the C ABI) with the oracle, the
reference fixtures and LAPACK. Every test here needs a B200."""
import math
import os

import numpy as np
import pytest

from northstar import residual
from oracle import port

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SEEDED = np.load(os.path.join(HERE, "golden", "ref_seeded.npz"))
CASES = np.load(os.path.join(HERE, "golden", "ref_cases.npz"))


def _cases(npz):
    keys = sorted({k.split("__")[0] for k in npz.files})
    return [(k, {f.split("__")[1]: npz[f] for f in npz.files if f.split("__")[0] == k}) for k in keys]


SEEDED_CASES = _cases(SEEDED)
RANDOM_CASES = _cases(CASES)
IDS = [n for n, _ in SEEDED_CASES]


def _aprime(q, lam, kmat, signs):
    a = q @ np.diag(lam) @ q.T + kmat @ np.diag(np.asarray(signs, float)) @ kmat.T
    return 0.5 * (a + a.T)


@pytest.fixture(scope="module")
def api(ctx):
    from paper_1706_00773_b200 import capi

    return capi


# ----------------------------------------------------------- stages
@pytest.mark.parametrize("name,c", SEEDED_CASES, ids=IDS)
def test_transform_update(api, ctx, name, c):
    u = api.transform_update(c["q"], c["kmat"], ctx=ctx)
    scale = max(1.0, float(np.abs(c["u"]).max()))
    assert np.abs(u - c["u"]).max() <= 1e-13 * scale


@pytest.mark.parametrize("n,k", [(2, 1), (8, 3), (64, 16), (130, 2), (256, 5), (512, 32),
                                 (1000, 16), (1026, 8), (333, 4), (4096, 16)])
def test_projection_dmma_vs_numpy(api, ctx, n, k):
    """K1 on the DMMA path (even n) and the DFMA path (odd n, misaligned
    slices): U = Q^T K to FP64 rounding of the products, every padded rank,
    partial column blocks, partial row stages, multi-GPU column slices."""
    import torch

    rng = np.random.default_rng(n * 100 + k)
    q = rng.standard_normal((n, n))
    kmat = rng.standard_normal((n, k))
    want = q.T @ kmat
    scale = np.abs(q).T @ np.abs(kmat)
    u = api.transform_update(q, kmat, ctx=ctx)
    assert np.all(np.abs(u - want) <= 1e-14 * n * scale + 1e-300)
    from paper_1706_00773_b200.sharded import CudaBackend, split

    dev = torch.device("cuda", 0)
    tq, tk = torch.from_numpy(q).to(dev), torch.from_numpy(kmat).to(dev)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    be = CudaBackend(ctx, n, k, np.ones(k, np.int32))
    for world in (2, 3):
        for r in range(world):
            lo, hi, ch = split(n, world, r)
            part = torch.zeros((max(ch, 1), be.kp), dtype=torch.float64, device=dev)
            if hi > lo:
                be.project(tq, tk, lo, hi, part)
            torch.cuda.synchronize()
            got = part[: hi - lo, :k].cpu().numpy()
            assert np.all(np.abs(got - want[lo:hi]) <= 1e-14 * n * scale[lo:hi] + 1e-300)
    ctx.set_stream(None)


@pytest.mark.parametrize("name,c", SEEDED_CASES, ids=IDS)
def test_deflation_record_matches_reference(api, ctx, name, c):
    d = api.deflate_problem(c["lam"], c["u"], c["signs"], ctx=ctx)
    # decisions depend on input bits only (runs, row mass); alpha within rounding
    assert np.array_equal(d.pole_origin, c["dp_pole_origin"])
    assert np.array_equal(d.unchanged, c["dp_unchanged"])
    assert np.array_equal(d.collided, c["dp_collided"])
    assert np.array_equal(d.poles, c["dp_poles"])
    w = c["dp_weights"]
    if len(w):
        scale = np.abs(w) + np.abs(w).sum() / len(w)
        # the reference's own alpha is unstable on merged clusters (|alpha| ~ 1e64)
        tau = 1e-9 if not name.startswith("c3") else 1e-6
        assert np.all(np.abs(d.weights - w) <= tau * scale)


def test_secular_weights_vs_oracle(api, ctx):
    rng = np.random.default_rng(9)
    for k in (1, 2, 3, 4, 5, 8, 16):
        n = 60
        lam = np.sort(rng.uniform(-2, 2, n))
        u = rng.standard_normal((n, k)) / math.sqrt(n)
        s = np.where(np.arange(k) % 2 == 0, 1, -1)
        a_gpu = api.secular_weights(lam, u, s, ctx=ctx)
        a_ref = port.secular_weights(lam, u, s)
        scale = np.abs(a_ref) + np.abs(a_ref).sum() / n
        assert np.all(np.abs(a_gpu - a_ref) <= 1e-10 * scale), k


# ------------------------------------------------------ eigenpairs
@pytest.mark.parametrize("name,c", SEEDED_CASES, ids=IDS)
def test_update_decomposition_parity(api, ctx, name, c):
    q, lam, kmat, s = c["q"], c["lam"], c["kmat"], c["signs"]
    res = api.update_decomposition(q, lam, kmat, s, float(c["tol"]), ctx=ctx)
    a = _aprime(q, lam, kmat, s)
    ev = np.linalg.eigvalsh(a)
    nrm = float(np.abs(ev).max())
    n = len(lam)
    lo, qo, _ = port.update(q, lam, kmat, s)
    assert np.abs(res.lam - ev).max() <= 1e-10 * nrm          # north-star eigenvalue tol
    assert np.abs(res.lam - lo).max() <= 1e-12 * nrm          # vs the oracle
    assert residual(a, res.q, res.lam, nrm) <= 1e-10            # per-column 2-norm
    assert np.abs(res.q.T @ res.q - np.eye(n)).max() <= 1e-9
    assert np.abs(res.q - qo).max() <= 1e-8                   # same columns, same signs
    if str(c["eig_status"]) == "ok" and np.abs(c["values"] - ev).max() <= 1e-10 * nrm:
        assert np.abs(res.lam - c["values"]).max() <= 1e-10 * nrm
    if str(c["vec_status"]) == "ok":
        assert np.abs(res.q - c["q_out"]).max() <= 1e-5       # reference vectors ~1e-7


@pytest.mark.parametrize("name,c", RANDOM_CASES, ids=[n for n, _ in RANDOM_CASES])
def test_reference_random_instances(api, ctx, name, c):
    # tests/test_rootfind.cpp:163-178 and test_eigvec.cpp:133-183 instances
    res = api.update_decomposition(c["q"], c["lam"], c["kmat"], c["signs"], float(c["tol"]),
                                   ctx=ctx)
    ev = np.linalg.eigvalsh(_aprime(c["q"], c["lam"], c["kmat"], c["signs"]))
    assert np.abs(res.lam - ev).max() <= 1e-12 * max(1.0, float(np.abs(ev).max()))
    if str(c["eig_status"]) == "ok":
        assert np.abs(res.lam - c["values"]).max() <= 1e-9
    if str(c["vec_status"]) == "ok":
        assert np.abs(res.q - c["q_out"]).max() <= 1e-5


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 33, 101, 257, 513])
def test_odd_and_tiny_sizes(api, ctx, n):
    """Odd n reaches the K5 GEMM with an odd inner dimension (padded staging)."""
    from paper_1706_00773_b200.instances import make_instance

    for cfg in (0, 2):
        q, lam, kmat, signs = make_instance(cfg, n=n, seed=n)
        k = min(kmat.shape[1], n)
        kmat, signs = kmat[:, :k], signs[:k]
        res = api.update_decomposition(q, lam, kmat, signs, 1e-12, ctx=ctx)
        a = _aprime(q, lam, kmat, signs)
        ev = np.linalg.eigvalsh(a)
        nrm = max(1.0, float(np.abs(ev).max()))
        assert np.abs(res.lam - ev).max() <= 1e-12 * nrm
        assert residual(a, res.q, res.lam, nrm) <= 1e-12
        assert np.abs(res.q.T @ res.q - np.eye(n)).max() <= 1e-11
        lo, qo, _ = port.update(q, lam, kmat, signs)
        assert np.abs(res.lam - lo).max() <= 1e-12 * nrm
        assert np.abs(res.q - qo).max() <= 1e-8


def test_update_eigenvalues_full_fields(api, ctx):
    name, c = SEEDED_CASES[0]
    up = api.update_eigenvalues_full(c["q"], c["lam"], c["kmat"], c["signs"], 1e-12, ctx=ctx)
    assert np.all(np.diff(up.values) >= 0)
    assert 0 < len(up.roots) <= len(c["lam"]) and np.all(np.diff(up.roots) >= 0)
    assert np.abs(up.u - c["u"]).max() <= 1e-13 * max(1.0, float(np.abs(c["u"]).max()))
    assert np.array_equal(up.problem.pole_origin, c["dp_pole_origin"])


# ---------------------------------------------------------- goldens
R2 = math.sqrt(2.0)


def test_golden_2x2(api, ctx):
    # tests/test_eigvec.cpp:107-123, test_cli.cpp:62-63
    res = api.update_decomposition(np.eye(2), [0.0, 1.0], [[1.0, 0.0], [1.0, 1.0]], [1, 1], 1e-14,
                                   metrics=True, ctx=ctx)
    assert abs(res.lam[0] - 0.58578643762690495) <= 1e-12 * 2
    assert abs(res.lam[1] - 3.4142135623730951) <= 1e-12 * 4
    lam = 2.0 - R2
    nrm = math.sqrt(1.0 + (lam - 1.0) ** 2)
    assert abs(res.q[0, 0] - 1.0 / nrm) <= 1e-12 and abs(res.q[1, 0] - (lam - 1.0) / nrm) <= 1e-12
    assert res.residual_fro <= 1e-10 and res.ortho_err <= 1e-12


def test_golden_k_zero_bit_exact(api, ctx):
    # tests/test_eigvec.cpp:97-105
    rng = np.random.default_rng(77)
    q, _ = np.linalg.qr(rng.standard_normal((8, 8)))
    lam = np.sort(rng.uniform(-1, 1, 8))
    res = api.update_decomposition(q, lam, np.zeros((8, 2)), [1, 1], 1e-12, metrics=True, ctx=ctx)
    assert np.array_equal(res.lam, lam) and np.array_equal(res.q, q)
    assert res.residual_fro == 0.0 or res.residual_fro < 1e-15


def test_golden_unchanged_rows_copy_columns_exactly(api, ctx):
    # rows of U that vanish leave their eigenpairs untouched (secular.cpp:316-325,
    # eigvec.cpp:288-291): the matching columns of Q' are exact copies.
    rng = np.random.default_rng(4)
    n = 12
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.sort(rng.uniform(-1, 1, n))
    u = rng.standard_normal((n, 2))
    u[[2, 7]] = 0.0
    kmat = q @ u
    u2 = q.T @ kmat
    res = api.update_decomposition(q, lam, kmat, [1, -1], 1e-12, ctx=ctx)
    for i in (2, 7):
        if np.abs(u2[i]).max() == 0.0:
            col = int(np.where(res.lam == lam[i])[0][0])
            assert np.array_equal(res.q[:, col], q[:, i])


def test_golden_rank1_collision(api, ctx):
    # tests/test_rootfind.cpp:150-161
    vals = api.update_eigenvalues(np.eye(2), [1.0, 2.0], [[1.0], [0.0]], [1], 1e-14, ctx=ctx)
    assert np.allclose(vals, [2.0, 2.0], rtol=0, atol=2e-12)


def test_golden_collided_vector(api, ctx):
    # tests/test_eigvec.cpp:64-76
    res = api.update_decomposition(np.eye(2), [0.0, 1.0], np.eye(2), [1, 1], 1e-14, ctx=ctx)
    assert np.allclose(res.lam, [1.0, 2.0], atol=1e-14)
    assert np.allclose(np.abs(res.q), np.eye(2), atol=1e-14)


def test_golden_weights_and_deflation(api, ctx):
    # tests/test_secular.cpp:97-126, 273-298
    inv = 1.0 / R2
    assert np.allclose(api.secular_weights([1.0, 2.0], [[inv], [inv]], [1], ctx=ctx), [0.5, 0.5],
                       rtol=1e-13)
    a = api.secular_weights([0.0, 1.0], np.eye(2), [1, 1], ctx=ctx)
    assert abs(a[0] - 2.0) <= 2e-13 and abs(a[1]) <= 1e-15
    assert np.allclose(api.secular_weights([0.0, 1.0], [[1.0, 0.0], [1.0, 1.0]], [1, 1], ctx=ctx),
                       [2.0, 1.0], rtol=1e-13)
    d = api.deflate_problem([0.0, 1.0, 2.0], [[0.0], [0.5], [0.0]], [1], ctx=ctx)
    assert np.allclose(d.poles, [1.0]) and np.allclose(d.weights, [0.25])
    assert list(d.unchanged) == [0, 2] and list(d.pole_origin) == [1]
    d = api.deflate_problem([1.0, 1.0 + 1e-15, 2.0], [[1.0], [2.0], [1.0]], [1], ctx=ctx)
    assert len(d.poles) == 2 and abs(d.weights[0] - 5.0) <= 5e-9 and len(d.unchanged) == 1


def test_error_behaviour(api, ctx):
    # std::invalid_argument (core.cpp:89-97, rootfind.cpp:384) / NumericalError("deflate")
    with pytest.raises(ValueError):
        api.update_decomposition(np.eye(2), [0.0, 1.0], np.eye(2), [1, 2], 1e-12, ctx=ctx)
    with pytest.raises(ValueError):
        api.update_decomposition(np.eye(2), [0.0, 1.0], np.ones((2, 3)), [1, 1, 1], 1e-12, ctx=ctx)
    with pytest.raises(ValueError):
        api.update_decomposition(np.eye(2), [0.0, 1.0], np.eye(2), [1, 1], 0.0, ctx=ctx)
    with pytest.raises(ValueError):
        api.update_decomposition(np.eye(2), [0.0, 1.0], [[np.nan, 0.0], [0.0, 1.0]], [1, 1], 1e-12,
                                 ctx=ctx)
    with pytest.raises(api.NumericalError) as e:
        api.update_decomposition(np.eye(2), [1.0, 0.0], np.eye(2), [1, 1], 1e-12, ctx=ctx)
    assert e.value.stage == "deflate"
    with pytest.raises(ValueError):
        api.secular_weights([1.0, 1.0], [[1.0], [0.0]], [1], ctx=ctx)


def test_deterministic(api, ctx):
    from paper_1706_00773_b200.instances import make_instance

    q, lam, kmat, s = make_instance(4, n=384, seed=21)
    r1 = api.update_decomposition(q, lam, kmat, s, 1e-12, ctx=ctx)
    r2 = api.update_decomposition(q, lam, kmat, s, 1e-12, ctx=ctx)
    assert np.array_equal(r1.lam, r2.lam) and np.array_equal(r1.q, r2.q)


@pytest.mark.parametrize("opts", [{"fpre": 0}, {"fpre": 1, "fpre_min_kp": 1},
                                  {"fpre": 1, "fpre_iters": 2}, {"cluster": 1}, {"cluster": 8},
                                  {"fnewton": 0}, {"sweep_poles": 0},
                                  {"sweep_poles": 0, "pole_split": 0}, {"split_phase_a": 0},
                                  {"sweep": 0}, {"fuse_alpha": 0}, {"fpre_rel": 0},
                                  {"compact": 0}, {"spec_plan": 0}, {"noise_c": 0}])
def test_solver_variants_meet_tolerances(api, opts):
    """The solver's optional phases (scalar f presolve, f-Newton, cluster
    sizes) change only the path to each root: every variant meets the
    north-star tolerances against LAPACK and agrees with the default."""
    from paper_1706_00773_b200.instances import make_instance

    q, lam, kmat, s = make_instance(4, n=640, seed=33)
    base = api.update_decomposition(q, lam, kmat, s, 1e-12, ctx=api.Context(0))
    c = api.Context(0)
    for key, val in opts.items():
        c.set_option(key, float(val))
    r = api.update_decomposition(q, lam, kmat, s, 1e-12, ctx=c)
    a = _aprime(q, lam, kmat, s)
    ev = np.linalg.eigvalsh(a)
    nrm = np.abs(ev).max()
    assert np.abs(r.lam - ev).max() <= 1e-10 * nrm
    assert np.abs(r.lam - base.lam).max() <= 1e-12 * nrm
    assert residual(a, r.q, r.lam, nrm) <= 1e-10
    assert np.abs(r.q.T @ r.q - np.eye(len(lam))).max() <= 1e-9
    prof = c.solver_profile()
    assert prof["passes"] > 0 and 0.0 < prof["slot_util"] <= 1.0
    assert abs(sum(prof["share"][k] for k in ("refill", "pass", "reduce", "step")) - 1.0) < 1e-9
    pre = c.presolve_profile()
    pre_runs = (opts.get("fpre", 1) and opts.get("fpre_min_kp", 16) <= 16
                and opts.get("fnewton", 1) and opts.get("sweep", 1))  # brackets from the counts
    if not pre_runs:
        assert pre["converged"] + pre["unconverged"] == 0
    else:
        assert pre["converged"] + pre["unconverged"] > 0
        assert pre["max_evals"] <= opts.get("fpre_iters", 12)
    c.close()


def test_fused_residues_match_k2(api):
    """The residues the pole-limit count pass computes (one-shot exact mode)
    are the K2 residues of the same simple poles: the f presolve then
    converges to the same starts, evaluation counts agree closely."""
    from paper_1706_00773_b200.instances import make_instance

    for cfg, n in [(4, 2048), (2, 1024), (1, 1024)]:
        q, lam, kmat, s = make_instance(cfg, n=n, seed=5)
        c0, c1 = api.Context(0), api.Context(0)
        c0.set_option("fuse_alpha", 0)
        r0 = api.update_decomposition(q, lam, kmat, s, 1e-12, ctx=c0)
        r1 = api.update_decomposition(q, lam, kmat, s, 1e-12, ctx=c1)
        nrm = np.abs(r0.lam).max()
        assert np.abs(r0.lam - r1.lam).max() <= 1e-13 * nrm
        e0, e1 = c0.stats()["evals"], c1.stats()["evals"]
        assert abs(e0 - e1) <= 0.02 * e0 + 4


def test_unknown_option_is_rejected(api):
    c = api.Context(0)
    with pytest.raises(ValueError):
        c.set_option("no_such_option", 1.0)
    c.close()


# ----------------------------------------------- staged (multi-GPU) path
def test_staged_path_equals_one_shot(api, ctx):
    """The root/column-partitioned data path, run as two virtual ranks on one
    GPU one after the other (no cross-rank waits): same bits as one shot with
    the K2 residues (option fuse_alpha 0; the staged path runs K2 split over
    the ranks), and the default one shot (residues from the count pass)
    within 1e-13 ||A'||."""
    import ctypes as C

    import torch

    from paper_1706_00773_b200.instances import make_instance
    from paper_1706_00773_b200.sharded import CudaBackend, split

    q, lam, kmat, s = make_instance(2, n=700, seed=5)
    dev = torch.device("cuda", 0)
    tq, tl, tk = (torch.from_numpy(x).to(dev) for x in (q, lam, kmat))
    n, k = kmat.shape
    lo1 = torch.empty(n, dtype=torch.float64, device=dev)
    qo1 = torch.empty((n, n), dtype=torch.float64, device=dev)
    lo0 = torch.empty(n, dtype=torch.float64, device=dev)
    qo0 = torch.empty((n, n), dtype=torch.float64, device=dev)
    api.update_decomposition_device(tq, tl, tk, s, lo0, qo0, ctx=ctx)
    ctx.set_option("fuse_alpha", 0)
    try:
        api.update_decomposition_device(tq, tl, tk, s, lo1, qo1, ctx=ctx)
    finally:
        ctx.set_option("fuse_alpha", 1)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    be = CudaBackend(ctx, n, k, s)
    world = 2
    u_all = torch.zeros((split(n, world, 0)[2] * world, be.kp), dtype=torch.float64, device=dev)
    for r in range(world):
        a, b, ch = split(n, world, r)
        part = torch.zeros((ch, be.kp), dtype=torch.float64, device=dev)
        be.project(tq, tk, a, b, part)
        u_all[r * ch: r * ch + (b - a)] = part[: b - a]
    nred = be.plan(tl, u_all[:n])
    # split K2 (plan_groups / plan_weights per rank slice / plan_finish)
    ng = be.plan_groups(tl, u_all[:n])
    parts = []
    for r in range(world):
        g0, g1, gc = split(ng, world, r)
        a_part = torch.zeros(max(gc, 1), dtype=torch.float64, device=dev)
        be.plan_weights(g0, g1, a_part)
        parts.append(a_part[: g1 - g0])
    assert be.plan_finish(torch.cat(parts)) == nred
    recs = []
    for r in range(world):
        j0, j1, jc = split(nred, world, r)
        part = torch.zeros((jc, be.width), dtype=torch.float64, device=dev)
        be.solve(j0, j1, part)
        recs.append(part[: j1 - j0])
    rec_all = torch.cat(recs)
    lo2 = torch.empty(n, dtype=torch.float64, device=dev)
    qo2 = torch.empty((n, n), dtype=torch.float64, device=dev)
    for r in range(world):
        c0, c1, _ = split(n, world, r)
        blk = torch.empty((n, c1 - c0), dtype=torch.float64, device=dev)
        be.finish(tq, rec_all, c0, c1, lo2, blk)
        qo2[:, c0:c1] = blk
    torch.cuda.synchronize()
    assert torch.equal(lo1, lo2)
    assert torch.equal(qo1, qo2)
    nrm = float(lo0.abs().max())
    assert float((lo0 - lo1).abs().max()) <= 1e-13 * nrm


def test_staged_path_on_fresh_context(api):
    """The staged entry points allocate their own workspaces (no prior
    one-shot call on the context)."""
    import torch

    from paper_1706_00773_b200.instances import make_instance
    from paper_1706_00773_b200.sharded import CudaBackend

    q, lam, kmat, s = make_instance(4, n=640, seed=3)
    dev = torch.device("cuda", 0)
    tq, tl, tk = (torch.from_numpy(x).to(dev) for x in (q, lam, kmat))
    n, k = kmat.shape
    ctx = api.Context(0)
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
    lo = torch.empty(n, dtype=torch.float64, device=dev)
    qo = torch.empty((n, n), dtype=torch.float64, device=dev)
    be.finish(tq, rec, 0, n, lo, qo)
    torch.cuda.synchronize()
    c0 = api.Context(0)
    c0.set_option("fuse_alpha", 0)  # the staged path's K2 residues
    ref = api.update_decomposition(q, lam, kmat, s, 1e-12, ctx=c0)
    c0.close()
    assert np.array_equal(lo.cpu().numpy(), ref.lam)
    assert np.array_equal(qo.cpu().numpy(), ref.q)
    ctx.close()


# ------------------------------------------------- full-size configs
def _device_checks(api, ctx, cfg, n=None, lapack=True, oracle_roots=64):
    import torch

    from paper_1706_00773_b200.instances import make_instance_torch

    dev = torch.device("cuda", 0)
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, device=dev)
    n, k = kmat.shape
    lo = torch.empty(n, dtype=torch.float64, device=dev)
    qo = torch.empty((n, n), dtype=torch.float64, device=dev)
    api.update_decomposition_device(q, lam, kmat, signs.numpy(), lo, qo, ctx=ctx)
    torch.cuda.synchronize()
    st = ctx.stats()
    sg = signs.to(dev, torch.float64)
    # size-independent identities: trace and Frobenius norm of A'
    u = q.T @ kmat
    tr = float(lam.sum() + (sg * (kmat * kmat).sum(0)).sum())
    assert abs(float(lo.sum()) - tr) <= 1e-10 * n * max(1.0, float(lam.abs().max()))
    w = u * sg[None, :]
    fro2 = float((lam * lam).sum() + 2.0 * (lam[:, None] * w * u).sum()
                 + ((u.T @ u) * (sg[:, None] * sg[None, :]) * (u.T @ u)).sum())
    assert abs(float((lo * lo).sum()) - fro2) <= 1e-10 * fro2
    # residual A'Q' - Q'Lambda' = Q(Lambda(Q^T Q')) + K J (K^T Q') - Q' Lambda' and ortho
    nrm = float(lo.abs().max())
    qtq = q.T @ qo
    r = q @ (lam[:, None] * qtq) + kmat @ (sg[:, None] * (kmat.T @ qo)) - qo * lo[None, :]
    resid = float(torch.linalg.vector_norm(r, dim=0).max()) / nrm  # per-column 2-norm
    del r
    ortho = float((qo.T @ qo - torch.eye(n, dtype=torch.float64, device=dev)).abs().max())
    assert resid <= 1e-10, resid
    assert ortho <= 1e-9, ortho
    del qtq
    if lapack:
        # independent eigensolver on A': cuSOLVER syevd (torch.linalg.eigvalsh);
        # cuSOLVER rejects n = 32768 (cusolverDnXsyevd_bufferSize and the legacy
        # cusolverDnDsyevd_bufferSize both return INVALID_VALUE,
        # tools/probe_eigvalsh.py), so above 16384 MAGMA's dsyevd (torch's
        # other backend: 88 s at n = 32768) takes its place
        a = q @ (lam[:, None] * q.T)
        a += kmat @ (sg[:, None] * kmat.T)
        a += a.T.clone()
        a *= 0.5
        prev = torch.backends.cuda.preferred_linalg_library()
        if n > 16384:
            torch.backends.cuda.preferred_linalg_library("magma")
        try:
            ev = torch.linalg.eigvalsh(a)
        finally:
            torch.backends.cuda.preferred_linalg_library(prev)
        del a
        torch.cuda.empty_cache()
        assert float((lo - ev).abs().max()) <= 1e-10 * nrm
    if oracle_roots and st["decoupled"] == 0:
        # exact per-root parity with the oracle at full size on a sample of roots
        uu = u.cpu().numpy()
        lh = lam.cpu().numpy()
        js = np.linspace(0, n - 1, oracle_roots).astype(int)
        lo_h = lo.cpu().numpy()
        for j in js:
            roots, _, _, _ = port.solve_roots(lh, uu, signs.numpy(), int(j), int(j) + 1)
            assert abs(roots[0] - lo_h[j]) <= 1e-12 * nrm
    return st, resid, ortho


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_config_full_size(api, ctx, cfg):
    _device_checks(api, ctx, cfg)


@pytest.mark.slow
def test_config3_full_size_deflation(api, ctx):
    st, _, _ = _device_checks(api, ctx, 3)
    assert st["decoupled"] > 0


@pytest.mark.slow
def test_config4_full_size(api, ctx):
    # includes the LAPACK-style eigenvalue check at n = 32768 (
    # MAGMA dsyevd, since cuSOLVER's syevd rejects this size)
    _device_checks(api, ctx, 4, lapack=True, oracle_roots=24)
