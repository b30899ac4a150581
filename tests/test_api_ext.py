"""The rest of the reference's public API on the path (VERDICT r1 missing #4,
next #3) through the C ABI, against the UNMODIFIED reference (oracle/_ref):

  assemble_eigenvectors  eigvec.hpp:29-31   consumes its plan (no K2/K3 relaunch)
  null_problem           eigvec.hpp:19      vs the reference, 1e-13 relative
  null_direction         eigvec.hpp:15      host k x k (CPU test)
  update_eigenvector     eigvec.hpp:25      vs the reference and our Q' column
  crossing_count         secular.hpp:48     bit-identical counts
  dnc_solve              rootfind.hpp:28    vs the reference within tol
  solve_rank1            rootfind.hpp:33    vs the reference within tol
  locate_rank2 / _k      locate.hpp:31,50   counts from the coefficients
  kernels::gemm_*        kernels.hpp:19-21  vs numpy
  multi-GPU context      SURVEY §8(b)       one device = the single-device path
"""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SEEDED = np.load(os.path.join(HERE, "golden", "ref_seeded.npz"))
CASES = sorted({k.split("__")[0] for k in SEEDED.files})


def _case(name):
    return {f.split("__")[1]: SEEDED[f] for f in SEEDED.files if f.split("__")[0] == name}


def _instance(n, k, seed, mixed=True):
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    q *= np.sign(np.diag(r))
    lam = np.sort(rng.uniform(-1, 1, n))
    kmat = rng.standard_normal((n, k)) / np.sqrt(n)
    signs = np.array([1 if (c % 2 == 0 or not mixed) else -1 for c in range(k)], np.int32)
    return q, lam, kmat, signs


# ------------------------------------------------------------------ CPU
def test_null_direction_matches_reference_host():
    from oracle import ref
    from paper_1706_00773_b200 import capi

    rng = np.random.default_rng(3)
    for k in (1, 2, 3, 5, 8, 16):
        m = rng.standard_normal((k, k))
        m[:, 0] = m[:, 1:].sum(axis=1) if k > 1 else 0.0  # singular
        d, r = capi.null_direction(m)
        dr, rr = ref.null_direction(m)
        assert abs(abs(d @ dr) - 1.0) <= 1e-10
        assert abs(r - rr) <= 1e-12 * max(1.0, np.abs(m).max())
        assert np.linalg.norm(m @ d) <= 1e-10 * max(1.0, np.linalg.norm(m))


def test_split_partition():
    from paper_1706_00773_b200 import capi
    from paper_1706_00773_b200.sharded import split

    for n in (0, 1, 7, 32768, 32769):
        for world in (1, 2, 3, 8):
            got = [capi.split(n, world, r) for r in range(world)]
            assert got == [split(n, world, r)[:2] for r in range(world)]
            assert sum(hi - lo for lo, hi in got) == n
    with pytest.raises(ValueError):
        capi.split(10, 2, 2)


def test_multi_context_without_gpu_fails_loudly():
    import torch

    from paper_1706_00773_b200 import capi

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(capi.DeviceError):
        capi.MultiContext([0])


# ------------------------------------------------------------------ GPU
gpu = pytest.mark.gpu


@gpu
def test_assemble_consumes_the_plan():
    from paper_1706_00773_b200 import capi

    q, lam, kmat, s = _instance(300, 4, 1)
    ctx = capi.Context(0)
    plan = capi.update_eigenvalues_full(q, lam, kmat, s, 1e-12, ctx=ctx)
    before = capi.stage_calls(ctx)
    lo, qo, path = capi.assemble_eigenvectors(q, lam, plan, ctx=ctx, return_path=True)
    after = capi.stage_calls(ctx)
    assert path == 1
    assert after["solve"] == before["solve"] and after["plan"] == before["plan"]
    assert after["project"] == before["project"] and after["columns"] == before["columns"] + 1
    full = capi.update_decomposition(q, lam, kmat, s, 1e-12, ctx=ctx)
    assert np.array_equal(lo, full.lam) and np.array_equal(qo, full.q)
    ctx.close()


@gpu
@pytest.mark.parametrize("name", [c for c in CASES if not c.startswith("c3")])
def test_assemble_accepts_the_reference_plan(name):
    """A plan produced by the reference (its roots and deflation record): not
    this context's plan, so it is checked against the secular equation and
    the columns are built for it (path 2)."""
    from paper_1706_00773_b200 import capi

    c = _case(name)
    q, lam, kmat, s = c["q"], c["lam"], c["kmat"], c["signs"]
    a = (q * lam) @ q.T + (kmat * s) @ kmat.T
    ev = np.linalg.eigvalsh(0.5 * (a + a.T))
    nrm = float(np.abs(ev).max())
    if str(c["eig_status"]) != "ok" or np.abs(c["values"] - ev).max() > 1e-10 * nrm:
        pytest.skip("the reference's eigenvalue stage failed or disagrees with LAPACK")
    prob = capi.DeflatedProblem(c["dp_poles"], c["dp_weights"], c["dp_pole_origin"],
                                c["dp_unchanged"], c["dp_collided"])
    plan = capi.EigenvalueUpdate(c["values"], c["roots"], prob, c["u"], s)
    ctx = capi.Context(0)
    lo, qo, path = capi.assemble_eigenvectors(q, lam, plan, ctx=ctx, return_path=True)
    assert path == 2
    ours = capi.update_decomposition(q, lam, kmat, s, 1e-12, ctx=ctx)
    # the plan's U is the reference's (CPU gemm_tn), ours comes from K1
    assert np.abs(lo - ours.lam).max() <= 1e-12 * nrm
    assert np.abs(qo - ours.q).max() <= 1e-8
    bad = capi.EigenvalueUpdate(c["values"], c["roots"] + 1e-3, prob, c["u"], s)
    with pytest.raises(capi.NumericalError) as e:
        capi.assemble_eigenvectors(q, lam, bad, ctx=ctx)
    assert e.value.stage == "assemble"
    short = capi.EigenvalueUpdate(c["values"], c["roots"][:-1], prob, c["u"], s)
    with pytest.raises(capi.NumericalError):  # eigvec.cpp:277-278 count mismatch
        capi.assemble_eigenvectors(q, lam, short, ctx=ctx)
    ctx.close()


@gpu
def test_null_problem_and_update_eigenvector_vs_reference():
    from oracle import ref
    from paper_1706_00773_b200 import capi

    q, lam, kmat, s = _instance(160, 3, 2)
    u = q.T @ kmat
    res = capi.update_decomposition(q, lam, kmat, s, 1e-12)
    for j in (0, 40, 159):
        root = res.lam[j]
        m = capi.null_problem(u, s, lam, root)
        mr = ref.null_problem(u, s, lam, root)
        assert np.abs(m - mr).max() <= 1e-12 * max(1.0, np.abs(mr).max())
        v = capi.update_eigenvector(q, lam, kmat, s, root)
        assert np.abs(v - res.q[:, j]).max() <= 1e-8
        vr = ref.update_eigenvector(q, lam, kmat, s, root)
        assert np.abs(v - vr).max() <= 1e-6
    # on an old eigenvalue whose row does not couple: the old vector exactly
    u2 = u.copy()
    u2[7] = 0.0
    k2 = q @ u2
    v = capi.update_eigenvector(q, lam, k2, s, lam[7])
    assert np.array_equal(v, q[:, 7])
    with pytest.raises(capi.NumericalError) as e:
        capi.update_eigenvector(q, lam, kmat, s, 0.5 * (res.lam[3] + res.lam[4]))
    assert e.value.stage == "eigvec"
    with pytest.raises(ValueError):
        capi.null_problem(u, s, lam, lam[3])


@gpu
@pytest.mark.parametrize("name", [c for c in CASES if not c.startswith("c3")])
def test_secular_functions_vs_reference(name):
    from oracle import ref
    from paper_1706_00773_b200 import capi

    c = _case(name)
    p, w = c["dp_poles"], c["dp_weights"]
    if len(p) < 3:
        pytest.skip("no secular problem")
    # eval_secular: the reference's rounding, bit for bit
    xs = np.concatenate([0.5 * (p[:-1] + p[1:]), p[:3] - 1e-3, [p[-1] + 0.7]])
    f, fp, hit = capi.secular_eval(p, w, xs, derivative=True)
    assert not hit.any()
    for x, fx in zip(xs, f):
        assert fx == ref.eval_secular(p, w, x)
    # crossing_count: identical counts
    for samples in (1, 8, 65, 500):
        assert capi.crossing_count(p, w, p[0] - 0.1, p[-1] + 0.1, samples) == \
            ref.crossing_count(p, w, p[0] - 0.1, p[-1] + 0.1, samples)
    # dnc_solve on one-root brackets between poles (counts from the coefficients)
    counts = capi.locate_coeffs(p, w)
    assert sum(counts) == len(p)
    tol = float(c["tol"])
    for i in np.linspace(1, len(p) - 1, 6).astype(int):
        if counts[i] != 1:
            continue
        gap = p[i] - p[i - 1]
        lo, hi = p[i - 1] + 1e-12 * gap, p[i] - 1e-12 * gap
        r = capi.dnc_solve(p, w, lo, hi, 1, tol)
        rr = ref.dnc_solve(p, w, lo, hi, 1, tol)
        assert len(r) == 1 and abs(r[0] - rr[0]) <= 2 * tol
    # locate from the coefficients = the reference's locate_rank2 / _k where it agrees
    sg = c["signs"]
    try:
        want = ref.locate_coeffs(p, w, sg)
    except Exception:
        want = None
    if want is not None and sum(want) == len(p):
        assert counts == want


@gpu
def test_solve_rank1_vs_reference():
    from oracle import ref
    from paper_1706_00773_b200 import capi

    rng = np.random.default_rng(8)
    for n, sigma in ((2, 1.0), (50, 1.0), (300, -0.7), (1000, 2.5)):
        p = np.sort(rng.uniform(-1, 1, n))
        z = rng.standard_normal(n) / np.sqrt(n)
        tol = 1e-13
        r = capi.solve_rank1(p, z, sigma, tol)
        rr = ref.solve_rank1(p, z, sigma, tol)
        ev = np.linalg.eigvalsh(np.diag(p) + sigma * np.outer(z, z))
        assert np.abs(r - ev).max() <= 1e-12 * max(1.0, np.abs(ev).max())
        assert np.abs(r - rr).max() <= 1e-10 * max(1.0, np.abs(ev).max())
    assert np.array_equal(capi.solve_rank1(p, z, 0.0, 1e-12), p)
    z[3] = 0.0
    with pytest.raises(ValueError):
        capi.solve_rank1(p, z, 1.0, 1e-12)


@gpu
def test_gemm_variants():
    from paper_1706_00773_b200 import capi

    rng = np.random.default_rng(4)
    # kk = 97 .. 1000: 7 .. 63 k-tiles, the 6-stage TMA ring refills and its
    # barrier parities wrap (the K5 main loop's incremental stage state)
    for m, nn, kk in ((1, 1, 1), (37, 5, 13), (130, 257, 64), (64, 64, 1), (130, 140, 97),
                      (129, 128, 200), (256, 130, 1000)):
        a = rng.standard_normal((m, kk))
        b = rng.standard_normal((kk, nn))
        assert np.abs(capi.gemm(a, b) - a @ b).max() <= 1e-12 * kk
        assert np.abs(capi.gemm(a.T.copy(), b, trans_a=True) - a @ b).max() <= 1e-12 * kk
        assert np.abs(capi.gemm(a, b.T.copy(), trans_b=True) - a @ b).max() <= 1e-12 * kk


@gpu
def test_multi_context_one_device_equals_single():
    from paper_1706_00773_b200 import capi

    q, lam, kmat, s = _instance(700, 8, 3)
    one = capi.update_decomposition(q, lam, kmat, s, 1e-12)
    mc = capi.MultiContext([0])
    multi = mc.update_decomposition(q, lam, kmat, s, 1e-12)
    vals = mc.update_eigenvalues(q, lam, kmat, s, 1e-12)
    assert np.array_equal(multi.lam, one.lam) and np.array_equal(multi.q, one.q)
    assert np.array_equal(vals, one.lam)
    # k_eff = 0: every pair passes through exactly
    z = mc.update_decomposition(q, lam, np.zeros_like(kmat), s, 1e-12)
    assert np.array_equal(z.lam, lam) and np.array_equal(z.q, q)
    with pytest.raises(ValueError):  # signs must be +1/-1 (core.cpp:89-97)
        mc.update_decomposition(q, lam, kmat, np.array([1, 2] * 4), 1e-12)
    mc.close()
    with pytest.raises(ValueError):
        capi.MultiContext([0, 0])
