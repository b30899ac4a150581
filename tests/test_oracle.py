"""Pins the CPU oracle (oracle/eigmod_oracle.c) before it is trusted as the
checker: against the reference's golden vectors (restated from its unit
tests), against fixtures produced by the unmodified reference
(tests/golden/ref_*.npz, see make_golden.py) and against LAPACK."""
import math

import numpy as np
import pytest

from northstar import residual
from oracle import port, ref

SEEDED = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden",
                                            "ref_seeded.npz"))
CASES = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden",
                                           "ref_cases.npz"))


def _cases(npz):
    keys = sorted({k.split("__")[0] for k in npz.files})
    return [(k, {f.split("__")[1]: npz[f] for f in npz.files if f.split("__")[0] == k}) for k in keys]


SEEDED_CASES = _cases(SEEDED)
RANDOM_CASES = _cases(CASES)


def _aprime(c):
    a = c["q"] @ np.diag(c["lam"]) @ c["q"].T + c["kmat"] @ np.diag(c["signs"].astype(float)) @ c["kmat"].T
    return 0.5 * (a + a.T)


# ------------------------------------------------------------- bit parity
@pytest.mark.parametrize("name,c", SEEDED_CASES, ids=[n for n, _ in SEEDED_CASES])
def test_transform_bit_identical_to_reference(name, c):
    # secular.cpp:155-161 / kernels.cpp:50-65, same loop order, no FMA contraction
    u = port.transform(c["q"], c["kmat"])
    assert np.array_equal(u, c["u"])


@pytest.mark.parametrize("name,c", SEEDED_CASES, ids=[n for n, _ in SEEDED_CASES])
def test_deflation_record_bit_identical_to_reference(name, c):
    # secular.cpp:278-340 (runs, group_weights/adjugate, classification)
    d = port.deflate(c["lam"], c["u"], c["signs"])
    assert np.array_equal(d["poles"], c["dp_poles"])
    assert np.array_equal(d["weights"], c["dp_weights"])
    assert np.array_equal(d["pole_origin"], c["dp_pole_origin"])
    assert np.array_equal(d["unchanged"], c["dp_unchanged"])
    assert np.array_equal(d["collided"], c["dp_collided"])


# --------------------------------------------------------- eigen-parity
@pytest.mark.parametrize("name,c", SEEDED_CASES, ids=[n for n, _ in SEEDED_CASES])
def test_oracle_eigenpairs_vs_lapack_and_reference(name, c):
    a = _aprime(c)
    ev = np.linalg.eigvalsh(a)
    nrm = float(np.abs(ev).max())
    n = len(ev)
    lo, qo, info = port.update(c["q"], c["lam"], c["kmat"], c["signs"])
    # north-star tolerances: 1e-10 ||A'|| per eigenvalue, residual 1e-10, ortho 1e-9
    assert np.abs(lo - ev).max() <= 1e-10 * nrm
    assert residual(a, qo, lo, nrm) <= 1e-10  # per-column 2-norm / ||A'||_2
    assert np.abs(qo.T @ qo - np.eye(n)).max() <= 1e-9
    if str(c["eig_status"]) == "ok":
        ref_ok = np.abs(c["values"] - ev).max() <= 1e-10 * nrm
        if ref_ok:  # oracle hierarchy: the reference where it agrees with LAPACK
            assert np.abs(lo - c["values"]).max() <= 1e-10 * nrm
    else:  # the reference fails on the config-3 clusters; LAPACK decides
        assert name.startswith("c3")
    if str(c["vec_status"]) == "ok":
        # reference vectors are accurate to ~1e-7 (root tolerance 1e-12*scale,
        # SURVEY §0.3); same column order and sign rule
        assert np.abs(qo - c["q_out"]).max() <= 1e-5
        assert np.array_equal(c["lam_out"].argsort(kind="stable"), np.arange(n))


@pytest.mark.parametrize("name,c", RANDOM_CASES, ids=[n for n, _ in RANDOM_CASES])
def test_oracle_vs_reference_random_instances(name, c):
    # tests/test_rootfind.cpp:163-178 (n=50, k=3, mixed signs, vs Jacobi 1e-9)
    lo, qo, _ = port.update(c["q"], c["lam"], c["kmat"], c["signs"])
    ev = np.linalg.eigvalsh(_aprime(c))
    assert np.abs(lo - ev).max() <= 1e-12 * max(1.0, float(np.abs(ev).max()))
    if str(c["eig_status"]) == "ok":
        assert np.abs(lo - c["values"]).max() <= 1e-9
    if str(c["vec_status"]) == "ok":
        assert np.abs(qo - c["q_out"]).max() <= 1e-5


# ---------------------------------------------------- restated goldens
R2 = math.sqrt(2.0)


def test_golden_2x2_update():
    # tests/test_eigvec.cpp:107-123, test_rootfind.cpp:135-140, test_cli.cpp:62-63
    lo, qo, _ = port.update(np.eye(2), np.array([0.0, 1.0]), np.array([[1.0, 0.0], [1.0, 1.0]]),
                            np.array([1, 1]))
    assert abs(lo[0] - 0.58578643762690495) <= 1e-12 * 2
    assert abs(lo[1] - 3.4142135623730951) <= 1e-12 * 4
    lam = 2.0 - R2
    nrm = math.sqrt(1.0 + (lam - 1.0) ** 2)
    assert abs(qo[0, 0] - 1.0 / nrm) <= 1e-12
    assert abs(qo[1, 0] - (lam - 1.0) / nrm) <= 1e-12


def test_golden_k_zero_is_exact_identity():
    # tests/test_eigvec.cpp:97-105 and test_rootfind.cpp:142-148
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((8, 8)))
    lam = np.sort(rng.uniform(-1, 1, 8))
    lo, qo, info = port.update(q, lam, np.zeros((8, 2)), np.array([1, 1]))
    assert np.array_equal(lo, lam) and np.array_equal(qo, q)


def test_golden_rank1_collision():
    # tests/test_rootfind.cpp:150-161: diag(1,2) + e1 e1^T = diag(2,2)
    lo, qo, _ = port.update(np.eye(2), np.array([1.0, 2.0]), np.array([[1.0], [0.0]]), np.array([1]))
    assert np.allclose(lo, [2.0, 2.0], rtol=0, atol=2e-12)
    assert np.abs(qo.T @ qo - np.eye(2)).max() <= 1e-12


def test_golden_collided_eigenvector():
    # tests/test_eigvec.cpp:64-76: diag(0,1) + I = diag(1,2): e1 for 1, e2 for 2
    lo, qo, info = port.update(np.eye(2), np.array([0.0, 1.0]), np.eye(2), np.array([1, 1]))
    assert np.allclose(lo, [1.0, 2.0], atol=1e-14)
    assert np.allclose(np.abs(qo), np.eye(2), atol=1e-14)
    assert info["collided"] == 1  # lambda' = 1 sits on the old eigenvalue 1


def test_golden_secular_weights():
    # tests/test_secular.cpp:97-126
    inv = 1.0 / R2
    a = port.secular_weights([1.0, 2.0], [[inv], [inv]], [1])
    assert np.allclose(a, [0.5, 0.5], rtol=1e-13)
    a = port.secular_weights([0.0, 1.0], np.eye(2), [1, 1])
    assert abs(a[0] - 2.0) <= 2e-13 and abs(a[1]) <= 1e-15
    a = port.secular_weights([0.0, 1.0], [[1.0, 0.0], [1.0, 1.0]], [1, 1])
    assert np.allclose(a, [2.0, 1.0], rtol=1e-13)


def test_golden_rank1_weights_are_zeta_squared():
    # tests/test_secular.cpp:128-145
    rng = np.random.default_rng(17)
    for _ in range(25):
        n = 2 + int(rng.integers(0, 9))
        lam = np.sort(rng.standard_normal(n))
        for i in range(1, n):
            lam[i] = max(lam[i], lam[i - 1] + 1e-4)
        u = rng.standard_normal((n, 1))
        a = port.secular_weights(lam, u, [1])
        assert np.all(a >= 0) and np.allclose(a, u[:, 0] ** 2, rtol=1e-13)


def test_residue_oracle():
    # tests/test_secular.cpp:147-176: alpha_i = lim (lambda_i - x) det[I - J U^T (x-L)^-1 U]
    rng = np.random.default_rng(29)
    for _ in range(20):
        n = 3 + int(rng.integers(0, 10))
        k = 1 + int(rng.integers(0, 3))
        lam = np.sort(rng.standard_normal(n))
        for i in range(1, n):
            lam[i] = max(lam[i], lam[i - 1] + 5e-2)
        u = rng.standard_normal((n, k))
        s = np.where(rng.integers(0, 2, k) == 1, 1, -1)
        alpha = port.secular_weights(lam, u, s)

        def det_id(x):
            m = np.eye(k) - (s[:, None] * (u.T / (x - lam)[None, :])) @ u
            return np.linalg.det(m)

        for i in range(n):
            gap = min(abs(lam[j] - lam[i]) for j in range(n) if j != i)
            h = 1e-6 * gap
            est = 0.5 * (h * det_id(lam[i] - h) - h * det_id(lam[i] + h))
            assert abs(est - alpha[i]) <= 1e-4 * abs(alpha[i]) + 1e-8


def test_golden_deflation_cases():
    # tests/test_secular.cpp:273-298
    d = port.deflate([0.0, 1.0, 2.0], [[0.0], [0.5], [0.0]], [1])
    assert np.allclose(d["poles"], [1.0]) and np.allclose(d["weights"], [0.25])
    assert list(d["unchanged"]) == [0, 2] and list(d["pole_origin"]) == [1]
    d = port.deflate([1.0, 1.0 + 1e-15, 2.0], [[1.0], [2.0], [1.0]], [1])
    assert len(d["poles"]) == 2 and abs(d["weights"][0] - 5.0) <= 5e-9
    assert len(d["unchanged"]) == 1


def test_inertia_count_matches_lapack():
    # #eig(A') < x = #{d_i < x} + m - nu(S(x))
    rng = np.random.default_rng(5)
    for k, signs in ((4, [1, -1, 1, -1]), (3, [1, 1, -1]), (1, [-1])):
        n = 40
        d = np.sort(rng.uniform(-1, 1, n))
        u = rng.standard_normal((n, k)) * 0.3
        a = np.diag(d) + u @ np.diag(np.array(signs, float)) @ u.T
        ev = np.linalg.eigvalsh(a)
        for x in rng.uniform(-3, 3, 200):
            assert port.count_below(d, u, signs, x) == int((ev < x).sum())


def test_config3_exact_mode_meets_tolerances():
    # the reference fails here (fixtures c3_*); exact mode is checked against LAPACK
    from paper_1706_00773_b200.instances import make_instance

    q, lam, kmat, s = make_instance(3, n=400, seed=3)
    a = q @ np.diag(lam) @ q.T + kmat @ np.diag(s.astype(float)) @ kmat.T
    a = 0.5 * (a + a.T)
    ev = np.linalg.eigvalsh(a)
    nrm = float(np.abs(ev).max())
    lo, qo, info = port.update(q, lam, kmat, s, run_rel=port.EXACT_RUN_REL)
    assert info["decoupled"] > 0
    assert np.abs(lo - ev).max() <= 1e-10 * nrm
    assert residual(a, qo, lo, nrm) <= 1e-10  # per-column 2-norm / ||A'||_2
    assert np.abs(qo.T @ qo - np.eye(len(lam))).max() <= 1e-9


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_fixture_replay_matches_live_reference():
    # the committed fixtures are what the reference produces here and now
    name, c = SEEDED_CASES[0]
    u = ref.transform_update(c["q"], c["lam"], c["kmat"], c["signs"])
    assert np.array_equal(u, c["u"])
