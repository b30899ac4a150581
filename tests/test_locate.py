"""Location vector: the CLI locate path
(tools/eigmod.cpp:143-161 -> deflate_problem -> locate_rank2 / locate_rank_k,
locate.hpp:13-50) against the reference fixtures (tests/golden/ref_locate.npz,
families of tests/test_locate.cpp:80-200) and LAPACK interval counts.

The reference's parity/Sturm scan is not always right (its fixtures record
the cases where it disagrees with LAPACK or throws); the oracle and the GPU
path count exactly (inertia limits at the poles), so LAPACK is the arbiter.
"""
import os

import numpy as np
import pytest

from oracle import port

HERE = os.path.dirname(os.path.abspath(__file__))
LOC = np.load(os.path.join(HERE, "golden", "ref_locate.npz"))
KEYS = sorted({k.split("__")[0] for k in LOC.files}, key=lambda s: int(s[1:]))
CASES = [(k, {f.split("__")[1]: LOC[f] for f in LOC.files if f.split("__")[0] == k}) for k in KEYS]


def _random_problem(rng, n, k, mixed=True):
    lam = np.sort(rng.uniform(-1.0, 1.0, n))
    u = rng.standard_normal((n, k)) * rng.uniform(0.05, 1.5)
    signs = rng.choice([-1, 1], k).astype(np.int32) if mixed else np.ones(k, np.int32)
    return lam, u, signs


def _lapack_counts(lam, u, signs):
    a = np.diag(lam) + (u * signs.astype(float)) @ u.T
    ev = np.linalg.eigvalsh(a)
    edges = np.concatenate([[-np.inf], lam, [np.inf]])
    return [int(((ev > edges[i]) & (ev < edges[i + 1])).sum()) for i in range(len(lam) + 1)]


# ------------------------------------------------------------------ oracle (CPU)
@pytest.mark.parametrize("name,c", CASES, ids=KEYS)
def test_oracle_locate_matches_lapack_fixture(name, c):
    assert port.locate_from_u(c["lam"], c["u"], c["signs"]) == list(c["truth"])


def test_reference_fixture_agreement_summary():
    """Where the reference succeeded its counts equal LAPACK's on these
    families (tests/test_locate.cpp asserts the same); the oracle agrees with
    both."""
    ok = [c for _, c in CASES if str(c["status"]) == "ok"]
    assert len(ok) >= 180
    for c in ok:
        assert list(c["ref"]) == list(c["truth"])


def test_oracle_locate_random_vs_lapack():
    rng = np.random.default_rng(11)
    for _ in range(120):
        n, k = int(rng.integers(3, 50)), int(rng.integers(1, 6))
        lam, u, signs = _random_problem(rng, n, k)
        assert port.locate_from_u(lam, u, signs) == _lapack_counts(lam, u, signs)


def test_oracle_locate_rank1_interlacing():
    rng = np.random.default_rng(3)
    lam, u, _ = _random_problem(rng, 30, 1)
    assert port.locate_from_u(lam, u, np.array([1])) == [0] + [1] * 30
    assert port.locate_from_u(lam, u, np.array([-1])) == [1] * 30 + [0]


def test_oracle_locate_null_update():
    lam = np.linspace(-1, 1, 7)
    assert port.locate_from_u(lam, np.zeros((7, 2)), np.array([1, -1])) == [0]


# ---------------------------------------------------------------- GPU path
@pytest.mark.gpu
def test_gpu_locate_fixtures(ctx):
    from paper_1706_00773_b200 import capi

    for name, c in CASES:
        got = capi.locate_from_u(c["lam"], c["u"], c["signs"], ctx=ctx)
        assert got == list(c["truth"]), name


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 2, 3, 4, 7, 8, 16, 24])
def test_gpu_locate_random_vs_oracle(ctx, k):
    from paper_1706_00773_b200 import capi

    rng = np.random.default_rng(100 + k)
    for n in (40, 300, 1000):
        lam, u, signs = _random_problem(rng, n, k)
        want = port.locate_from_u(lam, u, signs)
        assert capi.locate_from_u(lam, u, signs, ctx=ctx) == want
        assert sum(want) == len(port.deflate(lam, u, signs)["poles"])


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [0, 1, 2, 4])
def test_gpu_locate_configs(ctx, cfg):
    """Host-pointer CLI path (Q, Lambda, K) at the BASELINE config shapes."""
    from paper_1706_00773_b200 import capi
    from paper_1706_00773_b200.instances import make_instance

    q, lam, kmat, signs = make_instance(cfg, n=768, seed=40 + cfg)
    got = capi.locate(q, lam, kmat, signs, ctx=ctx)
    want = port.locate_from_u(lam, port.transform(q, kmat), signs)
    assert got == want
    assert sum(got) == len(port.deflate(lam, port.transform(q, kmat), signs)["poles"])


@pytest.mark.gpu
def test_gpu_locate_deflation_config(ctx):
    """Config 3 (clusters at 1e-12, tiny rows): merged runs with k = 8 have no
    exact meaning in the reference's merged secular function; the counts are
    still a valid partition of the reduced problem's roots."""
    from paper_1706_00773_b200 import capi
    from paper_1706_00773_b200.instances import make_instance

    q, lam, kmat, signs = make_instance(3, n=512, seed=7)
    got = capi.locate(q, lam, kmat, signs, ctx=ctx)
    dp = capi.deflate_problem(lam, port.transform(q, kmat), signs, ctx=ctx)
    assert len(got) == len(dp.poles) + 1
    assert min(got) >= 0
    assert sum(got) >= len(dp.poles)


@pytest.mark.gpu
def test_gpu_locate_edge_cases(ctx):
    from paper_1706_00773_b200 import capi

    lam = np.linspace(-1, 1, 9)
    assert capi.locate_from_u(lam, np.zeros((9, 3)), np.array([1, 1, -1]), ctx=ctx) == [0]
    with pytest.raises(ValueError):
        capi.locate_from_u(lam[::-1], np.ones((9, 1)), np.array([1]), ctx=ctx)
    rng = np.random.default_rng(5)
    lam, u, _ = _random_problem(rng, 64, 1)
    assert capi.locate_from_u(lam, u, np.array([1]), ctx=ctx) == [0] + [1] * 64
    assert capi.locate_from_u(lam, u, np.array([-1]), ctx=ctx) == [1] * 64 + [0]
