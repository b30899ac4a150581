"""Validation products on the GPU: reconstruct
(core.hpp:11, kernels.cpp:98-109), apply_update (core.hpp:14,
core.cpp:105-115) and ortho_error (kernels.hpp:36, kernels.cpp:150-154)
against fixtures of the unmodified reference (tests/golden/ref_validation.npz,
written by make_golden.py)."""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
VAL = np.load(os.path.join(HERE, "golden", "ref_validation.npz"))
KEYS = sorted({k.split("__")[0] for k in VAL.files})
CASES = [(k, {f.split("__")[1]: VAL[f] for f in VAL.files if f.split("__")[0] == k}) for k in KEYS]


@pytest.mark.parametrize("name,c", CASES, ids=KEYS)
def test_fixture_consistent_with_numpy(name, c):
    """Pins the fixtures: the reference's products agree with numpy."""
    a = (c["q"] * c["lam"]) @ c["q"].T
    a = 0.5 * (a + a.T)
    assert np.abs(c["reconstruct"] - a).max() <= 1e-13 * max(1.0, np.abs(a).max())
    b = c["reconstruct"] + (c["kmat"] * c["signs"].astype(float)) @ c["kmat"].T
    assert np.abs(c["apply_update"] - b).max() <= 1e-13 * max(1.0, np.abs(b).max())
    assert np.array_equal(c["apply_update"], c["apply_update"].T)
    g = c["q"].T @ c["q"] - np.eye(c["q"].shape[1])
    assert abs(float(c["ortho_q"]) - np.abs(g).max()) <= 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("name,c", CASES, ids=KEYS)
def test_gpu_apply_update_bit_identical(ctx, name, c):
    from paper_1706_00773_b200 import capi

    got = capi.apply_update(c["reconstruct"], c["kmat"], c["signs"], ctx=ctx)
    assert np.array_equal(got, c["apply_update"])


@pytest.mark.gpu
@pytest.mark.parametrize("name,c", CASES, ids=KEYS)
def test_gpu_reconstruct_and_ortho(ctx, name, c):
    from paper_1706_00773_b200 import capi

    a = capi.reconstruct(c["q"], c["lam"], ctx=ctx)
    assert np.array_equal(a, a.T)  # symmetrized exactly
    ref_a = c["reconstruct"]
    assert np.abs(a - ref_a).max() <= 1e-14 * c["q"].shape[0] * max(1.0, np.abs(ref_a).max())
    for key, mat in (("ortho_q", c["q"]), ("ortho_rect", c["rect"])):
        got = capi.ortho_error(mat, ctx=ctx)
        assert abs(got - float(c[key])) <= 1e-14 * mat.shape[0]


@pytest.mark.gpu
def test_gpu_validation_large(ctx):
    """Device forms at a size where the products run on full DMMA tiles."""
    import torch

    from paper_1706_00773_b200 import capi
    from paper_1706_00773_b200.instances import make_instance_torch

    dev = torch.device("cuda", 0)
    q, lam, kmat, signs = make_instance_torch(2, n=1536, device=dev)
    n, k = kmat.shape
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    a = torch.empty((n, n), dtype=torch.float64, device=dev)
    ctx.check(ctx._l.eigmod_b200_reconstruct_device(ctx.h, capi._ptr(q), capi._ptr(lam), n,
                                                    capi._ptr(a)))
    b = torch.empty_like(a)
    s = np.ascontiguousarray(signs.numpy(), np.int32)
    ctx.check(ctx._l.eigmod_b200_apply_update_device(
        ctx.h, capi._ptr(a), capi._ptr(kmat), s.ctypes.data_as(capi._I32), n, k, capi._ptr(b)))
    err = np.zeros(1)
    ctx.check(ctx._l.eigmod_b200_ortho_error_device(ctx.h, capi._ptr(q), n, n,
                                                    err.ctypes.data_as(capi._D)))
    torch.cuda.synchronize()
    want = (q * lam) @ q.T
    want = 0.5 * (want + want.T)
    assert float((a - want).abs().max()) <= 1e-13
    sg = signs.to(dev, torch.float64)
    want_b = a + (kmat * sg) @ kmat.T
    assert float((b - want_b).abs().max()) <= 1e-13
    g = q.T @ q - torch.eye(n, dtype=torch.float64, device=dev)
    assert abs(err[0] - float(g.abs().max())) <= 1e-14
