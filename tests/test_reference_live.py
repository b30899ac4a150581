"""Live parity with the UNMODIFIED reference at the sizes where it completes
(VERDICT r1 next #1): BASELINE config 0 at n = 512, config 1 at n = 4096 and
config 4 at n = 2048, several seeds. The reference (oracle/_ref, compiled from
its own sources; the .so travels to the GPU box) runs on the host cores in the
same process; the GPU path runs through the host-pointer C ABI.

  * the reference's status per stage equals the pinned record
    (tests/golden/ref_live_status.json, tests/golden/make_live_status.py):
    its eigenvector stage throws on 2 of 5 config-0 seeds and on every
    config-1 seed ("[assemble] root ... rejected by the null problem");
  * where it completes: |lambda'_gpu - lambda'_ref| <= 1e-10 ||A'||_2 (the
    north-star eigenvalue tolerance) and Q'_gpu = Q'_ref within 1e-7 (same
    column order and sign rule; the reference's own vectors carry ~1e-9
    errors from its absolute root tolerance);
  * always: the GPU result meets the north-star tolerances against LAPACK
    (eigenvalues, per-column residual, orthogonality), including the cases the
    reference cannot finish.
"""
import json
import os
import sys

import numpy as np
import pytest

from northstar import EIG_TOL, ORTHO_TOL, RESID_TOL, aprime, norm2, ortho, residual

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from make_live_status import LIVE_CASES, case_id, run_reference  # noqa: E402

pytestmark = pytest.mark.gpu

with open(os.path.join(HERE, "golden", "ref_live_status.json")) as _f:
    STATUS = json.load(_f)

PARAMS = [(cfg, n, s, stages) for cfg, n, seeds, stages in LIVE_CASES for s in seeds]


@pytest.mark.parametrize("cfg,n,s,stages", PARAMS, ids=[case_id(c, n, s) for c, n, s, _ in PARAMS])
def test_live_reference_parity(cfg, n, s, stages):
    from oracle import ref
    from paper_1706_00773_b200 import capi

    ref.set_parallel(True)
    (q, lam, kmat, signs), out = run_reference(cfg, n, s, stages)
    pinned = STATUS[case_id(cfg, n, s)]
    assert out["eig_status"] == pinned["eig_status"]
    assert out.get("vec_status") == pinned["vec_status"]

    res = capi.update_decomposition(q, lam, kmat, signs, out["tol"])
    a = aprime(q, lam, kmat, signs)
    ev = np.linalg.eigvalsh(a)
    nrm = norm2(ev)
    assert np.abs(res.lam - ev).max() <= EIG_TOL * nrm
    assert residual(a, res.q, res.lam, nrm) <= RESID_TOL
    assert ortho(res.q) <= ORTHO_TOL
    if out["eig_status"] == "ok":
        assert np.abs(res.lam - out["values"]).max() <= EIG_TOL * nrm
    if out.get("vec_status") == "ok":
        assert np.abs(res.lam - out["lam_out"]).max() <= EIG_TOL * nrm
        assert np.abs(res.q - out["q_out"]).max() <= 1e-7
        # the GPU vectors are the more accurate ones (north-star residual)
        assert residual(a, res.q, res.lam, nrm) <= residual(a, out["q_out"], out["lam_out"], nrm)
