"""Live parity with the UNMODIFIED reference at the sizes where it completes
(VERDICT r1 next #1): BASELINE config 0 at n = 512, config 1 at n = 4096 and
config 4 at n = 2048, several seeds. The reference (oracle/_ref, compiled from
its own sources; the .so travels to the GPU box) runs on the host cores in the
same process; the GPU path runs through the host-pointer C ABI.

  * the reference's status per stage is recorded (gpurun_out/
    ref_live_status_gpu.json on the GPU box; tests/golden/ref_live_status.json
    holds the build container's run of tests/golden/make_live_status.py). It is
    not asserted: the instances come from numpy's LAPACK QR, whose bits
    depend on the host CPU, and the reference's locate stage fails on some
    instances and not on their 1-ulp neighbours (in the build container its
    eigenvector stage throws on 2 of 5 config-0 seeds and on every config-1
    seed; on the GPU box its locate stage also threw on 2 of 3 config-4
    n = 2048 seeds);
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

RECORD = {}


def _record(key, value):
    RECORD[key] = value
    root = os.environ.get("GRAFT_REPO_ROOT")
    if root and os.path.isdir(os.path.join(root, "gpurun_out")):
        with open(os.path.join(root, "gpurun_out", "ref_live_status_gpu.json"), "w") as f:
            json.dump(RECORD, f, indent=1, sort_keys=True)


PARAMS = [(cfg, n, s, stages) for cfg, n, seeds, stages in LIVE_CASES for s in seeds]


@pytest.mark.parametrize("cfg,n,s,stages", PARAMS, ids=[case_id(c, n, s) for c, n, s, _ in PARAMS])
def test_live_reference_parity(cfg, n, s, stages):
    from oracle import ref
    from paper_1706_00773_b200 import capi

    ref.set_parallel(True)
    (q, lam, kmat, signs), out = run_reference(cfg, n, s, stages)
    res = capi.update_decomposition(q, lam, kmat, signs, out["tol"])
    a = aprime(q, lam, kmat, signs)
    ev = np.linalg.eigvalsh(a)
    nrm = norm2(ev)
    rec = {"eig_status": out["eig_status"], "vec_status": out.get("vec_status"),
           "gpu_eig_err_vs_lapack": float(np.abs(res.lam - ev).max() / nrm),
           "gpu_residual": residual(a, res.q, res.lam, nrm), "gpu_ortho": ortho(res.q)}
    if out["eig_status"] == "ok":
        rec["ref_eig_err_vs_lapack"] = float(np.abs(out["values"] - ev).max() / nrm)
        rec["gpu_vs_ref_eig"] = float(np.abs(res.lam - out["values"]).max() / nrm)
    if out.get("vec_status") == "ok":
        rec["ref_residual"] = residual(a, out["q_out"], out["lam_out"], nrm)
        rec["gpu_vs_ref_vectors_max"] = float(np.abs(res.q - out["q_out"]).max())
    _record(case_id(cfg, n, s), rec)
    assert np.abs(res.lam - ev).max() <= EIG_TOL * nrm
    assert residual(a, res.q, res.lam, nrm) <= RESID_TOL
    assert ortho(res.q) <= ORTHO_TOL
    # oracle hierarchy: the reference where it completes and
    # agrees with LAPACK within the north-star tolerance
    ref_ok = out["eig_status"] == "ok" and rec["ref_eig_err_vs_lapack"] <= EIG_TOL
    if ref_ok:
        assert np.abs(res.lam - out["values"]).max() <= EIG_TOL * nrm
    if ref_ok and out.get("vec_status") == "ok":
        assert np.abs(res.lam - out["lam_out"]).max() <= EIG_TOL * nrm
        # the reference's vectors carry its root tolerance (residual up to
        # ~1e-7 on some seeds): compare them where they meet the north-star
        # residual themselves; ours are never the less accurate ones
        if rec["ref_residual"] <= RESID_TOL:
            assert np.abs(res.q - out["q_out"]).max() <= 1e-7
        # the GPU vectors are the more accurate ones (north-star residual)
        assert residual(a, res.q, res.lam, nrm) <= residual(a, out["q_out"], out["lam_out"], nrm)
