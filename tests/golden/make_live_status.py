"""Records what the UNMODIFIED reference (oracle/_ref) does on the live-parity
cases of tests/test_reference_live.py: BASELINE configs 0, 1 and 4 at the
sizes where it still runs (config 0 n = 512, config 1 n = 4096, config 4
n = 2048), several seeds each. For every case: the reference's status per
stage ("ok" or its exception with the stage) and its accuracy against LAPACK.

    python tests/golden/make_live_status.py     # in the build container

Writes tests/golden/ref_live_status.json. The GPU test re-runs the reference
live on the GPU box's host cores (oracle/_ref travels with the snapshot) and
requires the same statuses, so the pinned failure record is the reference's
own behaviour on these bits, not an assumption.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from northstar import aprime, norm2, residual  # noqa: E402
from oracle import ref  # noqa: E402
from paper_1706_00773_b200.instances import default_seed, make_instance  # noqa: E402

# (config, n, seed offsets, stages): "pairs" = update_eigenvalues_full +
# assemble_eigenvectors, "values" = update_eigenvalues_full only
LIVE_CASES = [
    (0, 512, range(5), "pairs"),
    (1, 4096, range(2), "pairs"),
    (4, 2048, range(5), "pairs"),
]


def case_id(cfg, n, s):
    return f"cfg{cfg}_n{n}_s{s}"


def run_reference(cfg, n, s, stages):
    q, lam, kmat, signs = make_instance(cfg, n=n, seed=default_seed(cfg) + s)
    tol = ref.default_tolerance(lam, kmat, signs)
    out = {"tol": tol}
    try:
        vals, _, _ = ref.update_eigenvalues_full(q, lam, kmat, signs, tol)
        out["eig_status"], out["values"] = "ok", vals
    except Exception as e:  # noqa: BLE001 - the reference's failure is the record
        out["eig_status"] = f"{type(e).__name__}: {e}"
    if stages == "pairs":
        try:
            lo, qo, _ = ref.update_pairs(q, lam, kmat, signs, tol)
            out["vec_status"], out["lam_out"], out["q_out"] = "ok", lo, qo
        except Exception as e:  # noqa: BLE001
            out["vec_status"] = f"{type(e).__name__}: {e}"
    return (q, lam, kmat, signs), out


def main():
    ref.set_parallel(True)
    rec = {}
    for cfg, n, seeds, stages in LIVE_CASES:
        for s in seeds:
            (q, lam, kmat, signs), out = run_reference(cfg, n, s, stages)
            a = aprime(q, lam, kmat, signs)
            ev = np.linalg.eigvalsh(a)
            nrm = norm2(ev)
            r = {"eig_status": out["eig_status"], "vec_status": out.get("vec_status")}
            if out["eig_status"] == "ok":
                r["eig_err_vs_lapack"] = float(np.abs(out["values"] - ev).max() / nrm)
            if out.get("vec_status") == "ok":
                r["vec_residual"] = residual(a, out["q_out"], out["lam_out"], nrm)
            rec[case_id(cfg, n, s)] = r
            print(case_id(cfg, n, s), r, flush=True)
    with open(os.path.join(HERE, "ref_live_status.json"), "w") as f:
        json.dump(rec, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
