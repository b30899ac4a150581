"""Generates the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists and
`make -C oracle ref` has built oracle/_ref/libeigmod_ref.so):

    python tests/golden/make_golden.py

Writes tests/golden/ref_seeded.npz and tests/golden/ref_cases.npz. Inputs
are stored next to the reference outputs so the fixtures do not depend on
LAPACK bits of the machine that replays them. The GPU box never reads
/root/reference: it only reads these files.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_1706_00773_b200.instances import make_instance  # noqa: E402


def run_case(q, lam, kmat, signs, tol=None):
    out = {"q": q, "lam": lam, "kmat": kmat, "signs": np.asarray(signs, np.int32)}
    tol = ref.default_tolerance(lam, kmat, signs) if tol is None else tol
    out["tol"] = np.array(tol)
    out["u"] = ref.transform_update(q, lam, kmat, signs)
    dp = ref.deflate_problem(lam, out["u"], signs)
    for key, v in dp.items():
        out["dp_" + key] = v
    try:
        vals, roots, _ = ref.update_eigenvalues_full(q, lam, kmat, signs, tol)
        out["values"], out["roots"], out["eig_status"] = vals, roots, np.array("ok")
    except Exception as e:  # the reference's own failure, recorded
        out["eig_status"] = np.array(f"{type(e).__name__}: {e}")
    try:
        lo, qo, _ = ref.update_pairs(q, lam, kmat, signs, tol)
        out["lam_out"], out["q_out"], out["vec_status"] = lo, qo, np.array("ok")
    except Exception as e:
        out["vec_status"] = np.array(f"{type(e).__name__}: {e}")
    return out


def main():
    ref.set_parallel(False)
    seeded = {}
    for cfg in (0, 1, 2, 3, 4):
        for n in (48, 160):
            for seed in (1, 2):
                q, lam, kmat, signs = make_instance(cfg, n=n, seed=1000 * cfg + 10 * n + seed)
                case = run_case(q, lam, kmat, signs)
                for key, v in case.items():
                    seeded[f"c{cfg}_n{n}_s{seed}__{key}"] = v
                print(f"cfg{cfg} n={n} seed={seed}: eig {case['eig_status']}, vec {case['vec_status']}")
    np.savez_compressed(os.path.join(HERE, "ref_seeded.npz"), **seeded)

    cases = {}
    # reference generator (core.cpp:117-150), mixed signs as in
    # tests/test_rootfind.cpp:163-178 (n=50, k=3)
    for t in range(25):
        seed = 2000 + t
        q, lam, kmat = ref.random_instance(50, 3, 0.4 + 0.2 * (t % 4), seed)
        signs = np.array([1, -1 if t % 2 else 1, -1 if t % 5 > 2 else 1], np.int32)
        c = run_case(q, lam, kmat, signs)
        for key in ("q", "lam", "kmat", "signs", "values", "eig_status", "lam_out", "q_out",
                    "vec_status", "tol"):
            if key in c:
                cases[f"rnd{t}__{key}"] = c[key]
    # tests/test_eigvec.cpp:133-183 style rank-2 (+1,-1) n=24
    for t in range(5):
        q, lam, kmat = ref.random_instance(24, 2, 1.0, 6000 + t)
        signs = np.array([1, -1], np.int32)
        c = run_case(q, lam, kmat, signs, tol=1e-13)
        for key in ("q", "lam", "kmat", "signs", "values", "eig_status", "lam_out", "q_out",
                    "vec_status", "tol"):
            if key in c:
                cases[f"r2_{t}__{key}"] = c[key]
    np.savez_compressed(os.path.join(HERE, "ref_cases.npz"), **cases)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
