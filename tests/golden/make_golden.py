"""Generates the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists and
`make -C oracle ref` has built oracle/_ref/libeigmod_ref.so):

    python tests/golden/make_golden.py

Writes tests/golden/ref_seeded.npz, ref_cases.npz, ref_locate.npz and
ref_validation.npz (`--only-locate` / `--only-validation` rewrite one alone). Inputs
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


def _truth_counts(q, lam, kmat, signs, dp):
    """Eigenvalues of A' = Q diag(lam) Q^T + K J K^T per open interval of the
    deflated poles (the check of tests/test_locate.cpp: classify_intervals over
    oracle_eigenvalues), by LAPACK. Eigenvalues of deflated pairs (unchanged
    and collided poles, which leave the secular coefficients) are removed,
    each as the eigenvalue nearest its pole."""
    poles = dp["poles"]
    a = (q * lam) @ q.T + (kmat * np.asarray(signs, float)) @ kmat.T
    ev = list(np.linalg.eigvalsh(0.5 * (a + a.T)))
    for i in list(dp["unchanged"]) + list(dp["collided"]):
        ev.pop(int(np.argmin(np.abs(np.asarray(ev) - lam[i]))))
    ev = np.asarray(ev)
    edges = np.concatenate([[-np.inf], poles, [np.inf]])
    return np.array([int(((ev > edges[i]) & (ev < edges[i + 1])).sum())
                     for i in range(len(poles) + 1)], np.int64)


def make_locate():
    """Location-vector fixtures (CLI locate path, tools/eigmod.cpp:143-161),
    instance families of tests/test_locate.cpp:80-200 plus a random mixed-sign
    family: inputs (lam, u, signs), the reference's counts (or its error) and
    the LAPACK interval counts."""
    out = {}
    idx = 0

    def add(q, lam, kmat, signs, family):
        nonlocal idx
        signs = np.asarray(signs, np.int32)
        u = ref.transform_update(q, lam, kmat, signs)
        dp = ref.deflate_problem(lam, u, signs)
        try:
            counts = np.array(ref.locate_from_u(lam, u, signs), np.int64)
            status = "ok"
        except Exception as e:  # the reference's own failure, recorded
            counts = np.zeros(0, np.int64)
            status = f"{type(e).__name__}: {e}"
        key = f"L{idx}"
        out[key + "__lam"] = lam
        out[key + "__u"] = u
        out[key + "__signs"] = signs
        out[key + "__ref"] = counts
        out[key + "__status"] = np.array(status)
        out[key + "__truth"] = _truth_counts(q, lam, kmat, signs, dp)
        out[key + "__family"] = np.array(family)
        idx += 1

    kinds = {"double_right": [1, 1], "double_left": [-1, -1], "mixed": [1, -1]}
    for ki, (kind, sg) in enumerate(kinds.items()):  # test_locate.cpp:80-115
        for seed in range(0, 100, 4):
            q, lam, kmat = ref.random_instance(4, 2, 0.9, seed * 3 + ki)
            add(q, lam, kmat, sg, "rank2_" + kind)
    q, lam, kmat = ref.random_instance(5, 1, 0.8, 31)  # :156-165
    add(q, lam, kmat, [1], "rank1_classic")
    for seed in range(40):  # :167-181
        q, lam, kmat = ref.random_instance(10, 3, 1.2, seed + 70)
        add(q, lam, kmat, [1, -1 if seed % 2 else 1, 1 if seed % 3 else -1], "rank3")
    for seed in range(0, 60, 2):  # :183-200 sizes
        n = 4 + seed % 17
        sg = list(kinds.values())[seed % 3]
        q, lam, kmat = ref.random_instance(n, 2, 0.8 + 0.05 * (seed % 5), seed + 1300)
        add(q, lam, kmat, sg, "rank2_sizes")
    rng = np.random.default_rng(170600773)
    for t in range(40):  # random mixed signs, n <= 60, k <= 6
        n, k = int(rng.integers(6, 61)), int(rng.integers(1, 7))
        q, lam, kmat = ref.random_instance(n, k, float(rng.uniform(0.2, 3.0)), 7000 + t)
        add(q, lam, kmat, rng.choice([-1, 1], k), "mixed_random")
    q, lam, kmat = ref.random_instance(5, 1, 0.8, 31)  # null update
    add(q, lam, np.zeros_like(kmat), [1], "null_update")
    np.savez_compressed(os.path.join(HERE, "ref_locate.npz"), **out)
    print("locate fixtures:", idx)


def make_validation():
    """reconstruct / apply_update / ortho_error fixtures (core.hpp:11-14,
    kernels.hpp:36) from the reference, on its own generator's instances."""
    out = {}
    for t, (n, k) in enumerate([(7, 2), (40, 3), (96, 5), (130, 8)]):
        q, lam, kmat = ref.random_instance(n, k, 0.7, 8100 + t)
        signs = np.array([1 if r % 3 else -1 for r in range(k)], np.int32)
        a = ref.reconstruct(q, lam)
        out[f"V{t}__q"], out[f"V{t}__lam"], out[f"V{t}__kmat"] = q, lam, kmat
        out[f"V{t}__signs"] = signs
        out[f"V{t}__reconstruct"] = a
        out[f"V{t}__apply_update"] = ref.apply_update(a, kmat, signs)
        out[f"V{t}__ortho_q"] = np.array(ref.ortho_error(q))
        rect = q[:, : max(1, n // 3)] * 1.0000001
        out[f"V{t}__rect"] = rect
        out[f"V{t}__ortho_rect"] = np.array(ref.ortho_error(rect))
    np.savez_compressed(os.path.join(HERE, "ref_validation.npz"), **out)
    print("validation fixtures:", len(out) // 9)


def main():
    if "--only-locate" in sys.argv:
        make_locate()
        return
    if "--only-validation" in sys.argv:
        make_validation()
        return
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
    make_locate()
    make_validation()
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
