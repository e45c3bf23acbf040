"""Generate tests/golden/hodlr_golden.json: the reference's own HMatrix::initialize + matvec
(hmatrix.hpp:50-179, cluster_tree.hpp) compiled in place into oracle/_ref, on seeded point clouds
(oracle points: SplitMix64 uniform, regenerated bit-identically on the GPU box) and seeded
Gaussian vectors — fixtures for tests/test_gpu_hmatrix.py, where /root/reference does not exist.

Usage: python tests/golden/make_hodlr_golden.py   (needs oracle/_ref, i.e. /root/reference)
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

OUT = Path(__file__).with_name("hodlr_golden.json")
# (d, N, kernel, policy, n_max, eps, point seed)
CASES = [
    (1, 2000, "log_r", "weakdd", 64, 1e-8, 11),
    (2, 3000, "log_r", "weakdd", 100, 1e-8, 7),
    (2, 2500, "one_over_r", "strong", 80, 1e-6, 3),
    (2, 2500, "exp_neg_r", "weakall", 80, 1e-10, 5),
    (3, 2000, "one_over_r", "weakdd", 60, 1e-6, 9),
]


def main():
    O.build()
    out = {"source": "hmatrix.hpp / cluster_tree.hpp compiled in oracle/_ref", "cases": []}
    for (d, n, kname, pol, nmax, eps, seed) in CASES:
        x = O.points(d, [0.0] * d, 1.0, n, O.UNIFORM, seed, 0)
        q = np.random.default_rng(seed).standard_normal((n, 2))
        b, rep, perm = O.ref_hmatrix_matvec(O.KERNEL_IDS[kname], x, [0.0] * d, 1.0, pol, nmax, eps, q)
        K = O.assemble(O.KERNEL_IDS[kname], x, x, nthreads=8)
        err = float(np.linalg.norm(K @ q - b) / np.linalg.norm(K @ q))
        out["cases"].append({"d": d, "N": n, "kernel": kname, "policy": pol, "n_max": nmax, "eps": eps,
                             "seed": seed, "report": rep, "perm": perm.tolist(), "b": b.tolist(),
                             "rel_err_vs_dense": err})
        print(d, n, kname, pol, rep, f"{err:.2e}", flush=True)
    OUT.write_text(json.dumps(out) + "\n")
    print(OUT, OUT.stat().st_size)


if __name__ == "__main__":
    main()
