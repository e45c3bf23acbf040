"""Generate tests/golden/baseline_ranks.json: CPU-oracle ε-ranks of the BASELINE sweep problems.

Problems (BASELINE.json configs): d = 1..4, every d' in {0..d-1} plus far-field,
kernels {log_r, one_over_r, exp_neg_r}, i.i.d. uniform points from the per-problem seed
problem_seed(0, d, d', N), tolerances 1e-12 (and 1e-10 for d = 4).  Ranks come from the oracle
(oracle/oracle.py: C entry restatement + LAPACK gesdd); every record stores σ₁, σ_p, σ_{p+1}
and the boundary gap so that a GPU mismatch can be judged against it.

Usage: python tests/golden/make_baseline_ranks.py [max_N] [d:kernel]
  (default 4000; 8000 takes ~1 h on 8 cores; "2:log_r" restricts to one dimension and kernel,
  used for the configs[1] N = 16000 entries)
Runs anywhere the oracle builds (no GPU, no /root/reference needed); results are merged into the
existing JSON so larger N can be added incrementally.
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

OUT = Path(__file__).with_name("baseline_ranks.json")
KERNELS = ["log_r", "one_over_r", "exp_neg_r"]
NS = [1000, 2000, 4000, 8000, 16000, 32000, 65536]


def geometries():
    for d in range(1, 5):
        for dp in list(range(d)) + [None]:
            yield d, dp


def main() -> int:
    max_n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
    only = sys.argv[2].split(":") if len(sys.argv) > 2 else None
    recs = json.loads(OUT.read_text()) if OUT.exists() else []
    have = {(r["d"], r["dprime"], r["kernel"], r["N"]) for r in recs}
    for n in [x for x in NS if x <= max_n]:
        for d, dp in geometries():
            seed = O.problem_seed(0, d, dp, n)
            x, y = O.pair_points(d, dp, n, O.UNIFORM, seed)
            if only and d != int(only[0]):
                continue
            for kname in KERNELS:
                if only and kname != only[1]:
                    continue
                if (d, dp, kname, n) in have:
                    continue
                tols = [1e-12, 1e-10] if d == 4 else [1e-12]
                t0 = time.time()
                K = O.assemble(O.KERNEL_IDS[kname], x, y, nthreads=os.cpu_count() or 1)
                s = O.singular_values(K)
                rr = [O.epsilon_rank_from_sigma(s, t) for t in tols]
                recs.append({
                    "d": d, "dprime": dp, "kernel": kname, "N": n, "seed": seed,
                    "tols": tols, "ranks": [r.rank for r in rr], "sigma1": rr[0].sigma1,
                    "sigma_r": [r.sigma_r for r in rr], "sigma_r1": [r.sigma_r1 for r in rr],
                    "gaps": [r.gap for r in rr], "oracle": "numpy.linalg.svd (LAPACK gesdd)",
                    "seconds": round(time.time() - t0, 2),
                })
                print(f"d={d} dp={dp} {kname} N={n}: ranks {[r.rank for r in rr]} "
                      f"gaps {[f'{r.gap:.1e}' for r in rr]} {time.time() - t0:.1f}s", flush=True)
                OUT.write_text(json.dumps(recs, indent=0) + "\n")
    OUT.write_text(json.dumps(recs, indent=0) + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
