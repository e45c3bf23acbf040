"""Generate tests/golden/baseline_ranks.json: CPU-oracle ε-ranks of the BASELINE sweep problems.

Problems (BASELINE.json configs): d = 1..4, every d' in {0..d-1} plus far-field,
kernels {log_r, one_over_r, exp_neg_r}, i.i.d. uniform points from the per-problem seed
problem_seed(0, d, d', N), tolerances 1e-12 (and 1e-10 for d = 4).  Ranks come from the oracle
(oracle/oracle.py: C entry restatement + LAPACK gesdd); every record stores σ₁, σ_p, σ_{p+1}
and the boundary gap so that a GPU mismatch can be judged against it.

Large N (``--certified``): the full SVD is O(N³), so N ≥ 16000 problems use the certified
truncated route of oracle/certified.py (LAPACK dgeqp3rk + dgesdd on R_k + Weyl bracket with
δ = ‖A22‖_F), in the priority order of ``certified_plan()`` (configs[2], configs[3], the sweep at
N = 16000, then the large-N problems by predicted cost).  ``--validate`` first re-derives a few
N = 8000 full-SVD records through the certified route (tests/golden/certified_validation.json).

Usage: python tests/golden/make_baseline_ranks.py [max_N] [d:kernel]
       python tests/golden/make_baseline_ranks.py --certified [--validate] [--max-cost SECONDS] [--c3-first]
              [--skip-c3] [--out FILE] [--deadline SECONDS]
       python tests/golden/make_baseline_ranks.py --merge FILE
  (default 4000; 8000 takes ~1 h on 8 cores; "2:log_r" restricts to one dimension and kernel,
  used for the configs[1] N = 16000 entries)
Runs anywhere the oracle builds (no GPU, no /root/reference needed); results are merged into the
existing JSON so larger N can be added incrementally.
"""
import json
import math
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


def predicted_rank(recs, d, dp, kname, n, tol_index=0):
    """p̂(N) extrapolated from the largest two full-SVD N (geometric growth per doubling)."""
    byn = {r["N"]: r["ranks"][tol_index] for r in recs
           if (r["d"], r["dprime"], r["kernel"]) == (d, dp, kname) and r["N"] <= 8000}
    n1, n2 = sorted(byn)[-2:]
    g = max(1.0, byn[n2] / max(1, byn[n1])) ** (1.0 / math.log2(n2 / n1))
    return byn[n2] * g ** math.log2(n / n2)


def certified_plan(recs):
    """Problems for the certified route, in priority order (VERDICT r1 'do this' 1)."""
    plan = []
    c2 = [(3, dp, "one_over_r", n) for n in (16000, 32768) for dp in (2, 1, 0, None)]
    c3_16 = [(4, dp, "exp_neg_r", 16000) for dp in (3, 2, 1, 0, None)]
    sw16 = [(d, dp, k, 16000) for d, dp in geometries() for k in KERNELS]
    c3_32 = [(4, dp, "exp_neg_r", 32000) for dp in (3, 2, 1, 0, None)]
    large = [(d, dp, k, n) for n in (32000, 65536) for d, dp in geometries() for k in KERNELS]
    cost = lambda p: p[3] ** 2 * 1.4 * predicted_rank(recs, *p)
    low = sorted([p for p in large if predicted_rank(recs, *p) <= 2000], key=cost)
    rest = sorted([p for p in large if p not in low], key=cost)
    for p in c2 + sorted(c3_16, key=cost) + sorted(sw16, key=cost) + low + c3_32 + rest:
        if p not in plan:
            plan.append(p)
    return plan


def certified_record(d, dp, kname, n, nthreads):
    from oracle import certified as C
    seed = O.problem_seed(0, d, dp, n)
    tols = [1e-12, 1e-10] if d == 4 else [1e-12]
    t0 = time.time()
    x, y = O.pair_points(d, dp, n, O.UNIFORM, seed)
    K = O.assemble(O.KERNEL_IDS[kname], x, y, nthreads=nthreads)
    ta = time.time() - t0
    c = C.certified_rank(K, tols)
    del K
    return {
        "d": d, "dprime": dp, "kernel": kname, "N": n, "seed": seed, "tols": tols,
        "ranks": c.ranks, "rank_lo": c.rank_lo, "rank_hi": c.rank_hi, "sigma1": c.sigma1,
        "sigma_r": c.sigma_r, "sigma_r1": c.sigma_r1, "gaps": c.gaps, "k": c.k,
        "delta_F": c.delta_F, "fp_band": c.fp_band, "in_fp_band": c.in_fp_band,
        "oracle": "certified: LAPACK dgeqp3rk (truncated) + dgesdd on R_k, Weyl bracket "
                  "delta = ||A22||_F (oracle/certified.py)",
        "seconds": round(time.time() - t0, 2),
        "phase_s": {"assemble": round(ta, 2), **{k: round(v, 2) for k, v in c.seconds.items()}},
    }


def main_certified(argv) -> int:
    nthreads = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    recs = json.loads(OUT.read_text())
    if "--validate" in argv:
        vout = OUT.with_name("certified_validation.json")
        vals = json.loads(vout.read_text()) if vout.exists() else []
        done = {(v["d"], v["dprime"], v["kernel"], v["N"]) for v in vals}
        for key in [(4, 3, "one_over_r", 8000), (3, 2, "log_r", 8000), (2, 1, "one_over_r", 8000),
                    (4, 0, "exp_neg_r", 8000), (4, None, "log_r", 8000)]:
            if key in done:
                continue
            full = next(r for r in recs if (r["d"], r["dprime"], r["kernel"], r["N"]) == key)
            c = certified_record(*key, nthreads)
            c["full_svd_ranks"] = full["ranks"]
            c["equal"] = c["ranks"] == full["ranks"] and c["rank_lo"] == c["rank_hi"]
            vals.append(c)
            print(f"validate {key}: certified {c['ranks']} full {full['ranks']} k={c['k']} "
                  f"{c['seconds']}s", flush=True)
            vout.write_text(json.dumps(vals, indent=0) + "\n")
    max_cost = float(argv[argv.index("--max-cost") + 1]) if "--max-cost" in argv else math.inf
    # --out FILE: append the new records to FILE instead of the tracked fixture (a second machine
    # working on another part of the plan; merge with --merge FILE afterwards)
    out = Path(argv[argv.index("--out") + 1]) if "--out" in argv else OUT
    deadline = time.time() + float(argv[argv.index("--deadline") + 1]) if "--deadline" in argv else math.inf
    plan = certified_plan(recs)
    c3 = [k for k in plan if k[0] == 4 and k[2] == "exp_neg_r"]
    if "--c3-first" in argv:  # the bench default's own problems (configs[3]) before the rest
        plan = c3 + [k for k in plan if k not in c3]
    if "--skip-c3" in argv:
        plan = [k for k in plan if k not in c3]
    for key in plan:
        recs = json.loads(OUT.read_text())
        extra = json.loads(out.read_text()) if out != OUT and out.exists() else []
        if any((r["d"], r["dprime"], r["kernel"], r["N"]) == key for r in recs + extra):
            continue
        est = 4.0 * key[3] ** 2 * 1.4 * predicted_rank(recs, *key) / 20e9
        if est > max_cost:
            print(f"skip {key}: predicted {est:.0f}s > {max_cost}", flush=True)
            continue
        if time.time() + 1.3 * est > deadline:
            print(f"skip {key}: predicted {est:.0f}s would pass the deadline", flush=True)
            continue
        rec = certified_record(*key, nthreads)
        if out == OUT:
            recs = json.loads(OUT.read_text())
            recs.append(rec)
            OUT.write_text(json.dumps(recs, indent=0) + "\n")
        else:
            extra = json.loads(out.read_text()) if out.exists() else []
            extra.append(rec)
            out.write_text(json.dumps(extra, indent=0) + "\n")
        print(f"{key}: ranks {rec['ranks']} [{rec['rank_lo']}, {rec['rank_hi']}] k={rec['k']} "
              f"gaps {[f'{g:.1e}' for g in rec['gaps']]} {rec['seconds']}s {rec['phase_s']}",
              flush=True)
    return 0


def main_merge(path) -> int:
    """Merge records produced elsewhere with --out into the tracked fixture (no duplicates)."""
    recs = json.loads(OUT.read_text())
    have = {(r["d"], r["dprime"], r["kernel"], r["N"]) for r in recs}
    new = [r for r in json.loads(Path(path).read_text())
           if (r["d"], r["dprime"], r["kernel"], r["N"]) not in have]
    OUT.write_text(json.dumps(recs + new, indent=0) + "\n")
    print(f"merged {len(new)} records -> {len(recs) + len(new)}")
    return 0


def main() -> int:
    if "--merge" in sys.argv:
        return main_merge(sys.argv[sys.argv.index("--merge") + 1])
    if "--certified" in sys.argv:
        return main_certified(sys.argv)
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
