"""Per-problem breakdown of a bench workload, each problem run alone on one context
(after a warm-up): rank, k, device seconds, phase times.  Usage: python tools/c1_breakdown.py [c1|c2|c3]"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2209_05819_b200 as hb  # noqa: E402

wl = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c1")
out = []
with hb.Context(0) as ctx:
    for (d, dp, k, n, tols) in wl:
        kern = hb.make_kernel(k)
        pair = hb.make_pair(d, dp, n, hb.UNIFORM, hb.problem_seed(0, d, dp, n))
        ctx.rank(kern, pair, tols)
        ctx.set_profiling(True)
        ctx.reset_stats() if hasattr(ctx, "reset_stats") else None
        s0 = ctx.stats()
        r = ctx.rank(kern, pair, tols)[0]
        s1 = ctx.stats()
        ctx.set_profiling(False)
        ph = {kk: round(s1["phase_ms"][kk] - s0["phase_ms"][kk], 2) for kk in s1["phase_ms"]}
        row = {"d": d, "dp": dp, "k": k, "N": n, "rank": r.rank, "kf": r.k_factored,
               "ms": [round(1e3 * x, 2) for x in r.sec], "phase": ph,
               "launches": s1["launches"] - s0["launches"]}
        print(json.dumps(row), flush=True)
