"""Run one rank problem (after a warm-up run) — the target command for ncu captures.
Usage: python tools/profile_one.py d dprime kernel N [reps]"""
import sys

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402

d = int(sys.argv[1])
dp = None if sys.argv[2] in ("far", "None", "-1") else int(sys.argv[2])
kname = sys.argv[3]
n = int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
seed = hb.problem_seed(0, d, dp, n)
with hb.Context(0) as ctx:
    for _ in range(reps):
        r = ctx.rank(hb.make_kernel(kname), hb.make_pair(d, dp, n, hb.UNIFORM, seed), [1e-12])[0]
    print(f"rank {r.rank} k={r.k_factored} sec={[round(s, 4) for s in r.sec]}", flush=True)
