"""Solo device time of every problem of the sweep (configs[4]) on cuda:0, one hb_sweep call per
problem (no other problem in flight), for calibrating the LPT cost model of hb_partition.
Usage: python tools/solo_all.py out.json [max_N]"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2209_05819_b200 as hb  # noqa: E402

out = sys.argv[1]
max_n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 30
wl = [w for w in bench.workload("sweep") if w[3] <= max_n]
probs = bench.to_problems(hb, wl)
hb.sweep(probs[:20], [0])  # warm-up
recs = []
for w, p in zip(wl, probs):
    best = None
    for rep in range(2 if w[3] <= 16000 else 1):
        res, st, ds = hb.sweep([p], [0], with_times=True)
        assert st[0] == 0
        best = ds[0] if best is None else min(best, ds[0])
    r = res[0]
    recs.append({"d": w[0], "dprime": w[1], "kernel": w[2], "N": w[3], "ntol": len(w[4]),
                 "ranks": [x.rank for x in r], "k": r[0].k_factored, "device_s": best})
    print(json.dumps(recs[-1]), flush=True)
json.dump(recs, open(out, "w"))
print("sum", sum(r["device_s"] for r in recs))
