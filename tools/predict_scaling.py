"""Predicted 2/4/8-GPU time of the full sweep (configs[4]) from 1-GPU measurements (only one GPU
is available to this build): every rank's share (hb_partition, the LPT split bench.py uses under
torchrun) is run as its own hb_sweep call on cuda:0, exactly what that rank would run on its own
GPU, and the job time is the max over shares.  Efficiency = T(1) / (N * max_share T).
Usage: python tools/predict_scaling.py [out.json] [N ...]   (default N = 2 4 8)"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2209_05819_b200 as hb  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/predict_scaling.json"
ns = [int(v) for v in sys.argv[2:]] or [2, 4, 8]
wl = bench.workload("sweep")
probs = bench.to_problems(hb, wl)
entries = sum(w[3] ** 2 for w in wl)


def run(idx):
    sub = [probs[i] for i in idx]
    res, st, ds = hb.sweep(sub, [0], with_times=True)
    assert all(s == 0 for s in st), st
    return ds[0], [[x.rank for x in r] for r in res]


hb.sweep(probs[:40], [0])  # warm-up: module load, pools
t1, ranks1 = run(range(len(probs)))
rec = {"workload": "configs[4] sweep, 294 problems", "t1_s": t1, "g_entries_s_1": entries / t1 / 1e9,
       "predicted": []}
print(f"N=1: {t1:.2f} s", flush=True)
for n in ns:
    own = hb.partition(probs, n)
    shares = []
    for r in range(n):
        idx = [i for i, o in enumerate(own) if o == r]
        t, rk = run(idx)
        assert rk == [ranks1[i] for i in idx], "ranks changed with the partition"
        shares.append({"rank": r, "problems": len(idx), "seconds": t,
                       "largest_N": max(wl[i][3] for i in idx)})
        print(f"N={n} share {r}: {len(idx)} problems {t:.2f} s", flush=True)
    tmax = max(s["seconds"] for s in shares)
    rec["predicted"].append({"n_gpus": n, "job_s": tmax, "g_entries_s": entries / tmax / 1e9,
                             "efficiency": t1 / (n * tmax), "shares": shares})
    print(f"N={n}: job {tmax:.2f} s, efficiency {t1 / (n * tmax):.3f}", flush=True)
json.dump(rec, open(out, "w"), indent=1)
