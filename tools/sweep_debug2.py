"""Reproduce: 4D N=8000 problems through the concurrent small-problem path with profiling on."""
import sys
sys.path.insert(0, ".")
import bench
import paper_2209_05819_b200 as hb
wl = [w for w in bench.workload("sweep") if 4000 <= w[3] <= 8000 and w[0] == 4]
probs = bench.to_problems(hb, wl)
for rep in range(3):
    res, st, ds = hb.sweep(probs, [0], profiling=True, with_times=True)
    bad = [(w, s) for w, s in zip(wl, st) if s != 0]
    print(f"rep {rep}: {len(wl)} problems, {len(bad)} failed, device {ds[0]:.2f}s", flush=True)
    for w, s in bad[:10]:
        print("  FAIL", w, s, flush=True)
    print("  err:", hb.load().hb_last_error(None).decode(), flush=True)
