"""Run a subset of the sweep through hb_sweep_ex and print per-problem status / errors."""
import sys
sys.path.insert(0, ".")
import bench
import paper_2209_05819_b200 as hb
maxn = int(sys.argv[1]) if len(sys.argv) > 1 else 8000
minn = int(sys.argv[2]) if len(sys.argv) > 2 else 8000
wl = [w for w in bench.workload("sweep") if minn <= w[3] <= maxn]
probs = bench.to_problems(hb, wl)
for rep in range(2):
    res, st, ds = hb.sweep(probs, [0], with_times=True)
    bad = [(w, s) for w, s in zip(wl, st) if s != 0]
    print(f"rep {rep}: {len(wl)} problems, {len(bad)} failed, device {ds[0]:.2f}s", flush=True)
    for w, s in bad[:10]:
        print("  FAIL", w, s, flush=True)
print(hb.load().hb_last_error(None).decode())
