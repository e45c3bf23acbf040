"""Solo time of one rank problem on cuda:0 (one warm-up, then timed reps), with the per-phase
device-time split.  Usage: python tools/solo.py d dprime kernel N [reps] [tols...]"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402

d = int(sys.argv[1])
dp = None if sys.argv[2] in ("far", "None", "-1") else int(sys.argv[2])
kname, n = sys.argv[3], int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
tols = [float(t) for t in sys.argv[6:]] or ([1e-12, 1e-10] if d == 4 else [1e-12])
prob = hb.make_problem(kname, d, dp, n, tols)
hb.sweep([prob], [0])  # warm-up (allocations, module load)
for it in range(reps):
    hb.reset_global_stats()
    t0 = time.perf_counter()
    res, st, ds = hb.sweep([prob], [0], profiling=(it == reps - 1), with_times=True)
    wall = time.perf_counter() - t0
    r = res[0]
    print(json.dumps({"problem": [d, dp, kname, n], "ranks": [x.rank for x in r],
                      "k": r[0].k_factored, "device_s": round(ds[0], 4), "wall_s": round(wall, 4),
                      "cert": [x.certificate for x in r], "gaps": [x.gap for x in r],
                      "sec": [round(s, 4) for s in r[0].sec], "status": st[0]}), flush=True)
st = hb.global_stats()
print(json.dumps({"phase_ms": {k: round(v, 1) for k, v in st["phase_ms"].items()},
                  "gemm_ms": round(st["gemm_ms"], 1),
                  "gemm_tflops": round(st["gemm_flops"] / max(st["gemm_ms"], 1e-9) / 1e9, 2)}))
