#!/usr/bin/env python
"""bench.py — rank-revealed kernel entries per second on B200 (BASELINE.json metric).

Default workload "c3" = BASELINE.json configs[3]: d = 4, the unit hyper-cube against neighbours
sharing d' = 0..3 hyper-surfaces plus far-field, F = exp(-r), N in {2000, 4000, 8000, 16000,
32000, 65536} i.i.d. uniform FP64 points per cube from per-problem seeds (hb_problem_seed(0, d,
d', N)), tolerances 1e-12 and 1e-10 -> 30 problems, Σ N² = 2.8e10 entries per step.  One step =
one pass of the whole path over the config: generate points, assemble K, sketch-pivoted QR,
certify the ε-rank.  (configs[4], the 294-problem sweep, is `--workload sweep`; one sweep step
takes ~110 s, so 25 driver steps would not fit the arm's time budget — VERDICT r1 item 2.)

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c0|c1|c2|c3|sweep]

N > 1 runs under torchrun (one process per GPU, NCCL only for the final result gather).
Per-config workloads (c0..c3) scale WEAK: every rank runs the whole config on its own
independent problems (per-problem seeds from base seed = rank; rank 0's are the golden ones), so
the work per GPU is fixed and `value` = all ranks' entries / max-over-ranks device time.
The full sweep (configs[4], which BASELINE.json states as partitioned across 1/2/4/8 B200) is
LPT-partitioned over the ranks (hb_partition): total work fixed -> strong scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

NS = [1000, 2000, 4000, 8000, 16000, 32000, 65536]
KERNELS = ["log_r", "one_over_r", "exp_neg_r"]
METRIC = "rank-revealed kernel entries/sec (G/s)"
FP64_PEAK_FILE = ROOT / "profiles" / "fp64_peak_r01.json"
# c_F: FP64 flops per assembled entry (distance + sqrt + F), from the static SASS count of the
# 2-D assembly kernel (DFMA = 2 flops, DADD/DMUL = 1)
C_F = {"log_r": 84.0, "one_over_r": 76.0, "exp_neg_r": 69.0}


# BASELINE.json configs, exactly as stated there ("doubling" frozen per SURVEY.md §8(d))
CONFIGS = {
    # configs[0]: d=1, [0,1] vs [1,2] (vertex), N=1000, log r, tol 1e-12
    "c0": {"dims": {1: [0]}, "N": {1: [1000]}, "kernel": {1: "log_r"}, "tols": [1e-12]},
    # configs[1]: d=2, edge / vertex / far, N in {1000..16000}, log r, tol 1e-12
    "c1": {"dims": {2: [1, 0, None]}, "N": {2: [1000, 2000, 4000, 8000, 16000]},
           "kernel": {2: "log_r"}, "tols": [1e-12]},
    # configs[2]: d=3, face / edge / vertex / far, N = 1000..32768 doubling, 1/r, tol 1e-12
    "c2": {"dims": {3: [2, 1, 0, None]}, "N": {3: [1000, 2000, 4000, 8000, 16000, 32768]},
           "kernel": {3: "one_over_r"}, "tols": [1e-12]},
    # configs[3]: d=4, d' = 0..3 + far, N = 2000..65536 doubling, exp(-r), tol 1e-10 and 1e-12
    "c3": {"dims": {4: [0, 1, 2, 3, None]}, "N": {4: [2000, 4000, 8000, 16000, 32000, 65536]},
           "kernel": {4: "exp_neg_r"}, "tols": [1e-12, 1e-10]},
}


def workload(name: str):
    """List of (d, d', kernel, N, tols).  "sweep" = configs[4] (294 problems)."""
    probs = []
    if name == "sweep":
        for n in NS:
            for d in (1, 2, 3, 4):
                for dp in list(range(d)) + [None]:
                    for k in KERNELS:
                        probs.append((d, dp, k, n, [1e-12, 1e-10] if d == 4 else [1e-12]))
        return probs
    cfg = CONFIGS[name]
    for d, dps in cfg["dims"].items():
        for n in cfg["N"][d]:
            for dp in dps:
                probs.append((d, dp, cfg["kernel"][d], n, list(cfg["tols"])))
    return probs


def to_problems(hb, wl, base_seed: int = 0):
    return [hb.make_problem(k, d, dp, n, tols, base_seed=base_seed) for (d, dp, k, n, tols) in wl]


def alg_flops(n: int, p: int, kernel: str) -> float:
    """FLOP_alg = N²c_F + 4N²p − 4Np² + (4/3)p³."""
    return n * n * C_F[kernel] + 4.0 * n * n * p - 4.0 * n * p * p + 4.0 / 3.0 * p ** 3


def fp64_peak():
    try:
        j = json.loads(FP64_PEAK_FILE.read_text())
        return float(j["dmma_m8n8k4_tflops"]), "own probe tools/fp64_peak.cu (DMMA m8n8k4; " \
            "MEASURED_PEAKS.json has no FP64 entry)"
    except Exception:
        return 37.0, "nominal B200 FP64 (probe file missing)"


def ncu_traffic():
    """DRAM bytes (read + write) of one captured launch of the dominant DMMA GEMM, from the
    committed ncu --set full summary (profiles/<round>/dgemm_ncu_full.json), or None."""
    files = sorted(ROOT.glob("profiles/r*/dgemm_ncu_full.json"))
    if not files:
        return None, "no ncu --set full capture committed"
    try:
        j = json.loads(files[-1].read_text())["roofline_traffic_launch"]
        return int(j["dram_bytes"]), (f"{files[-1].relative_to(ROOT)}: {j['shape']}, grid {j['grid']}, "
                                      f"{j['duration_ms']:.3f} ms; algorithmic {j['algorithmic_bytes']} B")
    except Exception as e:  # noqa: BLE001
        return None, f"unreadable ncu summary: {e}"


def hbm_peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback B200_PROFILING.md"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        if os.environ.get("HB_BENCH_SMI_MS") == "0":  # experiments: no sampler
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms",
                 os.environ.get("HB_BENCH_SMI_MS", "100")],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout: float = 15.0):
        """nvidia-smi's start-up (NVML load, first query) costs host CPU for up to seconds on a
        fresh box; wait for its first sample so that cost lands before the timed region (host
        round trips of the sweep driver are inside the device-timed span)."""
        t0 = time.perf_counter()
        while self.proc and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)
        self.skip = len(self.lines)

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[getattr(self, "skip", 0):] or self.lines[-1:]:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if s > 600] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline_run(wl_sample, threads: int):
    """The reference's CPU path on a bounded sample: entries/s on the host cores.  Assembly is
    the reference's own hodlr::assemble_dense (kernel.hpp:168-181, serial as written) compiled
    from /root/reference into oracle/_ref when that library is present, else the oracle's C
    restatement on all threads; the ε-rank is LAPACK gesdd on all threads (SPEC epsilon_rank —
    the reference has no rank driver in code).  Returns (G/s, s, entries, kind)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    from oracle import oracle as O
    O.build()
    use_ref = O.ref_available()
    t0 = time.perf_counter()
    ent = 0
    for (d, dp, k, n, tols) in wl_sample:
        seed = O.problem_seed(0, d, dp, n)
        x, y = O.pair_points(d, dp, n, O.UNIFORM, seed)
        if use_ref:
            K = O.ref_assemble(O.KERNEL_IDS[k], x, y)
        else:
            K = O.assemble(O.KERNEL_IDS[k], x, y, nthreads=threads)
        s = O.singular_values(K)
        [O.epsilon_rank_from_sigma(s, t) for t in tols]
        ent += n * n
    dt = time.perf_counter() - t0
    return ent / dt / 1e9, dt, ent, ("reference" if use_ref else "port")


def _assembly_desc(kind: str, threads: int) -> str:
    return ("the reference's assemble_dense (kernel.hpp, compiled in oracle/_ref), serial"
            if kind == "reference" else f"oracle C assembly on {threads} threads")


def golden_map():
    p = ROOT / "tests" / "golden" / "baseline_ranks.json"
    if not p.exists():
        return {}
    return {(r["d"], r["dprime"], r["kernel"], r["N"]): r for r in json.loads(p.read_text())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 3; 1 for the two-minute sweep workload)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=["c0", "c1", "c2", "c3", "sweep"],
                    help="BASELINE.json configs[0..3] (c0..c3) or the full configs[4] sweep")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-max-n", type=int, default=4000,
                    help="CPU baseline sample: the workload's problems with N <= this")
    ap.add_argument("--ref-sample-max-n", type=int, default=2000,
                    help="--impl reference: per-step sample = the workload's problems with N <= this "
                         "(bounded so warmup + 25 steps fit the arm's time budget)")
    ap.add_argument("--details", default="", help="write per-problem results/stats JSON here")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 1 if args.workload == "sweep" else 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    wl = workload(args.workload)
    threads = os.cpu_count() or 1
    names = {"c0": "BASELINE.json configs[0] (d=1 vertex, log r, N=1000)",
             "c1": "BASELINE.json configs[1] (d=2 edge/vertex/far, log r, N=1000..16000)",
             "c2": "BASELINE.json configs[2] (d=3 face/edge/vertex/far, 1/r, N=1000..32768)",
             "c3": "BASELINE.json configs[3] (d=4 d'=0..3/far, exp(-r), N=2000..65536, 2 tols)",
             "sweep": "BASELINE.json configs[4] full sweep (294 problems)"}
    cfg = {"workload": names[args.workload], "problems": len(wl),
           "N": sorted({w[3] for w in wl}), "kernels": sorted({w[2] for w in wl}),
           "points": "iid uniform fp64 per cube, seed = hb_problem_seed(0, d, d', N)",
           "tol": sorted({t for w in wl for t in w[4]}),
           "entries_per_step": sum(n * n for (_, _, _, n, _) in wl),
           "l2": "inputs larger than L2: every step regenerates points and re-assembles K (sum 8N^2 = "
                 f"{8 * sum(n * n for (_, _, _, n, _) in wl) / 1e12:.2f} TB written per step)",
           "parallelism": (f"replicated config x{world} (independent seeds per rank)"
                           if args.workload != "sweep" else f"lpt-partition x{world}")}
    if args.workload != "sweep":
        cfg["entries_per_step_whole_job"] = cfg["entries_per_step"] * world
    sample = [w for w in wl if w[3] <= args.cpu_sample_max_n]

    if args.impl == "reference":
        # the reference's CPU path for this workload = the oracle port (the reference ships no
        # rank driver and needs Eigen), on a bounded sample of the same workload
        if rank != 0:
            return 0
        sample = [w for w in wl if w[3] <= args.ref_sample_max_n] or sorted(wl, key=lambda w: w[3])[:3]
        args.cpu_sample_max_n = max(w[3] for w in sample)
        for _ in range(args.warmup):
            cpu_baseline_run(sample[:3], threads)
        vals, dts = [], []
        kind = "port"
        for _ in range(args.steps):
            v, dt, ent, kind = cpu_baseline_run(sample, threads)
            vals.append(v)
            dts.append(dt)
        v = statistics.median(vals)
        line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "G entries/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(1e3 * statistics.median(dts), 1), "higher_is_better": True,
                "scaling": "strong" if args.workload == "sweep" else "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": cfg,
                "cpu_baseline": {"value": round(v, 6), "unit": "G entries/s", "cores": threads,
                                 "kind": kind,
                                 "sample": f"{len(sample)} workload problems with N <= "
                                           f"{args.cpu_sample_max_n} ({_assembly_desc(kind, threads)} "
                                           f"+ numpy/LAPACK gesdd on {threads} threads)"},
                "e2e": {"value": round(v, 6), "unit": "G entries/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import paper_2209_05819_b200 as hb
    from paper_2209_05819_b200 import dist as hbd
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
        torch.cuda.set_device(local)
    dev = local
    weak = args.workload != "sweep"
    if weak:  # every rank: the whole config on its own seeds (rank 0 = the golden seeds)
        problems = [pr for r in range(world) for pr in to_problems(hb, wl, base_seed=r)]
        mine = list(range(rank * len(wl), (rank + 1) * len(wl)))
    else:
        problems = to_problems(hb, wl)
        mine = hbd.my_share(problems, rank, world)
    my_probs = [problems[i] for i in mine]

    def barrier():
        if dist:
            dist.barrier(device_ids=[dev])
        torch.cuda.synchronize()

    clk = ClockSampler(dev)
    clk.start()
    clk.wait_first()
    for _ in range(args.warmup):
        hb.sweep(my_probs, [dev])
    hb.reset_global_stats()
    launches0 = hb.global_stats()["launches"]
    barrier()
    dev_secs, walls, my_res, statuses = [], [], None, []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        my_res, st, ds = hb.sweep(my_probs, [dev], profiling=False, with_times=True)
        walls.append(time.perf_counter() - t0)
        dev_secs.append(ds[0])
        statuses = st
    barrier()
    clocks = clk.stop()
    stats = hb.global_stats()
    launches = stats["launches"] - launches0
    # The dominant kernel (the DMMA GEMM) measured without overlap: one untimed, profiled pass of
    # this rank's costliest problem alone on one stream after the timed region — CUDA events
    # around every GEMM launch on the stream it runs on, so the GEMM time is a share of that
    # problem's device time (never more), and the phase split of the same pass.
    iso = None
    if my_probs:
        crit = max(my_probs, key=lambda p: (p.pair.n_target, p.pair.d_prime))
        hb.reset_global_stats()
        _, _, ds1 = hb.sweep([crit], [dev], profiling=True, with_times=True)
        st1 = hb.global_stats()
        if st1["gemm_ms"] > 0:
            iso = {"kernel": "dgemm (FP64 DMMA m8n8k4): trailing update, sketch, WY and "
                             "certification-QR GEMMs",
                   "achieved": round(st1["gemm_flops"] / (st1["gemm_ms"] * 1e-3) / 1e12, 3),
                   "gemm_ms": round(st1["gemm_ms"], 1), "problem_ms": round(ds1[0] * 1e3, 1),
                   "gemm_share": round(st1["gemm_ms"] / (ds1[0] * 1e3), 4),
                   "gemm_launches": st1["gemm_launches"],
                   "problem": f"d={crit.pair.target.d} d'={crit.pair.d_prime} N={crit.pair.n_target}",
                   "phase_ms": {k: round(v, 1) for k, v in st1["phase_ms"].items()},
                   "note": "untimed solo pass of the costliest problem after the timed region "
                           "(one stream, no overlap): achieved = sum 2MNK / sum of per-launch "
                           "CUDA-event times"}
    t_dev = sum(dev_secs)
    t_wall = sum(walls)
    if dist:
        tt = torch.tensor([t_dev, t_wall], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev, t_wall = tt.tolist()
        full = hbd.gather_results(problems, mine, my_res, device=torch.device("cuda", dev))
        lt = torch.tensor([launches, stats["gemm_ms"], stats["gemm_flops"]], dtype=torch.float64, device="cuda")
        dist.all_reduce(lt)
        launches, gemm_ms_all, gemm_fl_all = lt.tolist()
    else:
        full = my_res
        gemm_ms_all, gemm_fl_all = stats["gemm_ms"], stats["gemm_flops"]
    if rank != 0:
        dist.destroy_process_group()
        return 0

    entries = cfg["entries_per_step"] * (world if weak else 1)
    value = entries * args.steps / t_dev / 1e9
    e2e = entries * args.steps / t_wall / 1e9
    peak, peak_src = fp64_peak()
    # parity vs the committed oracle golden file (problems the CPU oracle could do)
    gm = golden_map()
    checked = equal = 0
    mism = []
    total_alg = 0.0
    for j, res in enumerate(full):
        d, dp, k, n, tols = wl[j % len(wl)]
        for t, r in enumerate(res):
            total_alg += alg_flops(n, r.rank, k) if t == 0 else 0.0
        g = gm.get((d, dp, k, n)) if j < len(wl) else None  # golden seeds: rank 0's copy
        if g:
            for t, r in enumerate(res):
                checked += 1
                if r.rank == g["ranks"][t]:
                    equal += 1
                else:
                    mism.append({"d": d, "dprime": dp, "kernel": k, "N": n, "tol": tols[t],
                                 "gpu": r.rank, "oracle": g["ranks"][t], "gap_oracle": g["gaps"][t],
                                 "gap_gpu": r.gap})
    uncert = sum(1 for res in full for r in res if r.certificate == 0)
    # exact-arithmetic brackets whose σ sit within the QR's rounding band of the threshold
    in_band = [{"problem": list(wl[j % len(wl)][:4]), "tol": wl[j % len(wl)][4][t], "gap": r.gap,
                "fp_band": r.fp_band} for j, res in enumerate(full) for t, r in enumerate(res)
               if r.gap < r.fp_band]
    prob_cert = sum(1 for res in full for r in res if r.certificate == 2)
    path_tf = total_alg * args.steps / t_dev / 1e12
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "G entries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t_dev / args.steps, 1),
        "higher_is_better": True, "scaling": "weak" if weak else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": cfg,
        "e2e": {"value": round(e2e, 4), "unit": "G entries/s",
                "h2d_bytes_per_step": len(problems) * __import__("ctypes").sizeof(hb.hb_problem),
                "d2h_bytes_per_step": sum(p.ntol for p in problems) * __import__("ctypes").sizeof(hb.hb_rank_result),
                "note": "whole job (all ranks)",
                "api": "hb_sweep_ex (C ABI) from host descriptors to host result records; points are "
                       "generated on device from the seeds (k1)"},
        "roofline": {
            "bound": "tensor", "achieved": round(path_tf, 3), "peak": peak, "unit": "TFLOP/s",
            "frac": round(path_tf / peak, 4), "traffic": ncu_traffic()[0],
            "scope": "north-star path fraction: FLOP_alg per step / device time per step / FP64 "
                     "peak, FLOP_alg = sum over problems of N^2 c_F + 4N^2 p - 4N p^2 + 4/3 p^3 "
                     "(SURVEY.md 8(d), p = certified rank)",
            "peak_source": peak_src, "traffic_source": ncu_traffic()[1],
            "kernel": (dict(iso, peak=peak, frac=round(iso["achieved"] / peak, 4)) if iso else None)},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "parity": {"checked_vs_oracle": checked, "equal": equal, "mismatches": mism[:20],
                   "uncertified_brackets": uncert, "probabilistic_certificates": prob_cert,
                   "rounding_sensitive": {"count": len(in_band), "cases": in_band[:10],
                                          "rule": "gap < fp_band = sqrt(N) u ||A||_F / thr"},
                   "statuses_ok": all(s == 0 for s in statuses),
                   "failed": [[list(w[:4]), s] for w, s in zip([wl[i % len(wl)] for i in mine], statuses) if s != 0][:10],
                   "last_error": hb.load().hb_last_error(None).decode()[:200]},
    }
    if world == 1 and not args.no_cpu_baseline:
        v, dt, ent, kind = cpu_baseline_run(sample, threads)
        line["cpu_baseline"] = {"value": round(v, 6), "unit": "G entries/s", "cores": threads,
                                "kind": kind,
                                "sample": f"{len(sample)} workload problems with N <= "
                                          f"{args.cpu_sample_max_n} ({dt:.1f} s; {_assembly_desc(kind, threads)} "
                                          f"+ numpy/LAPACK gesdd on {threads} threads)"}
    if args.details:
        Path(args.details).write_text(json.dumps({
            "results": [[r.__dict__ for r in res] for res in full], "workload": wl,
            "stats": stats, "dev_secs": dev_secs, "walls": walls}, default=str))
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
