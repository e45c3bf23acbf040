"""Top SASS instructions by warp-stall samples from an ncu report.
Usage: python tools/ncu_hot.py report.ncu-rep [top] [context]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, ln in enumerate(lines) if ln.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
print(f"{len(rows)} instructions, {tot} samples")
order = sorted(range(len(rows)), key=lambda i: -int(rows[i]["Warp Stall Sampling (All Samples)"] or 0))
shown = set()
for i in order[:top]:
    for j in range(max(0, i - ctx), min(len(rows), i + ctx + 1)):
        if j in shown:
            continue
        shown.add(j)
        r = rows[j]
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        print(f"{j:5d} {100 * s / tot:5.1f}% ex={r['Instructions Executed']:>8s} {r['Source'].strip()}")
    if ctx:
        print("  --")
