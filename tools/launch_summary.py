"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): time share per kernel.
Usage: python tools/launch_summary.py launches.csv [top]"""
import collections
import csv
import re
import sys


def load(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
        name = re.sub(r"<.*", "", name).replace("hb::", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        rows.append((name, v * scale))
    return rows


def main():
    rows = load(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for n, ms in rows:
        tot[n] += ms
        cnt[n] += 1
    all_ms = sum(tot.values())
    print(f"{len(rows)} launches, {all_ms:.1f} ms total")
    for n, ms in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        print(f"{n:34s} {ms:9.2f} ms {100 * ms / all_ms:5.1f}%  n={cnt[n]:6d} avg={1e3 * ms / cnt[n]:8.1f} us")


if __name__ == "__main__":
    main()
