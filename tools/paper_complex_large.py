"""The paper's complex F3 / F4 columns at larger N on the GPU (hb_rank_complex) against the
published tables.  Usage: python tools/paper_complex_large.py [max_n]"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402

max_n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
tabs = json.load(open("tests/golden/paper_tables.json"))
cols = {"F3": ("helmholtz3d_re", "helmholtz3d_im"), "F4": ("hankel_h12_re", "hankel_h12_im")}
ok = bad = 0
with hb.Context(0) as ctx:
    for tab in tabs:
        for row in tab["rows"]:
            if not (5000 < row["N"] <= max_n):
                continue
            for col, (kre, kim) in cols.items():
                want = row["ranks"][tab["columns"].index(col)]
                mode = hb.GRID_CLOSED if tab["dprime"] is None else hb.GRID_INTERIOR
                t = time.perf_counter()
                r = ctx.rank_complex(hb.make_kernel(kre), hb.make_kernel(kim),
                                     hb.make_pair(tab["d"], tab["dprime"], row["N"], mode, 0), [1e-12])[0]
                dt = time.perf_counter() - t
                good = r.rank == want
                ok += good
                bad += not good
                print(json.dumps({"table": tab["label"], "N": row["N"], "col": col, "paper": want,
                                  "gpu": r.rank, "cert": r.certificate, "gap": r.gap, "s": round(dt, 2)}),
                      flush=True)
print(f"{ok} equal, {bad} different")
