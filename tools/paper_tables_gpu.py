"""Every published rank of the paper's 14 tables (tests/golden/paper_tables.json)
recomputed on the GPU: real columns F1, F2, F5-F8 by hb_rank, complex F3 / F4 by hb_rank_complex
(real embedding), ε = 1e-12, interior grid near-field / closed grid far-field.
Usage: python tools/paper_tables_gpu.py [max_n [min_n]] > log   (JSON line per value, summary last)"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402

max_n = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
min_n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tabs = json.load(open("tests/golden/paper_tables.json"))
cplx = {"F3": ("helmholtz3d_re", "helmholtz3d_im"), "F4": ("hankel_h12_re", "hankel_h12_im")}
ok = bad = 0
mism = []
with hb.Context(0) as ctx:
    for tab in tabs:
        for row in tab["rows"]:
            if row["N"] > max_n or row["N"] <= min_n:
                continue
            mode = hb.GRID_CLOSED if tab["dprime"] is None else hb.GRID_INTERIOR
            pair = hb.make_pair(tab["d"], tab["dprime"], row["N"], mode, 0)
            for col, kname, want in zip(tab["columns"], tab["kernels"], row["ranks"]):
                t = time.perf_counter()
                if col in cplx:
                    r = ctx.rank_complex(hb.make_kernel(cplx[col][0]), hb.make_kernel(cplx[col][1]),
                                         pair, [1e-12])[0]
                else:
                    r = ctx.rank(hb.make_kernel(kname), pair, [1e-12])[0]
                good = r.rank == want
                ok += good
                bad += not good
                rec = {"table": tab["label"], "N": row["N"], "col": col, "paper": want, "gpu": r.rank,
                       "cert": r.certificate, "gap": r.gap, "s": round(time.perf_counter() - t, 2)}
                if not good:
                    mism.append(rec)
                print(json.dumps(rec), flush=True)
print(json.dumps({"summary": {"min_n": min_n, "max_n": max_n, "equal": ok, "different": bad, "mismatches": mism}}))
