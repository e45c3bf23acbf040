"""Freeze the reference's own ACA (aca.hpp compress + apply, compiled in place from
/root/reference by oracle/Makefile into oracle/_ref/libhb_ref.so) on tests/golden/aca_cases.py
into tests/golden/aca_golden.json, so parity can be checked where /root/reference is absent.
Usage: python tests/golden/make_aca_golden.py"""
import ctypes
import json
import math
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE))
from aca_cases import CASES, case_block, case_points, case_q  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    O.build()
    out = []
    for case in CASES:
        name, d, dp, kern, nt, ns, seed, blk, eps, mr, shift, sc = case
        x, y = case_points(O, case)
        rb, rows, cb, cols = case_block(case)
        q = case_q(case)
        try:
            a = O.aca_compress(O.KERNEL_IDS[kern], x, y, eps, mr, rb, rows, cb, cols, q=q, impl="ref")
        except O.OracleError as e:
            out.append({"name": name, "status": e.status})
            continue
        O.aca_compress(O.KERNEL_IDS[kern], x, y, eps, mr, rb, rows, cb, cols)  # for the path only
        path = ctypes.c_int.in_dll(O.lib(), "hbo_aca_last_path").value
        out.append({
            "name": name, "status": 0, "rank": a.rank, "met": a.met, "oracle_path": path,
            "sigma": a.sigma.tolist(), "tau": a.tau.tolist(),
            "L_fsum": math.fsum(a.L.ravel(order="F")).hex(),
            "U_fsum": math.fsum(a.U.ravel(order="F")).hex(),
            "U_diag": [float(v).hex() for v in a.U.diagonal()],
            "b": [float(v).hex() for v in a.b],
        })
        print(name, a.rank, a.met)
    # singular: log r without a diagonal on coincident points -> runtime_error (kernel.hpp:152)
    x, _ = case_points(O, CASES[0])
    try:
        O.aca_compress(O.KERNEL_IDS["log_r"], x, x, 1e-8, 10, has_diag=False, impl="ref")
        st = 0
    except O.OracleError as e:
        st = e.status
    out.append({"name": "singular_self_log_nodiag", "status": st})
    (HERE / "aca_golden.json").write_text(json.dumps(out, indent=0))


if __name__ == "__main__":
    main()
