"""Generate tests/golden/cheb_golden.json: the reference's own interpolation_decay
(chebyshev.hpp:151-177), chebyshev_nodes, fit_decay_rate and v_d_constant, compiled in place into
oracle/_ref, on seeded target clouds separated from the interpolation cube — fixtures for the GPU
test (tests/test_gpu_chebyshev.py), where /root/reference does not exist.

Usage: python tests/golden/make_cheb_golden.py   (needs oracle/_ref, i.e. /root/reference)
"""
import ctypes
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

OUT = Path(__file__).with_name("cheb_golden.json")
# (d, kernel, T, targets' cube offset, interpolation cube lower, side, p_list)
CASES = [
    (1, "log_r", 40, [2.0], [0.0], 1.0, [1, 2, 4, 6, 8, 10, 12]),
    (2, "one_over_r", 60, [2.0, 0.0], [0.0, 0.0], 1.0, [1, 2, 4, 6, 8]),
    (2, "exp_neg_r", 30, [1.5, 1.5], [0.0, 0.0], 1.0, [2, 4, 6, 8, 10]),
    (3, "one_over_r", 32, [2.0, 0.0, 0.0], [0.0, 0.0, 0.0], 1.0, [1, 2, 3, 4, 6]),
    (4, "exp_neg_r", 8, [2.0, 0.0, 0.0, 0.0], [0.0, 0.0, 0.0, 0.0], 1.0, [1, 2, 3]),
]


def main():
    O.build()
    L = O.ref_lib()
    cases = []
    for (d, kname, T, toff, lower, side, ps) in CASES:
        x = O.points(d, toff, 1.0, T, O.UNIFORM, 2022 + d, 0)
        dec = O.ref_interpolation_decay(O.KERNEL_IDS[kname], x, lower, side, ps)
        cases.append({"d": d, "kernel": kname, "targets": x.tolist(), "lower": lower, "side": side,
                      "p": ps, "err": [e for _, e in dec]})
        print(d, kname, [f"{e:.3e}" for _, e in dec], flush=True)
    nodes = {}
    for p in (0, 1, 2, 5, 8, 13):
        out = np.zeros(p + 1)
        assert L.hbr_chebyshev_nodes(p, out.ctypes.data) == 0
        nodes[str(p)] = out.tolist()
    fits = []
    for c in cases:
        ps = np.ascontiguousarray(c["p"], dtype=np.int32)
        es = np.ascontiguousarray(c["err"])
        rho = ctypes.c_double()
        assert L.hbr_fit_decay_rate(ps.ctypes.data, es.ctypes.data, len(ps), ctypes.byref(rho)) == 0
        vd = ctypes.c_double()
        st = L.hbr_v_d_constant(c["d"], rho.value, ctypes.byref(vd))
        fits.append({"rho": rho.value, "v_d": vd.value if st == 0 else None})
    OUT.write_text(json.dumps({"source": "chebyshev.hpp compiled in oracle/_ref", "cases": cases,
                               "nodes": nodes, "fits": fits}) + "\n")
    print(OUT)


if __name__ == "__main__":
    main()
