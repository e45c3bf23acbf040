"""Generate tests/golden/classify_golden.json: the reference's own hodlr::classify_pair
(geometry.hpp:109-118) and box_grid (geometry.hpp:123-131), compiled in place into
oracle/_ref/libhb_ref.so, over every box pair of small uniform subdivisions.  The fixture lets the
ABI test run where /root/reference is absent (the GPU box).

Usage: python tests/golden/make_classify_golden.py   (needs oracle/_ref, i.e. /root/reference)
"""
import ctypes
import itertools
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

OUT = Path(__file__).with_name("classify_golden.json")
CASES = [(1, 3), (2, 2), (3, 2), (4, 1)]  # (d, level): every ordered pair of boxes


def ref_classify(L, d, la, ga, lb, gb):
    a = (ctypes.c_int32 * d)(*ga)
    b = (ctypes.c_int32 * d)(*gb)
    kind, sdim = ctypes.c_int32(), ctypes.c_int32()
    st = L.hbr_classify_pair(d, la, a, lb, b, ctypes.byref(kind), ctypes.byref(sdim))
    return st, kind.value, sdim.value


def main():
    O.build()
    L = O.ref_lib()
    out = {"source": "hodlr::classify_pair / box_grid (geometry.hpp) compiled in oracle/_ref",
           "cases": []}
    for d, level in CASES:
        nbox = 1 << (d * level)
        grids = []
        for i in range(nbox):
            g = (ctypes.c_int32 * d)()
            assert L.hbr_box_grid(d, level, i, g) == 0
            grids.append(list(g))
        kinds = []
        for a, b in itertools.product(range(nbox), repeat=2):
            st, kind, sdim = ref_classify(L, d, level, grids[a], level, grids[b])
            assert st == 0
            kinds.append(kind * 16 + (sdim + 1))  # packed: kind << 4 | (d' + 1)
        out["cases"].append({"d": d, "level": level, "grids": grids, "packed": kinds})
    st, _, _ = ref_classify(L, 2, 1, [0, 0], 2, [0, 0])  # different levels -> invalid_argument
    out["different_levels_status"] = st
    OUT.write_text(json.dumps(out, separators=(",", ":")) + "\n")
    print(OUT, sum(len(c["packed"]) for c in out["cases"]), "pairs")


if __name__ == "__main__":
    main()
