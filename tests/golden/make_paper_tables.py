"""Extract the paper's published ε-rank tables into tests/golden/paper_tables.json.

Run once in the build container (it reads /root/reference/PAPER.md, which does not exist on
the GPU box); the JSON it writes is the committed fixture.  Source: the 14 active tables of
doc A; commented-out ``\\cmt{...}`` tables (e.g.
``tab:res_1d_farc`` at PAPER.md:295) are skipped.  Geometry per table caption: Y=[0,1]^d
sources, X = Y - o targets; grids per SURVEY.md A.1 (closed grid for far-field, interior grid
for near-field).  Columns F1..F8; F3/F4 are complex kernels and are kept in
the file for completeness but only the real kernels are used by the tests.
"""
import json
import re
import sys
from pathlib import Path

PAPER = Path("/root/reference/PAPER.md")
OUT = Path(__file__).with_name("paper_tables.json")

# label -> (d, dprime or None for far)
TABLES = {
    "tab:res_1d_far": (1, None), "tab:res_1d_vert": (1, 0),
    "tab:res_2d_far": (2, None), "tab:res_2d_ver": (2, 0), "tab:res_2d_edge": (2, 1),
    "tab:res_3d_far": (3, None), "tab:res_3d_ver": (3, 0), "tab:res_3d_edge": (3, 1),
    "tab:res_3d_face": (3, 2),
    "tab:res_4d_far": (4, None), "tab:res_4d_ver": (4, 0), "tab:res_4d_h1": (4, 1),
    "tab:res_4d_h2": (4, 2), "tab:res_4d_h3": (4, 3),
}
# paper column -> reference KernelId name (kernel.hpp:112-129); None = complex kernel
COLUMNS = ["one_over_r", "log_r", None, None, "r", "sin_r", "inv_sqrt_1_plus_r", "exp_neg_r"]


def main() -> int:
    lines = PAPER.read_text().splitlines()[:1825]  # doc A only (PAPER.md:1825 separator)
    out = []
    for ln, text in enumerate(lines, start=1):
        m = re.search(r"\\label\{(tab:res_[a-z0-9_]+)\}", text)
        if not m or m.group(1) not in TABLES:
            continue
        label = m.group(1)
        # walk back to the tabular start
        start = ln - 1
        while "\\begin{tabular}" not in lines[start - 1]:
            start -= 1
        rows = []
        for row in lines[start:ln]:
            cells = [c.strip() for c in row.split("\\\\")[0].split("&")]
            if len(cells) == 9 and cells[0].isdigit():
                rows.append([int(c) for c in cells])
        d, dprime = TABLES[label]
        out.append({
            "label": label, "source": f"PAPER.md:{start}-{ln}", "d": d, "dprime": dprime,
            "grid": "closed" if dprime is None else "interior", "epsilon": 1e-12,
            "columns": ["F1", "F2", "F3", "F4", "F5", "F6", "F7", "F8"],
            "kernels": COLUMNS,
            "rows": [{"N": r[0], "ranks": r[1:]} for r in rows],
        })
    assert len(out) == 14, len(out)
    OUT.write_text(json.dumps(out, indent=1) + "\n")
    print(f"wrote {OUT} ({sum(len(t['rows']) for t in out)} N rows)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
