"""C-ABI library checks that need no GPU: the library loads, exports every symbol the headers in
include/ declare, the ctypes struct layouts match the C compiler's, and the pure-host entry
points (status strings, scalar kernel evaluation, seeds, LPT partition, argument validation)
behave like the reference interface (kernel.hpp / geometry.hpp exceptions -> status codes)."""
import ctypes
import math
import re
import subprocess

import pytest

from conftest import ROOT


def declared_functions():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b(hb_\w+)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return sorted(names)


def test_library_exports_every_declared_symbol(hb):
    L = hb.load()
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) <= set(hb.EXPORTS) | {"hb_sweep"}


def test_version_and_status_strings(hb):
    L = hb.load()
    assert b"sm_100a" in L.hb_version()
    for s in range(9):
        assert L.hb_status_string(s)
    assert L.hb_phase_name(4) == b"update"


def test_struct_layouts_match_c(tmp_path, hb):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "hb.h"\nint main(){printf("%zu %zu %zu %zu %zu %zu %zu %zu\\n",'
                   'sizeof(hb_kernel),sizeof(hb_cube),sizeof(hb_pair),sizeof(hb_rank_result),'
                   'sizeof(hb_problem),sizeof(hb_stats),sizeof(hb_sweep_opts),offsetof(hb_pair,seed));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(t) for t in (hb.hb_kernel, hb.hb.hb_cube, hb.hb_pair, hb.hb_rank_result,
                                       hb.hb_problem, hb.hb_stats, hb.hb.hb_sweep_opts)]
    want.append(hb.hb_pair.seed.offset)
    assert got == want


def test_eval_radial_host_known_answers(hb):
    assert hb.eval_radial_host(hb.make_kernel("log_r"), 1.0) == 0.0
    assert hb.eval_radial_host(hb.make_kernel("one_over_r"), 2.0) == 0.5
    assert hb.eval_radial_host(hb.make_kernel("exp_neg_r"), 0.0) == 1.0
    assert hb.eval_radial_host(hb.make_kernel("log_r"), 0.0) == 0.0  # catalog diagonal
    assert hb.eval_radial_host(hb.make_kernel("exp_neg_r", diagonal=None), 0.0) == 1.0
    assert hb.eval_radial_host(hb.make_kernel("sin_r"), math.pi / 2) == 1.0
    with pytest.raises(hb.HBError) as e:
        hb.eval_radial_host(hb.make_kernel("one_over_r", diagonal=None), 0.0)
    assert e.value.status == 4  # ESINGULAR (kernel.hpp:152-153)
    with pytest.raises(hb.HBError) as e:
        hb.eval_radial_host(hb.make_kernel("custom"), 1.0)
    assert e.value.status == 5  # EUNSUPPORTED: std::function cannot cross the ABI
    with pytest.raises(hb.HBError) as e:
        hb.eval_radial_host(hb.make_kernel(99), 1.0)
    assert e.value.status == 1


def test_problem_seed_matches_oracle(hb, oracle):
    for d, dp, n in [(1, 0, 1000), (2, None, 16000), (4, 3, 65536), (3, 2, 32000)]:
        assert hb.problem_seed(0, d, dp, n) == oracle.problem_seed(0, d, dp, n)
        assert hb.problem_seed(5, d, dp, n) != hb.problem_seed(0, d, dp, n)


def sweep_problems(hb, ns=(1000, 2000, 4000, 8000, 16000, 32000, 65536)):
    probs = []
    for n in ns:
        for d in range(1, 5):
            for dp in list(range(d)) + [None]:
                for k in ("log_r", "one_over_r", "exp_neg_r"):
                    probs.append(hb.make_problem(k, d, dp, n, [1e-12, 1e-10] if d == 4 else [1e-12]))
    return probs


def test_partition_lpt(hb):
    probs = sweep_problems(hb)
    assert len(probs) == 294
    for parts in (1, 2, 4, 8):
        own = hb.partition(probs, parts)
        assert len(own) == 294 and set(own) <= set(range(parts))
        assert hb.partition(probs, parts) == own  # deterministic
        if parts > 1:
            assert len(set(own)) == parts


def test_argument_validation_without_gpu(hb):
    L = hb.load()
    probs = (hb.hb_problem * 1)(hb.make_problem("log_r", 1, 0, 10, [1e-12]))
    out = (hb.hb_rank_result * 1)()
    devs = (ctypes.c_int32 * 1)(0)
    assert L.hb_sweep(probs, -1, devs, 1, out, None) == hb.hb.EINVAL
    assert L.hb_sweep(probs, 1, devs, 0, out, None) == hb.hb.EINVAL
    own = (ctypes.c_int32 * 1)()
    assert L.hb_partition(probs, 1, 0, own) == hb.hb.EINVAL


def test_context_create_without_gpu_fails_loudly(hb):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(hb.HBError):
        hb.Context(0)


# ---- classify_pair (geometry.hpp:109-118) ------------------------------------------------------

def _golden_classify():
    import json
    from conftest import GOLDEN
    return json.loads((GOLDEN / "classify_golden.json").read_text())


def test_classify_pair_matches_reference_golden(hb):
    """hb_classify_pair equals the reference's own classify_pair (compiled in oracle/_ref and
    frozen by tests/golden/make_classify_golden.py) on every ordered box pair of the uniform
    subdivisions d=1 level 3, d=2/3 level 2, d=4 level 1."""
    g = _golden_classify()
    n = 0
    for case in g["cases"]:
        d, level, grids = case["d"], case["level"], case["grids"]
        nb = len(grids)
        for a in range(nb):
            for b in range(nb):
                want = case["packed"][a * nb + b]
                kind, sdim = hb.classify_pair(level, grids[a], level, grids[b])
                assert (kind, sdim) == (want >> 4, (want & 15) - 1), (d, grids[a], grids[b])
                n += 1
    assert n == 4672
    with pytest.raises(hb.HBError) as e:
        hb.classify_pair(1, [0, 0], 2, [0, 0])
    assert e.value.status == g["different_levels_status"] == hb.hb.EINVAL


def test_classify_pair_matches_compiled_reference_live(hb, oracle):
    """Same check against the live compiled reference (skipped where /root/reference is absent),
    plus random grids at deeper levels."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (no /root/reference)")
    import random
    L = oracle.ref_lib()
    rng = random.Random(5)
    for _ in range(3000):
        d = rng.randint(1, 6)
        level = rng.randint(0, 6)
        ga = [rng.randrange(1 << level) for _ in range(d)]
        gb = [min((1 << level) - 1, max(0, x + rng.randint(-2, 2))) for x in ga]
        a = (ctypes.c_int32 * d)(*ga)
        b = (ctypes.c_int32 * d)(*gb)
        kind, sdim = ctypes.c_int32(), ctypes.c_int32()
        assert L.hbr_classify_pair(d, level, a, level, b, ctypes.byref(kind), ctypes.byref(sdim)) == 0
        assert hb.classify_pair(level, ga, level, gb) == (kind.value, sdim.value)


def test_classify_cubes_and_pair_geometry(hb):
    """The BASELINE pair geometry (source = target + o) classifies to the d' it
    is built for; non-grid cube pairs are rejected like a different-level BoxIndex pair."""
    for d in range(1, 5):
        for dp in list(range(d)) + [None]:
            p = hb.make_pair(d, dp, 10, hb.UNIFORM, 0)
            kind, sdim = hb.classify_cubes(p.target, p.source)
            if dp is None:
                assert kind == hb.IC_FAR
            else:
                assert (kind, sdim) == (hb.IC_SURFACE, dp)
    c = hb.make_cube([0.0, 0.0])
    assert hb.classify_cubes(c, c) == (hb.IC_SELF, -1)
    with pytest.raises(hb.HBError):
        hb.classify_cubes(c, hb.make_cube([0.5, 0.0]))       # not on one grid
    with pytest.raises(hb.HBError):
        hb.classify_cubes(c, hb.make_cube([1.0, 0.0], 2.0))  # different sides


# ---- fit_growth on the paper's own tables ------------------------------------

def _series(paper_tables, label, kernel):
    tab = next(t for t in paper_tables if t["label"] == label)
    ci = tab["kernels"].index(kernel)
    return [r["N"] for r in tab["rows"]], [r["ranks"][ci] for r in tab["rows"]]


def test_fit_growth_spec_examples(hb, paper_tables):
    """SPEC.md:585-588 / acceptance 2: far field constant (max/min <= 1.3), vertex best fit log with
    a power exponent < 0.2, 2-D edge exponent 0.5 +- 0.1, 3-D face 0.667 +- 0.1 — on the paper's
    published table values as fixtures."""
    f = hb.fit_growth(*_series(paper_tables, "tab:res_2d_far", "one_over_r"))
    assert f["best"] == "constant" and f["max_min_ratio"] <= 1.3
    for label in ("tab:res_2d_ver", "tab:res_1d_vert", "tab:res_3d_ver"):
        f = hb.fit_growth(*_series(paper_tables, label, "one_over_r"))
        assert f["best"] == "log" and f["rss"]["log"] < f["rss"]["power"] and f["power"][1] < 0.2
    f = hb.fit_growth(*_series(paper_tables, "tab:res_2d_edge", "log_r"))
    assert f["best"] == "power" and abs(f["power"][1] - 0.5) <= 0.1
    f = hb.fit_growth(*_series(paper_tables, "tab:res_3d_face", "one_over_r"))
    assert f["best"] == "power" and abs(f["power"][1] - 2.0 / 3.0) <= 0.1


def test_fit_growth_refuses_short_series(hb):
    with pytest.raises(hb.HBError) as e:  # fewer than 4 points -> fit refused
        hb.fit_growth([1000, 2000, 4000, 4000], [5, 6, 7, 7])
    assert e.value.status == 1
    with pytest.raises(hb.HBError):
        hb.fit_growth([1000, 0, 4000, 8000], [5, 6, 7, 8])
    f = hb.fit_growth([1000, 2000, 4000, 8000], [10.0, 20.0, 40.0, 80.0])  # exact N^1
    assert f["best"] == "power" and f["power"][1] == pytest.approx(1.0, abs=1e-6)
