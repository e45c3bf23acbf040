"""SPEC cli `rank-bench` built on the C++ host mirror (host/hb200.hpp)."""
import subprocess

import pytest

from conftest import ROOT

EXE = ROOT / "paper_2209_05819_b200" / "lib" / "rank-bench"


def run(*args):
    return subprocess.run([str(EXE), *args], capture_output=True, text=True, timeout=600)


def test_cli_usage_errors():
    if not EXE.exists():
        pytest.skip("rank-bench not built")
    assert run("--d", "1").returncode == 64                       # missing required flag
    assert run("--d", "1", "--interaction", "far", "--kernel", "nope", "--N", "10").returncode == 64
    assert run("--d", "1", "--interaction", "far", "--kernel", "log_r", "--N", "10",
               "--grid", "weird").returncode == 64


@pytest.mark.gpu
@pytest.mark.parametrize("args,want", [
    (["--d", "1", "--interaction", "far", "--kernel", "log_r", "--N", "1000", "--grid", "closed"], 7),
    (["--d", "2", "--interaction", "surface:0", "--kernel", "one_over_r", "--N", "10000",
      "--grid", "interior"], 104),  # SPEC.md:637 example (paper 2D vertex F1, N=10000)
    (["--d", "3", "--interaction", "surface:2", "--kernel", "one_over_r", "--N", "1000",
      "--grid", "interior"], 312),
    # complex columns (PAPER.md:1357-1369 3-D face F3 / F4 at N = 125; :682-692 2-D vertex F4)
    (["--d", "3", "--interaction", "surface:2", "--kernel", "helmholtz3d", "--N", "125",
      "--grid", "interior"], 99),
    (["--d", "3", "--interaction", "surface:2", "--kernel", "hankel_h12", "--N", "125",
      "--grid", "interior"], 119),
    (["--d", "2", "--interaction", "surface:0", "--kernel", "hankel_h12", "--N", "1600",
      "--grid", "interior"], 94),
])
def test_cli_paper_values(args, want):
    r = run(*args)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0].startswith("kernel,d,interaction,dprime,N,epsilon,rank,seconds")
    assert int(lines[1].split(",")[6]) == want


@pytest.mark.gpu
def test_cli_fit_growth():
    """--fit 1: SPEC fit_growth on the computed series (2-D edge, log r, interior grids): the
    power law wins with exponent near d'/d = 1/2."""
    r = run("--d", "2", "--interaction", "surface:1", "--kernel", "log_r", "--N",
            "1600,3600,6400,10000,14400", "--grid", "interior", "--fit", "1")
    assert r.returncode == 0, r.stderr
    line = next(ln for ln in r.stderr.splitlines() if ln.startswith("# fit log_r"))
    assert "best power" in line
    c = float(line.split("N^")[1].split(",")[0])
    assert abs(c - 0.5) <= 0.15, line
