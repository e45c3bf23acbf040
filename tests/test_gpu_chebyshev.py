"""§8(f)4: the Chebyshev interpolation bound check (chebyshev.hpp:125-193) on the device, against the
reference's own interpolation_decay compiled in oracle/_ref (frozen in tests/golden/cheb_golden.json
by tests/golden/make_cheb_golden.py)."""
import json

import numpy as np
import pytest

from conftest import GOLDEN

GOLD = json.loads((GOLDEN / "cheb_golden.json").read_text())


def test_chebyshev_nodes_and_fits_match_reference(hb):
    """Host functions, no GPU: chebyshev_nodes bit for bit, fit_decay_rate and v_d_constant."""
    for p, want in GOLD["nodes"].items():
        assert hb.chebyshev_nodes(int(p)) == want
    for case, fit in zip(GOLD["cases"], GOLD["fits"]):
        rho = hb.fit_decay_rate(case["p"], case["err"])
        assert rho == pytest.approx(fit["rho"], rel=1e-14)
        if fit["v_d"] is not None:
            assert hb.v_d_constant(case["d"], rho) == pytest.approx(fit["v_d"], rel=1e-14)
    with pytest.raises(hb.HBError) as e:
        hb.chebyshev_nodes(-1)
    assert e.value.status == 1  # invalid_argument (chebyshev.hpp:17)
    with pytest.raises(hb.HBError) as e:
        hb.v_d_constant(2, 1.0)
    assert e.value.status == 2  # domain_error rho <= 1 (chebyshev.hpp:141)
    with pytest.raises(hb.HBError):
        hb.fit_decay_rate([2], [1e-3])  # fewer than two positive errors


@pytest.mark.gpu
@pytest.mark.parametrize("ci", range(len(GOLD["cases"])))
def test_interpolation_decay_matches_reference(ctx, hb, ci):
    """err_p = max |K - U V| per degree: within rounding of the reference (the DMMA GEMM sums in
    another order than Eigen's), and decaying geometrically like the reference's."""
    c = GOLD["cases"][ci]
    x = np.array(c["targets"])
    cube = hb.make_cube(c["lower"], c["side"])
    got = ctx.interpolation_decay(hb.make_kernel(c["kernel"]), x, cube, c["p"])
    for (p, e), want in zip(got, c["err"]):
        tol = 1e-7 * want + 1e-12  # |K| <= ~1.5 here; GEMM rounding ~ sqrt(M) u |U||V|
        assert abs(e - want) <= tol, (c["d"], c["kernel"], p, e, want)
    rho_gpu = hb.fit_decay_rate([p for p, _ in got], [e for _, e in got])
    assert rho_gpu == pytest.approx(GOLD["fits"][ci]["rho"], rel=1e-4)


@pytest.mark.gpu
def test_interpolation_decay_errors(ctx, hb):
    cube = hb.make_cube([0.0, 0.0], 1.0)
    touching = np.array([[1.0, 2.0], [0.5, 0.5]])  # first target on the cube's face
    with pytest.raises(hb.HBError) as e:
        ctx.interpolation_decay(hb.make_kernel("log_r"), touching, cube, [2])
    assert e.value.status == 1  # chebyshev.hpp:153-155
    with pytest.raises(hb.HBError):
        ctx.interpolation_decay(hb.make_kernel("log_r"), np.array([[3.0], [0.5]]), cube, [-1])


@pytest.mark.gpu
def test_interpolation_decay_4d_large(ctx, hb, oracle):
    """d = 4 at the reference's full sample density (20^4 = 160000 samples) and degree 8 (6561
    nodes): a T x 6561 x 160000 DMMA GEMM per degree; the decay stays geometric (rho > 1)."""
    x = oracle.points(4, [2.0, 0.0, 0.0, 0.0], 1.0, 256, oracle.UNIFORM, 5, 0)
    got = ctx.interpolation_decay(hb.make_kernel("exp_neg_r"), x, hb.make_cube([0.0] * 4, 1.0),
                                  [2, 4, 6, 8])
    errs = [e for _, e in got]
    assert all(a > b for a, b in zip(errs, errs[1:]))
    assert hb.fit_decay_rate([p for p, _ in got], errs) > 1.5
