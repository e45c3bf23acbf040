"""ACA oracle pins (CPU).  The C restatement (oracle/hb_oracle.c, aca.hpp:16-213) is checked
  * bit for bit against the reference's own aca.hpp / kernel.hpp compiled in place
    (oracle/_ref/libhb_ref.so; skipped where /root/reference is absent), and
  * against the frozen outputs of that reference (tests/golden/aca_golden.json) everywhere.
Also: the reference's assemble_dense (kernel.hpp:168-181) against the oracle's entries."""
import json
import math
import sys

import numpy as np
import pytest

from conftest import GOLDEN

sys.path.insert(0, str(GOLDEN))
from aca_cases import CASES, case_block, case_points, case_q  # noqa: E402

GOLD = {r["name"]: r for r in json.loads((GOLDEN / "aca_golden.json").read_text())}


def run(oracle, case, impl):
    name, d, dp, kern, nt, ns, seed, blk, eps, mr, shift, sc = case
    x, y = case_points(oracle, case)
    rb, rows, cb, cols = case_block(case)
    return oracle.aca_compress(oracle.KERNEL_IDS[kern], x, y, eps, mr, rb, rows, cb, cols,
                               q=case_q(case), impl=impl)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_oracle_matches_golden(oracle, case):
    g = GOLD[case[0]]
    a = run(oracle, case, "oracle")
    assert g["status"] == 0
    assert a.rank == g["rank"] and a.met == g["met"]
    assert a.sigma.tolist() == g["sigma"] and a.tau.tolist() == g["tau"]
    assert math.fsum(a.L.ravel(order="F")).hex() == g["L_fsum"]
    assert math.fsum(a.U.ravel(order="F")).hex() == g["U_fsum"]
    assert [float(v).hex() for v in a.U.diagonal()] == g["U_diag"]
    assert [float(v).hex() for v in a.b] == g["b"]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_oracle_bit_exact_vs_compiled_reference(oracle, case):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    a = run(oracle, case, "oracle")
    r = run(oracle, case, "ref")
    assert (a.rank, a.met) == (r.rank, r.met)
    assert np.array_equal(a.sigma, r.sigma) and np.array_equal(a.tau, r.tau)
    assert np.array_equal(a.L, r.L) and np.array_equal(a.U, r.U) and np.array_equal(a.b, r.b)


def test_aca_errors_match_reference(oracle):
    x, y = oracle.pair_points(2, 1, 50, 0, 1)
    k = oracle.KERNEL_IDS["log_r"]
    for kw, st in ((dict(eps=0.0, max_rank=5), 1), (dict(eps=1e-8, max_rank=0), 1)):
        with pytest.raises(oracle.OracleError) as e:
            oracle.aca_compress(k, x, y, **kw)
        assert e.value.status == st
        if oracle.ref_available():
            with pytest.raises(oracle.OracleError) as e2:
                oracle.aca_compress(k, x, y, impl="ref", **kw)
            assert e2.value.status == st
    with pytest.raises(oracle.OracleError) as e:  # empty block (aca.hpp:174-175)
        oracle.aca_compress(k, x, y, 1e-8, 5, rows=0)
    assert e.value.status == 1
    with pytest.raises(oracle.OracleError) as e:  # r == 0, no diagonal (kernel.hpp:152-153)
        oracle.aca_compress(k, x, x, 1e-8, 10, has_diag=False)
    assert e.value.status == GOLD["singular_self_log_nodiag"]["status"] == 4


@pytest.mark.parametrize("d,dp,kern", [(1, 0, "log_r"), (2, 1, "log_r"), (3, 2, "one_over_r"),
                                       (4, 3, "exp_neg_r"), (2, None, "inv_sqrt_1_plus_r"),
                                       (3, 0, "helmholtz3d_re"), (4, None, "exp_neg_r2")])
def test_reference_assemble_dense_equals_oracle(oracle, d, dp, kern):
    """The entry rule (kernel.hpp:168-181, Eigen's left-to-right strided-row norm) compiled from
    the reference equals the oracle's restatement bit for bit."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    x, y = oracle.pair_points(d, dp, 300, 0, 7)
    k = oracle.KERNEL_IDS[kern]
    assert np.array_equal(oracle.ref_assemble(k, x, y), oracle.assemble(k, x, y))


def test_reference_entry_cap(oracle):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    x, y = oracle.pair_points(2, 1, 100, 0, 7)
    with pytest.raises(oracle.OracleError) as e:  # kernel.hpp:174-175 length_error
        oracle.ref_assemble(1, x, y, entry_cap=9999)
    assert e.value.status == 3
    with pytest.raises(oracle.OracleError) as e2:
        oracle.assemble(1, x, y, entry_cap=9999)
    assert e2.value.status == 3
