"""Device ACA (csrc/aca.cu, aca.hpp:16-213) against the oracle restatement — itself pinned bit
for bit to the reference's own aca.hpp (tests/test_aca_oracle.py) — through the C ABI:
pivot sequences, rank and tolerance_met identical; L / U / apply(q) bit-identical for kernels
whose entries are exactly rounded on both sides (1/r, r: IEEE div / sqrt) and within the stated
tolerances for libdevice log / exp / sin entries (<= 2 ulp per entry, amplified by the residual
cancellation of late pivots); batched blocks, the multi-CTA group path, U/V growth, and the
reference's error behaviour."""
import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
sys.path.insert(0, str(GOLDEN))
from aca_cases import CASES, case_block, case_points, case_q  # noqa: E402

EXACT = {"one_over_r", "r"}  # entries bit-identical on both sides
# libdevice entries (<= 2 ulp each): apply(q) within B_TOL relative.  U(k, :) = pivot_k v_k(τ) is
# a residual row, absolute error ~ ulp * max|K| (growing mildly with k): within LU_TOL * max|pivot|;
# L(:, k) = u_k(σ) / pivot_k divides such a residual by pivot_k: within LU_TOL * max|pivot| /
# |pivot_k| (times the column's own scale) — the amplification ACA itself introduces.
# apply(q): t = K(σ, J) q is a reduction, summed in a different order than Eigen's, so b is
# compared within B_TOL relative for every kernel (L / U are bit-identical for EXACT kernels).
B_TOL, LU_TOL = 1e-9, 1e-11
GOLD = {r["name"]: r for r in json.loads((GOLDEN / "aca_golden.json").read_text())}


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def gpu_aca(ctx, hb, kern, x, y, blocks, eps, mr, q=None):
    X, Y = dev(x), dev(y)
    torch.cuda.synchronize()
    d, nt = x.shape
    ns = y.shape[1]
    K = hb.make_kernel(kern)
    fs = ctx.aca_compress(K, X.data_ptr(), nt, Y.data_ptr(), ns, d, blocks, eps, mr)
    out = []
    for f in fs:
        sig, tau, L, U = f.arrays()
        b = None
        if q is not None:
            Q = dev(q)
            B = torch.empty(f.block.rows, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            ctx.aca_apply(f, K, X.data_ptr(), nt, Y.data_ptr(), ns, d, Q.data_ptr(), B.data_ptr())
            b = B.cpu().numpy()
        out.append(dict(rank=f.rank, met=f.tolerance_met, sigma=sig, tau=tau, L=L, U=U, b=b,
                        mem=f.memory_bytes))
        f.close()
    return out


def check_same(g, o, kern, what=""):
    assert (g["rank"], g["met"]) == (o.rank, o.met), what
    assert np.array_equal(g["sigma"], o.sigma) and np.array_equal(g["tau"], o.tau), what
    if o.b is not None and np.abs(o.b).max() > 0:
        assert np.linalg.norm(g["b"] - o.b) <= B_TOL * np.linalg.norm(o.b), what
    if kern in EXACT:
        assert np.array_equal(g["L"], o.L) and np.array_equal(g["U"], o.U), what
    else:
        if o.rank:
            piv = np.abs(np.diag(o.U))
            pmax = piv.max()
            for k in range(o.rank):
                sL = max(np.abs(o.L[:, k]).max(), 1.0)
                assert np.abs(g["L"][:, k] - o.L[:, k]).max() <= LU_TOL * pmax / piv[k] * sL, (what, k)
                assert np.abs(g["U"][k, :] - o.U[k, :]).max() <= LU_TOL * pmax, (what, k)
    assert g["mem"] == 2 * o.rank * o.rank * 8 + 2 * o.rank * 8


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_aca_matches_oracle_and_reference(ctx, hb, oracle, case):
    name, d, dp, kern, nt, ns, seed, blk, eps, mr, shift, sc = case
    x, y = case_points(oracle, case)
    rb, rows, cb, cols = case_block(case)
    q = case_q(case)
    o = oracle.aca_compress(oracle.KERNEL_IDS[kern], x, y, eps, mr, rb, rows, cb, cols, q=q)
    g = gpu_aca(ctx, hb, kern, x, y, [(rb, rows, cb, cols)], eps, mr, q=q)[0]
    check_same(g, o, kern, name)
    gold = GOLD[name]  # the reference's own outputs (frozen)
    assert g["rank"] == gold["rank"] and g["sigma"].tolist() == gold["sigma"]
    assert g["tau"].tolist() == gold["tau"]


def test_aca_batched_blocks(ctx, hb, oracle):
    """Many blocks of one point set in one call (one CTA each, one launch)."""
    x, y = oracle.pair_points(3, 2, 900, 0, 31)
    kern = "one_over_r"
    blocks = [(0, 300, 0, 300), (300, 300, 0, 300), (600, 300, 600, 300), (0, 900, 450, 200),
              (123, 77, 456, 333), (0, 1, 0, 900), (899, 1, 899, 1), (10, 500, 10, 500)]
    g = gpu_aca(ctx, hb, kern, x, y, blocks, 1e-9, 900)
    for b, gi in zip(blocks, g):
        o = oracle.aca_compress(oracle.KERNEL_IDS[kern], x, y, 1e-9, 900, *b)
        check_same(gi, o, kern, str(b))


@pytest.mark.parametrize("d,dp,kern,n,eps", [(2, 1, "one_over_r", 3000, 1e-10),
                                              (2, 1, "log_r", 2500, 1e-10),
                                              (3, 2, "one_over_r", 5000, 1e-6),
                                              (4, 3, "exp_neg_r", 2000, 1e-8)])
def test_aca_multi_cta_group(ctx, hb, oracle, d, dp, kern, n, eps):
    """Blocks large enough for a cooperative group of CTAs (G > 1, two barriers per pivot)."""
    x, y = oracle.pair_points(d, dp, n, 0, 41)
    q = np.random.default_rng(5).standard_normal(n)
    o = oracle.aca_compress(oracle.KERNEL_IDS[kern], x, y, eps, n, q=q)
    g = gpu_aca(ctx, hb, kern, x, y, [(0, n, 0, n)], eps, n, q=q)[0]
    check_same(g, o, kern)


def test_aca_growth_path(ctx, hb, oracle):
    """U / V start with 3 columns and grow by doubling (state carried across relaunches)."""
    case = [c for c in CASES if c[0] == "face3d_inv_sub"][0]
    x, y = case_points(oracle, case)
    blk = case_block(case)
    o = oracle.aca_compress(0, x, y, case[8], case[9], *blk, q=case_q(case))
    os.environ["HB_ACA_INIT_CAP"] = "3"
    try:
        g = gpu_aca(ctx, hb, "one_over_r", x, y, [blk], case[8], case[9], q=case_q(case))[0]
        x2, y2 = oracle.pair_points(2, 1, 3000, 0, 41)
        o2 = oracle.aca_compress(0, x2, y2, 1e-10, 3000)
        g2 = gpu_aca(ctx, hb, "one_over_r", x2, y2, [(0, 3000, 0, 3000)], 1e-10, 3000)[0]
    finally:
        del os.environ["HB_ACA_INIT_CAP"]
    check_same(g, o, "one_over_r")
    check_same(g2, o2, "one_over_r")


def test_aca_errors(ctx, hb, oracle):
    x, y = oracle.pair_points(2, 1, 64, 0, 3)
    X, Y = dev(x), dev(y)
    torch.cuda.synchronize()
    K = hb.make_kernel("log_r")
    for blocks, eps, mr in (([(0, 64, 0, 64)], 0.0, 5), ([(0, 64, 0, 64)], 1e-8, 0),
                            ([(0, 0, 0, 64)], 1e-8, 5), ([(10, 60, 0, 64)], 1e-8, 5)):
        with pytest.raises(hb.HBError) as e:
            ctx.aca_compress(K, X.data_ptr(), 64, Y.data_ptr(), 64, 2, blocks, eps, mr)
        assert e.value.status == hb.hb.EINVAL
    Kn = hb.make_kernel("log_r", diagonal=None)
    with pytest.raises(hb.HBError) as e:  # r == 0 without a diagonal (kernel.hpp:152-153)
        ctx.aca_compress(Kn, X.data_ptr(), 64, X.data_ptr(), 64, 2, [(0, 64, 0, 64)], 1e-8, 10)
    assert e.value.status == hb.hb.ESINGULAR == GOLD["singular_self_log_nodiag"]["status"]
    with pytest.raises(hb.HBError) as e:
        ctx.aca_compress(hb.make_kernel("custom"), X.data_ptr(), 64, Y.data_ptr(), 64, 2,
                         [(0, 64, 0, 64)], 1e-8, 10)
    assert e.value.status == hb.hb.EUNSUPPORTED
