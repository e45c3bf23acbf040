"""ACA parity cases shared by tests/golden/make_aca_golden.py (fixtures from the reference's own
aca.hpp compiled in oracle/_ref), tests/test_aca_oracle.py and tests/test_gpu_aca.py.
Points: the oracle's seeded uniform cube pair, optionally scaled / shifted (numpy, exact ops)
to produce exactly-zero blocks (exp(-r^2) underflow) and coincident points."""
import numpy as np

# name, d, d', kernel, n_target, n_source, seed, block (rb, rows, cb, cols) or None, eps,
# max_rank, source shift along axis 0 (applied to the last `shift_cols` sources; 0 = none)
CASES = [
    ("edge2d_log_full_e6", 2, 1, "log_r", 600, 600, 11, None, 1e-6, 600, 0.0, 0),
    ("edge2d_log_full_e12", 2, 1, "log_r", 600, 600, 11, None, 1e-12, 600, 0.0, 0),
    ("face3d_inv_sub", 3, 2, "one_over_r", 500, 520, 12, (100, 300, 50, 400), 1e-10, 500, 0.0, 0),
    ("dp3_4d_exp_trunc", 4, 3, "exp_neg_r", 400, 400, 13, None, 1e-10, 50, 0.0, 0),
    ("vertex1d_log", 1, 0, "log_r", 300, 300, 14, None, 1e-12, 300, 0.0, 0),
    ("far2d_log_degenerate", 2, None, "log_r", 300, 300, 15, None, 1e-15, 300, 0.0, 0),
    ("far3d_gauss_zero_block", 3, None, "exp_neg_r2", 200, 150, 16, None, 1e-8, 200, 40.0, 150),
    ("edge2d_gauss_half_zero", 2, 1, "exp_neg_r2", 256, 256, 17, None, 1e-10, 256, 40.0, 128),
    ("vertex2d_inv_maxrank1", 2, 0, "one_over_r", 100, 90, 18, None, 1e-12, 1, 0.0, 0),
    ("face3d_inv_one_row", 3, 2, "one_over_r", 64, 64, 19, (5, 1, 0, 64), 1e-12, 64, 0.0, 0),
    ("face3d_inv_one_col", 3, 2, "one_over_r", 64, 64, 19, (0, 64, 7, 1), 1e-12, 64, 0.0, 0),
    ("dp2_4d_sinr", 4, 2, "sin_r", 300, 280, 20, None, 1e-9, 300, 0.0, 0),
    ("edge2d_r_exact_lowrank", 2, 1, "r", 200, 200, 21, None, 1e-13, 200, 0.0, 0),
    ("far3d_inv_degenerate", 3, None, "one_over_r", 200, 200, 5, None, 1e-15, 200, 0.0, 0),
    ("far1d_gauss_degenerate", 1, None, "exp_neg_r2", 200, 200, 5, None, 1e-13, 200, 0.0, 0),
]


def case_points(oracle, case):
    name, d, dp, kern, nt, ns, seed, blk, eps, mr, shift, shift_cols = case
    x = oracle.points(d, [0.0] * d, 1.0, nt, 0, seed, 0)
    from oracle.oracle import offset
    y = oracle.points(d, offset(d, dp), 1.0, ns, 0, seed, 1)
    if shift_cols:
        y = y.copy()
        y[0, ns - shift_cols:] = y[0, ns - shift_cols:] + shift
    return x, y


def case_block(case):
    _, _, _, _, nt, ns, _, blk, _, _, _, _ = case
    return blk if blk is not None else (0, nt, 0, ns)


def case_q(case):
    rb, rows, cb, cols = case_block(case)
    return np.random.default_rng(1000 + case[6]).standard_normal(cols)
