"""paper_2209_05819_b200 — B200-native (sm_100a) rank-reveal path of arxiv 2209.05819.

Seeded cube-pair points (k1) -> FP64 kernel-block assembly (k2) -> sketch-pivoted blocked QR with
DMMA trailing updates and bidiagonal certification (k3) -> multi-device sweep (k4), exposed
through the C ABI in include/hb.h and bound here with ctypes (hb.py).  The CUDA library is the
only implementation; there is no CPU fallback.
"""
from .hb import (  # noqa: F401
    CATALOG_DIAG, EXPORTS, GRID_CLOSED, GRID_INTERIOR, KERNEL_IDS, KERNEL_NAMES, LIB_PATH,
    UNIFORM, Context, HBError, RankResult, eval_radial_host, hb_kernel, hb_pair, hb_problem,
    hb_rank_result, load, make_cube, make_kernel, make_pair, make_problem, offset, partition,
    problem_seed, sweep, global_stats, reset_global_stats, sweep_release, hb_stats, PHASES,
    ACAFactor, hb_block, classify_pair, classify_cubes, hb_interaction, hb_cube, IC_SELF,
    IC_SURFACE, IC_FAR, DPRIME_FAR, DPRIME_SELF, fit_growth,
    chebyshev_nodes, fit_decay_rate, v_d_constant, HMatrix, hb_build_report, POLICIES,
)
