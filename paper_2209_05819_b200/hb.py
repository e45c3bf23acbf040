"""ctypes binding of the C ABI in include/hb.h (libhb200.so, sm_100a).

This is the Python stub a maintainer would add on the reference side; tests and
bench.py call the product only through it.  There is no CPU fallback: if the CUDA library is
missing or no GPU is present, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "lib" / "libhb200.so"

# status codes (hb.h)
OK, EINVAL, EDOMAIN, ECAP, ESINGULAR, EUNSUPPORTED, ENOMEM, ECUDA, ENCCL = range(9)
STATUS_NAMES = ["OK", "EINVAL", "EDOMAIN", "ECAP", "ESINGULAR", "EUNSUPPORTED", "ENOMEM", "ECUDA",
                "ENCCL"]

# KernelId order of kernel.hpp:19-32; names of kernel_from_string (kernel.hpp:112-129)
KERNEL_IDS = {
    "one_over_r": 0, "log_r": 1, "helmholtz3d_re": 2, "helmholtz3d_im": 3,
    "hankel_h12_re": 4, "hankel_h12_im": 5, "r": 6, "sin_r": 7,
    "inv_sqrt_1_plus_r": 8, "exp_neg_r": 9, "exp_neg_r2": 10, "custom": 11,
}
KERNEL_NAMES = {v: k for k, v in KERNEL_IDS.items()}
# KernelSpec::catalog diagonal values (kernel.hpp:46-61)
CATALOG_DIAG = {0: 0.0, 1: 0.0, 2: 0.0, 5: 0.0, 3: 1.0, 8: 1.0, 9: 1.0, 10: 1.0, 4: 0.0, 6: 0.0,
                7: 0.0}
UNIFORM, GRID_INTERIOR, GRID_CLOSED = 0, 1, 2
MAX_TOLS = 4


class HBError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{where}: {name}" + (f" ({detail})" if detail else ""))
        self.status = status


class hb_kernel(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int32), ("has_diag", ctypes.c_int32), ("diag", ctypes.c_double)]


class hb_cube(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("lower", ctypes.c_double * 8), ("side", ctypes.c_double)]


class hb_pair(ctypes.Structure):
    _fields_ = [("target", hb_cube), ("source", hb_cube), ("d_prime", ctypes.c_int32),
                ("point_mode", ctypes.c_int32), ("n_target", ctypes.c_int64),
                ("n_source", ctypes.c_int64), ("seed", ctypes.c_uint64)]


class hb_rank_result(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("rank_lo", ctypes.c_int32), ("rank_hi", ctypes.c_int32),
                ("k_factored", ctypes.c_int32), ("sigma1", ctypes.c_double),
                ("sigma_r", ctypes.c_double), ("sigma_r1", ctypes.c_double),
                ("gap", ctypes.c_double), ("resid", ctypes.c_double),
                ("sec", ctypes.c_double * 4), ("certificate", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("fp_band", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {f: (list(getattr(self, f)) if f == "sec" else getattr(self, f))
                for f, _ in self._fields_}


NPHASE = 11
PHASES = ["assembly", "sketch", "pivot", "panel", "update", "downdate", "sigma1", "cert_qr",
          "bidiag", "bisect", "chase"]
MAX_DEVICES = 64


class hb_stats(ctypes.Structure):
    _fields_ = [("phase_ms", ctypes.c_double * NPHASE), ("gemm_ms", ctypes.c_double),
                ("gemm_flops", ctypes.c_double), ("gemm_launches", ctypes.c_uint64),
                ("launches", ctypes.c_uint64), ("problems", ctypes.c_uint64)]

    def as_dict(self) -> dict:
        return {"phase_ms": dict(zip(PHASES, list(self.phase_ms))), "gemm_ms": self.gemm_ms,
                "gemm_flops": self.gemm_flops, "gemm_launches": self.gemm_launches,
                "launches": self.launches, "problems": self.problems}


class hb_sweep_opts(ctypes.Structure):
    _fields_ = [("profiling", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("device_seconds", ctypes.c_double * MAX_DEVICES)]


class hb_block(ctypes.Structure):
    """BlockSpec index ranges (aca.hpp:16-28)."""
    _fields_ = [("row_begin", ctypes.c_int64), ("rows", ctypes.c_int64),
                ("col_begin", ctypes.c_int64), ("cols", ctypes.c_int64)]


class hb_interaction(ctypes.Structure):
    """InteractionClass (geometry.hpp:77-104): kind SELF / SURFACE / FAR + d'."""
    _fields_ = [("kind", ctypes.c_int32), ("surface_dim", ctypes.c_int32)]


IC_SELF, IC_SURFACE, IC_FAR = 0, 1, 2
DPRIME_FAR, DPRIME_SELF = -1, -2


class hb_growth_fit(ctypes.Structure):
    """SPEC fit_growth result."""
    _fields_ = [("best", ctypes.c_int32), ("n", ctypes.c_int32), ("constant", ctypes.c_double),
                ("log_a", ctypes.c_double), ("log_b", ctypes.c_double), ("pow_a", ctypes.c_double),
                ("pow_c", ctypes.c_double), ("rss", ctypes.c_double * 3),
                ("max_min_ratio", ctypes.c_double)]


GROWTH_MODELS = ["constant", "log", "power"]


class hb_build_report(ctypes.Structure):
    """BuildReport (hmatrix.hpp:19-26)."""
    _fields_ = [("init_seconds", ctypes.c_double), ("memory_bytes", ctypes.c_int64),
                ("max_block_rank", ctypes.c_int32), ("depth", ctypes.c_int32),
                ("num_low_rank_blocks", ctypes.c_int64), ("num_dense_entries", ctypes.c_int64),
                ("num_tolerance_failures", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


POLICIES = {"weakdd": 0, "strong": 1, "weakall": 2}  # AdmissibilityPolicy (cluster_tree.hpp:17-29)


class hb_problem(ctypes.Structure):
    _fields_ = [("kernel", hb_kernel), ("pair", hb_pair), ("tols", ctypes.c_double * MAX_TOLS),
                ("ntol", ctypes.c_int32), ("reserved", ctypes.c_int32)]


# every symbol include/hb.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "hb_version", "hb_status_string", "hb_last_error", "hb_context_create", "hb_context_destroy",
    "hb_context_stream", "hb_context_set_tuning", "hb_generate_points", "hb_assemble",
    "hb_eval_radial_host", "hb_rank_matrix", "hb_rank", "hb_last_sigma", "hb_sweep",
    "hb_partition", "hb_problem_seed", "hb_rank_complex", "hb_phase_name", "hb_context_set_profiling",
    "hb_stats_get", "hb_stats_reset", "hb_sweep_ex", "hb_sweep_release", "hb_context_set_stopping",
    "hb_classify_pair", "hb_classify_cubes", "hb_interaction_dprime", "hb_assemble_dense_host",
    "hb_fit_growth", "hb_chebyshev_nodes", "hb_interpolation_decay", "hb_fit_decay_rate",
    "hb_v_d_constant", "hb_hmatrix_build", "hb_hmatrix_matvec", "hb_hmatrix_matvec_device",
    "hb_hmatrix_tree_order", "hb_hmatrix_destroy",
    # include/hb_debug.h (test hooks)
    "hb_debug_dgemm", "hb_debug_dgemm_async", "hb_debug_dgemm_fro",
    # ACA (aca.hpp)
    "hb_aca_compress", "hb_aca_factor_info", "hb_aca_factor_copy", "hb_aca_apply",
    "hb_aca_factor_destroy",
]

_lib = None


def load(path: os.PathLike | str | None = None):
    """Load libhb200.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # HB200_LIB: another build of the library (A/B comparisons of kernels; tools only)
    p = Path(path) if path else Path(os.environ.get("HB200_LIB", LIB_PATH))
    if not p.exists():
        raise FileNotFoundError(f"{p} is missing: run `make -C paper_2209_05819_b200` "
                                f"(or __graft_entry__.build())")
    L = ctypes.CDLL(str(p))
    c_p = ctypes.c_void_p
    L.hb_version.restype = ctypes.c_char_p
    L.hb_status_string.restype = ctypes.c_char_p
    L.hb_status_string.argtypes = [ctypes.c_int]
    L.hb_last_error.restype = ctypes.c_char_p
    L.hb_last_error.argtypes = [c_p]
    L.hb_context_create.argtypes = [ctypes.c_int, ctypes.POINTER(c_p)]
    L.hb_context_destroy.argtypes = [c_p]
    L.hb_context_destroy.restype = None
    L.hb_context_stream.argtypes = [c_p]
    L.hb_context_stream.restype = c_p
    L.hb_context_set_tuning.argtypes = [c_p, ctypes.c_int32, ctypes.c_double]
    L.hb_context_set_stopping.argtypes = [c_p, ctypes.c_int32]
    L.hb_context_set_stopping.restype = ctypes.c_int
    L.hb_generate_points.argtypes = [c_p, ctypes.POINTER(hb_pair), c_p, c_p]
    L.hb_assemble.argtypes = [c_p, ctypes.POINTER(hb_kernel), c_p, ctypes.c_int64, c_p,
                              ctypes.c_int64, ctypes.c_int32, c_p, ctypes.c_int64]
    L.hb_classify_pair.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                   ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(hb_interaction)]
    L.hb_classify_cubes.argtypes = [ctypes.POINTER(hb_cube), ctypes.POINTER(hb_cube),
                                    ctypes.POINTER(hb_interaction)]
    L.hb_fit_growth.argtypes = [ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double),
                                ctypes.c_int32, ctypes.POINTER(hb_growth_fit)]
    L.hb_fit_growth.restype = ctypes.c_int
    L.hb_hmatrix_build.argtypes = [c_p, ctypes.POINTER(hb_kernel), c_p, ctypes.c_int64, ctypes.c_int32,
                                   ctypes.POINTER(hb_cube), ctypes.c_int32, ctypes.c_int64,
                                   ctypes.c_double, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(c_p),
                                   ctypes.POINTER(hb_build_report)]
    L.hb_hmatrix_matvec.argtypes = [c_p, c_p, c_p, ctypes.c_int32]
    L.hb_hmatrix_matvec_device.argtypes = [c_p, c_p, c_p]
    L.hb_hmatrix_tree_order.argtypes = [c_p, c_p]
    L.hb_hmatrix_destroy.argtypes = [c_p]
    L.hb_hmatrix_destroy.restype = None
    for name in ("hb_hmatrix_build", "hb_hmatrix_matvec", "hb_hmatrix_matvec_device",
                 "hb_hmatrix_tree_order"):
        getattr(L, name).restype = ctypes.c_int
    L.hb_chebyshev_nodes.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]
    L.hb_interpolation_decay.argtypes = [c_p, ctypes.POINTER(hb_kernel), c_p, ctypes.c_int64,
                                         ctypes.POINTER(hb_cube), ctypes.POINTER(ctypes.c_int32),
                                         ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]
    L.hb_fit_decay_rate.argtypes = [ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double),
                                    ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]
    L.hb_v_d_constant.argtypes = [ctypes.c_int32, ctypes.c_double, ctypes.POINTER(ctypes.c_double)]
    for name in ("hb_chebyshev_nodes", "hb_interpolation_decay", "hb_fit_decay_rate", "hb_v_d_constant"):
        getattr(L, name).restype = ctypes.c_int
    L.hb_interaction_dprime.argtypes = [hb_interaction]
    L.hb_interaction_dprime.restype = ctypes.c_int32
    L.hb_assemble_dense_host.argtypes = [c_p, ctypes.POINTER(hb_kernel), c_p, ctypes.c_int64, c_p,
                                         ctypes.c_int64, ctypes.c_int32, c_p, ctypes.c_int64,
                                         ctypes.c_int64]
    L.hb_eval_radial_host.argtypes = [ctypes.POINTER(hb_kernel), ctypes.c_double,
                                      ctypes.POINTER(ctypes.c_double)]
    L.hb_rank_matrix.argtypes = [c_p, c_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.POINTER(ctypes.c_double), ctypes.c_int32,
                                 ctypes.POINTER(hb_rank_result)]
    L.hb_rank.argtypes = [c_p, ctypes.POINTER(hb_kernel), ctypes.POINTER(hb_pair),
                          ctypes.POINTER(ctypes.c_double), ctypes.c_int32,
                          ctypes.POINTER(hb_rank_result)]
    L.hb_rank_complex.argtypes = [c_p, ctypes.POINTER(hb_kernel), ctypes.POINTER(hb_kernel),
                                  ctypes.POINTER(hb_pair), ctypes.POINTER(ctypes.c_double),
                                  ctypes.c_int32, ctypes.POINTER(hb_rank_result)]
    L.hb_rank_complex.restype = ctypes.c_int
    L.hb_last_sigma.argtypes = [c_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int64,
                                ctypes.POINTER(ctypes.c_int64)]
    L.hb_sweep.argtypes = [ctypes.POINTER(hb_problem), ctypes.c_int64,
                           ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                           ctypes.POINTER(hb_rank_result), ctypes.POINTER(ctypes.c_int32)]
    L.hb_partition.argtypes = [ctypes.POINTER(hb_problem), ctypes.c_int64, ctypes.c_int32,
                               ctypes.POINTER(ctypes.c_int32)]
    L.hb_problem_seed.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64]
    L.hb_problem_seed.restype = ctypes.c_uint64
    L.hb_phase_name.argtypes = [ctypes.c_int32]
    L.hb_phase_name.restype = ctypes.c_char_p
    L.hb_context_set_profiling.argtypes = [c_p, ctypes.c_int32]
    L.hb_stats_get.argtypes = [c_p, ctypes.POINTER(hb_stats)]
    L.hb_stats_reset.argtypes = [c_p]
    L.hb_sweep_ex.argtypes = [ctypes.POINTER(hb_problem), ctypes.c_int64,
                              ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                              ctypes.POINTER(hb_rank_result), ctypes.POINTER(ctypes.c_int32),
                              ctypes.POINTER(hb_sweep_opts)]
    L.hb_sweep_release.argtypes = []
    L.hb_sweep_release.restype = None
    dg = [c_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
          c_p, ctypes.c_int64, c_p, ctypes.c_int64, ctypes.c_double, c_p, ctypes.c_int64]
    L.hb_debug_dgemm.argtypes = dg
    L.hb_debug_dgemm_async.argtypes = dg + [ctypes.c_int32]
    L.hb_debug_dgemm_fro.argtypes = dg + [ctypes.c_int64, ctypes.POINTER(ctypes.c_double)]
    L.hb_debug_dgemm_fro.restype = ctypes.c_int
    L.hb_aca_compress.argtypes = [c_p, ctypes.POINTER(hb_kernel), c_p, ctypes.c_int64, c_p,
                                  ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(hb_block),
                                  ctypes.c_int64, ctypes.c_double, ctypes.c_int64,
                                  ctypes.POINTER(c_p)]
    L.hb_aca_factor_info.argtypes = [c_p, ctypes.POINTER(ctypes.c_int32),
                                     ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)]
    L.hb_aca_factor_copy.argtypes = [c_p, c_p, c_p, c_p, c_p]
    L.hb_aca_apply.argtypes = [c_p, c_p, ctypes.POINTER(hb_kernel), c_p, ctypes.c_int64, c_p,
                               ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(hb_block), c_p, c_p]
    L.hb_aca_factor_destroy.argtypes = [c_p]
    L.hb_aca_factor_destroy.restype = None
    for name in ("hb_aca_compress", "hb_aca_factor_info", "hb_aca_factor_copy", "hb_aca_apply"):
        getattr(L, name).restype = ctypes.c_int
    for name in ("hb_context_create", "hb_context_set_tuning", "hb_generate_points",
                 "hb_assemble", "hb_eval_radial_host", "hb_rank_matrix", "hb_rank",
                 "hb_last_sigma", "hb_sweep", "hb_partition", "hb_context_set_profiling",
                 "hb_stats_get", "hb_stats_reset", "hb_sweep_ex", "hb_debug_dgemm",
                 "hb_debug_dgemm_async", "hb_classify_pair", "hb_classify_cubes",
                 "hb_assemble_dense_host"):
        getattr(L, name).restype = ctypes.c_int
    if path is None:
        _lib = L
    return L


def _check(status: int, where: str, ctx=None):
    if status != OK:
        L = load()
        detail = L.hb_last_error(ctx).decode() if ctx is not None else L.hb_last_error(None).decode()
        raise HBError(status, where, detail)


# ---- descriptors mirroring the reference value types ------------------------------------------

def make_kernel(name_or_id, diagonal: float | None = "catalog") -> hb_kernel:
    """KernelSpec::catalog(id) (kernel.hpp:40-67); diagonal=None -> no diagonal value."""
    kid = KERNEL_IDS[name_or_id] if isinstance(name_or_id, str) else int(name_or_id)
    k = hb_kernel()
    k.id = kid
    if diagonal == "catalog":
        if kid in CATALOG_DIAG:
            k.has_diag, k.diag = 1, CATALOG_DIAG[kid]
    elif diagonal is not None:
        k.has_diag, k.diag = 1, float(diagonal)
    return k


def make_cube(lower: Sequence[float], side: float = 1.0) -> hb_cube:
    c = hb_cube()
    c.d = len(lower)
    for i, v in enumerate(lower):
        c.lower[i] = float(v)
    c.side = float(side)
    return c


def offset(d: int, dprime: int | None) -> list[float]:
    """Source-cube offset: far-field (2,0,..,0); d'-surface: d-d' leading ones."""
    o = [0.0] * d
    if dprime is None or dprime < 0:
        o[0] = 2.0
    else:
        for i in range(d - dprime):
            o[i] = 1.0
    return o


def make_pair(d: int, dprime: int | None, n: int, mode: int = UNIFORM, seed: int = 0,
              n_source: int | None = None) -> hb_pair:
    p = hb_pair()
    p.target = make_cube([0.0] * d)
    p.source = make_cube(offset(d, dprime))
    p.d_prime = -1 if dprime is None else int(dprime)
    p.point_mode = mode
    p.n_target = n
    p.n_source = n if n_source is None else n_source
    p.seed = seed & 0xFFFFFFFFFFFFFFFF
    return p


def problem_seed(base: int, d: int, dprime: int | None, n: int) -> int:
    return int(load().hb_problem_seed(base & 0xFFFFFFFFFFFFFFFF, d,
                                      -1 if dprime is None else dprime, n))


def make_problem(kernel: str, d: int, dprime: int | None, n: int, tols: Sequence[float],
                 mode: int = UNIFORM, seed: int | None = None, base_seed: int = 0) -> hb_problem:
    pr = hb_problem()
    pr.kernel = make_kernel(kernel)
    s = problem_seed(base_seed, d, dprime, n) if seed is None else seed
    pr.pair = make_pair(d, dprime, n, mode, s)
    for i, t in enumerate(tols):
        pr.tols[i] = float(t)
    pr.ntol = len(tols)
    return pr


def eval_radial_host(kernel: hb_kernel, r: float) -> float:
    out = ctypes.c_double()
    _check(load().hb_eval_radial_host(ctypes.byref(kernel), float(r), ctypes.byref(out)),
           "hb_eval_radial_host")
    return out.value


def classify_pair(level_a: int, grid_a: Sequence[int], level_b: int, grid_b: Sequence[int]):
    """hodlr::classify_pair (geometry.hpp:109-118) -> (kind, d') with kind IC_SELF / IC_SURFACE /
    IC_FAR.  Raises HBError(EINVAL) for different levels or dimensions, like the reference."""
    if len(grid_a) != len(grid_b):
        raise HBError(EINVAL, "classify_pair", "boxes have different dimensions")
    d = len(grid_a)
    ga = (ctypes.c_int32 * max(d, 1))(*grid_a)
    gb = (ctypes.c_int32 * max(d, 1))(*grid_b)
    out = hb_interaction()
    _check(load().hb_classify_pair(d, level_a, ga, level_b, gb, ctypes.byref(out)), "hb_classify_pair")
    return out.kind, out.surface_dim


def fit_growth(ns: Sequence[int], ranks: Sequence[float]) -> dict:
    """SPEC fit_growth through hb_fit_growth: constant / a + b ln N / a N^c."""
    n = len(ns)
    cn = (ctypes.c_int64 * max(n, 1))(*[int(v) for v in ns])
    cr = (ctypes.c_double * max(n, 1))(*[float(v) for v in ranks])
    out = hb_growth_fit()
    _check(load().hb_fit_growth(cn, cr, n, ctypes.byref(out)), "hb_fit_growth")
    return {"best": GROWTH_MODELS[out.best], "n": out.n, "constant": out.constant,
            "log": (out.log_a, out.log_b), "power": (out.pow_a, out.pow_c),
            "rss": dict(zip(GROWTH_MODELS, list(out.rss))), "max_min_ratio": out.max_min_ratio}


def chebyshev_nodes(p: int) -> list[float]:
    """hodlr::chebyshev_nodes (chebyshev.hpp:16-23)."""
    out = (ctypes.c_double * max(p + 1, 1))()
    _check(load().hb_chebyshev_nodes(p, out), "hb_chebyshev_nodes")
    return list(out[: p + 1])


def fit_decay_rate(ps: Sequence[int], errs: Sequence[float]) -> float:
    """hodlr::fit_decay_rate (chebyshev.hpp:180-193)."""
    n = len(ps)
    cp = (ctypes.c_int32 * max(n, 1))(*ps)
    ce = (ctypes.c_double * max(n, 1))(*errs)
    rho = ctypes.c_double()
    _check(load().hb_fit_decay_rate(cp, ce, n, ctypes.byref(rho)), "hb_fit_decay_rate")
    return rho.value


def v_d_constant(d: int, rho: float) -> float:
    """hodlr::v_d_constant (chebyshev.hpp:139-147)."""
    out = ctypes.c_double()
    _check(load().hb_v_d_constant(d, rho, ctypes.byref(out)), "hb_v_d_constant")
    return out.value


def classify_cubes(a: hb_cube, b: hb_cube):
    out = hb_interaction()
    _check(load().hb_classify_cubes(ctypes.byref(a), ctypes.byref(b), ctypes.byref(out)),
           "hb_classify_cubes")
    return out.kind, out.surface_dim


@dataclass
class RankResult:
    rank: int
    rank_lo: int
    rank_hi: int
    k_factored: int
    sigma1: float
    sigma_r: float
    sigma_r1: float
    gap: float
    resid: float
    sec: list
    certificate: int = 0  # 1 deterministic bracket, 2 probabilistic (<1e-27), 0 open
    fp_band: float = 0.0  # sqrt(N)·u·‖A‖_F / thr; gap < fp_band: rounding-sensitive count

    @classmethod
    def of(cls, r: hb_rank_result) -> "RankResult":
        return cls(r.rank, r.rank_lo, r.rank_hi, r.k_factored, r.sigma1, r.sigma_r, r.sigma_r1,
                   r.gap, r.resid, list(r.sec), r.certificate, r.fp_band)

    @property
    def in_fp_band(self) -> bool:
        return self.gap < self.fp_band


class Context:
    """One device, one CUDA stream (hb_context)."""

    def __init__(self, device: int = 0):
        self._lib = load()
        self._h = ctypes.c_void_p()
        _check(self._lib.hb_context_create(device, ctypes.byref(self._h)), "hb_context_create")
        self.device = device

    def close(self):
        if self._h:
            self._lib.hb_context_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(self._lib.hb_context_stream(self._h) or 0)

    def set_tuning(self, block_max: int = 120, eta: float = 0.01):
        _check(self._lib.hb_context_set_tuning(self._h, block_max, eta), "set_tuning", self._h)

    def generate_points(self, pair: hb_pair, d_tgt_ptr: int, d_src_ptr: int):
        _check(self._lib.hb_generate_points(self._h, ctypes.byref(pair), d_tgt_ptr, d_src_ptr),
               "hb_generate_points", self._h)

    def assemble(self, kernel: hb_kernel, d_tgt: int, T: int, d_src: int, N: int, d: int,
                 d_K: int, ldk: int):
        _check(self._lib.hb_assemble(self._h, ctypes.byref(kernel), d_tgt, T, d_src, N, d, d_K,
                                     ldk), "hb_assemble", self._h)

    def assemble_dense_host(self, kernel: hb_kernel, targets, sources, entry_cap: int = 400_000_000):
        """hodlr::assemble_dense (kernel.hpp:168-181) on host point sets: targets (d, T) and
        sources (d, N) SoA float64 arrays (the PointSet layout) -> host K (T, N), Fortran order."""
        import numpy as np
        x = np.ascontiguousarray(targets, dtype=np.float64)
        y = np.ascontiguousarray(sources, dtype=np.float64)
        d, T = x.shape
        d2, N = y.shape
        if d != d2:
            raise HBError(EINVAL, "assemble_dense", "point dimensions differ")
        K = np.empty((T, N), dtype=np.float64, order="F")
        _check(self._lib.hb_assemble_dense_host(self._h, ctypes.byref(kernel), x.ctypes.data, T,
                                                y.ctypes.data, N, d, K.ctypes.data, T, entry_cap),
               "hb_assemble_dense_host", self._h)
        return K

    def interpolation_decay(self, kernel: hb_kernel, targets, cube: hb_cube,
                            p_list: Sequence[int]) -> list[tuple[int, float]]:
        """hodlr::interpolation_decay (chebyshev.hpp:151-177) on the device: (p, max entry error
        of the degree-p tensor Chebyshev interpolant along `cube`) for each p; targets (d, T)."""
        import numpy as np
        x = np.ascontiguousarray(targets, dtype=np.float64)
        d, T = x.shape
        n = len(p_list)
        cp = (ctypes.c_int32 * max(n, 1))(*p_list)
        out = (ctypes.c_double * max(n, 1))()
        _check(self._lib.hb_interpolation_decay(self._h, ctypes.byref(kernel), x.ctypes.data, T,
                                                ctypes.byref(cube), cp, n, out),
               "hb_interpolation_decay", self._h)
        return list(zip(list(p_list), list(out[:n])))

    def rank(self, kernel: hb_kernel, pair: hb_pair, tols: Sequence[float]) -> list[RankResult]:
        nt = len(tols)
        ct = (ctypes.c_double * nt)(*tols)
        out = (hb_rank_result * nt)()
        _check(self._lib.hb_rank(self._h, ctypes.byref(kernel), ctypes.byref(pair), ct, nt, out),
               "hb_rank", self._h)
        return [RankResult.of(o) for o in out]

    def rank_complex(self, kernel_re: hb_kernel, kernel_im: hb_kernel, pair: hb_pair,
                     tols: Sequence[float]) -> list[RankResult]:
        """ε-rank of K_re + i·K_im (the paper's complex F3 / F4 kernels) via the real embedding."""
        nt = len(tols)
        ct = (ctypes.c_double * nt)(*tols)
        out = (hb_rank_result * nt)()
        _check(self._lib.hb_rank_complex(self._h, ctypes.byref(kernel_re), ctypes.byref(kernel_im),
                                         ctypes.byref(pair), ct, nt, out), "hb_rank_complex", self._h)
        return [RankResult.of(o) for o in out]

    def rank_matrix(self, d_A: int, m: int, n: int, ld: int, tols: Sequence[float]):
        nt = len(tols)
        ct = (ctypes.c_double * nt)(*tols)
        out = (hb_rank_result * nt)()
        _check(self._lib.hb_rank_matrix(self._h, d_A, m, n, ld, ct, nt, out), "hb_rank_matrix",
               self._h)
        return [RankResult.of(o) for o in out]

    def set_stopping(self, spectral: bool = True):
        _check(self._lib.hb_context_set_stopping(self._h, int(spectral)), "set_stopping", self._h)

    def set_profiling(self, on: bool = True):
        _check(self._lib.hb_context_set_profiling(self._h, int(on)), "set_profiling", self._h)

    def stats(self) -> dict:
        st = hb_stats()
        _check(self._lib.hb_stats_get(self._h, ctypes.byref(st)), "hb_stats_get", self._h)
        return st.as_dict()

    def dgemm(self, transA: bool, M: int, N: int, K: int, alpha: float, A: int, lda: int, B: int,
              ldb: int, beta: float, C: int, ldc: int, reps: int = 0):
        """Test hook (include/hb_debug.h): FP64 DMMA GEMM on device pointers; reps>0: async."""
        if reps:
            _check(self._lib.hb_debug_dgemm_async(self._h, int(transA), M, N, K, alpha, A, lda, B,
                                                  ldb, beta, C, ldc, reps), "dgemm", self._h)
        else:
            _check(self._lib.hb_debug_dgemm(self._h, int(transA), M, N, K, alpha, A, lda, B, ldb,
                                            beta, C, ldc), "dgemm", self._h)

    def dgemm_fro(self, transA: bool, M: int, N: int, K: int, alpha: float, A: int, lda: int,
                  B: int, ldb: int, beta: float, C: int, ldc: int, fro_row0: int) -> float:
        """Test hook: the GEMM with the trailing update's Frobenius epilogue; returns the sum of
        squares of the new C over rows >= fro_row0."""
        out = ctypes.c_double()
        _check(self._lib.hb_debug_dgemm_fro(self._h, int(transA), M, N, K, alpha, A, lda, B, ldb,
                                            beta, C, ldc, fro_row0, ctypes.byref(out)),
               "dgemm_fro", self._h)
        return out.value

    def aca_compress(self, kernel: hb_kernel, d_tgt: int, nt: int, d_src: int, ns: int, d: int,
                     blocks, eps: float, max_rank: int) -> list["ACAFactor"]:
        """hodlr::compress (aca.hpp:171-198) of each block (hb_block or (rb, rows, cb, cols))."""
        bl = [b if isinstance(b, hb_block) else hb_block(*b) for b in blocks]
        arr = (hb_block * max(len(bl), 1))(*bl)
        out = (ctypes.c_void_p * max(len(bl), 1))()
        _check(self._lib.hb_aca_compress(self._h, ctypes.byref(kernel), d_tgt, nt, d_src, ns, d,
                                         arr, len(bl), eps, max_rank, out), "hb_aca_compress",
               self._h)
        return [ACAFactor(self._lib, out[i], bl[i]) for i in range(len(bl))]

    def aca_apply(self, f: "ACAFactor", kernel: hb_kernel, d_tgt: int, nt: int, d_src: int,
                  ns: int, d: int, d_q: int, d_b: int, block: hb_block | None = None):
        """hodlr::apply (aca.hpp:202-213): b = K(I,τ) U⁻¹ L⁻¹ K(σ,J) q on device vectors."""
        blk = f.block if block is None else block
        _check(self._lib.hb_aca_apply(self._h, f._h, ctypes.byref(kernel), d_tgt, nt, d_src, ns, d,
                                      ctypes.byref(blk), d_q, d_b), "hb_aca_apply", self._h)

    def last_sigma(self, max_count: int | None = None) -> list[float]:
        cnt = ctypes.c_int64()
        _check(self._lib.hb_last_sigma(self._h, None, 0, ctypes.byref(cnt)), "hb_last_sigma",
               self._h)
        k = cnt.value if max_count is None else min(cnt.value, max_count)
        buf = (ctypes.c_double * max(k, 1))()
        _check(self._lib.hb_last_sigma(self._h, buf, k, ctypes.byref(cnt)), "hb_last_sigma",
               self._h)
        return list(buf[:k])


class HMatrix:
    """HODLRdD operator on the device (hmatrix.hpp:50-179): hodlr::HMatrix::initialize + matvec.
    points: (d, N) host array; domain: hb_cube; policy: "weakdd" | "strong" | "weakall"."""

    def __init__(self, ctx: "Context", kernel: hb_kernel, points, domain: hb_cube,
                 policy: str = "weakdd", n_max: int = 1000, epsilon: float = 1e-6,
                 max_rank: int = 1 << 14, dense_entry_cap: int = 0):
        import numpy as np
        self._lib = load()
        self._ctx = ctx  # the operator runs on (and keeps) this context
        x = np.ascontiguousarray(points, dtype=np.float64)
        self.d, self.n = x.shape
        self._h = ctypes.c_void_p()
        rep = hb_build_report()
        _check(self._lib.hb_hmatrix_build(ctx._h, ctypes.byref(kernel), x.ctypes.data, self.n, self.d,
                                          ctypes.byref(domain), POLICIES[policy], n_max, epsilon,
                                          max_rank, dense_entry_cap, ctypes.byref(self._h),
                                          ctypes.byref(rep)), "hb_hmatrix_build", ctx._h)
        self.report = rep.as_dict()

    def matvec(self, q):
        """b = H q in the original ordering; q of shape (N,) or (N, nvec)."""
        import numpy as np
        qq = np.asfortranarray(np.asarray(q, dtype=np.float64).reshape(self.n, -1))
        b = np.zeros_like(qq)
        _check(self._lib.hb_hmatrix_matvec(self._h, qq.ctypes.data, b.ctypes.data, qq.shape[1]),
               "hb_hmatrix_matvec", self._ctx._h)
        return b.reshape(np.shape(q))

    def matvec_device(self, d_q: int, d_b: int):
        _check(self._lib.hb_hmatrix_matvec_device(self._h, d_q, d_b), "hb_hmatrix_matvec_device",
               self._ctx._h)

    def tree_order(self):
        import numpy as np
        out = np.zeros(self.n, np.int64)
        _check(self._lib.hb_hmatrix_tree_order(self._h, out.ctypes.data), "hb_hmatrix_tree_order")
        return out

    def close(self):
        if self._h:
            self._lib.hb_hmatrix_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ACAFactor:
    """hodlr::ACAFactor (aca.hpp:50-62): pivots, unit-lower L and upper U stay on the device;
    .sigma / .tau / .L / .U copy them out (numpy)."""

    def __init__(self, lib, handle, block: hb_block):
        self._lib = lib
        self._h = ctypes.c_void_p(handle)
        self.block = block
        r, met, mem = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
        _check(lib.hb_aca_factor_info(self._h, ctypes.byref(r), ctypes.byref(met), ctypes.byref(mem)),
               "hb_aca_factor_info")
        self.rank, self.tolerance_met, self.memory_bytes = r.value, bool(met.value), mem.value

    def arrays(self):
        import numpy as np
        r = self.rank
        sig = np.zeros(max(r, 1), np.int64)
        tau = np.zeros(max(r, 1), np.int64)
        L = np.zeros(max(r * r, 1))
        U = np.zeros(max(r * r, 1))
        _check(self._lib.hb_aca_factor_copy(self._h, sig.ctypes.data, tau.ctypes.data,
                                            L.ctypes.data, U.ctypes.data), "hb_aca_factor_copy")
        return (sig[:r], tau[:r], L[:r * r].reshape(r, r, order="F"),
                U[:r * r].reshape(r, r, order="F"))

    def close(self):
        if self._h:
            self._lib.hb_aca_factor_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partition(problems: Sequence[hb_problem], nparts: int) -> list[int]:
    n = len(problems)
    arr = (hb_problem * max(n, 1))(*problems)
    own = (ctypes.c_int32 * max(n, 1))()
    _check(load().hb_partition(arr, n, nparts, own), "hb_partition")
    return list(own[:n])


def sweep(problems: Sequence[hb_problem], devices: Sequence[int] = (0,), profiling: bool = False,
          with_times: bool = False):
    """hb_sweep_ex: returns (results per problem [list per tol], statuses[, device seconds])."""
    n = len(problems)
    arr = (hb_problem * max(n, 1))(*problems)
    total = sum(p.ntol for p in problems)
    out = (hb_rank_result * max(total, 1))()
    st = (ctypes.c_int32 * max(n, 1))(*([-1] * max(n, 1)))  # -1: never written by the library
    devs = (ctypes.c_int32 * len(devices))(*devices)
    opts = hb_sweep_opts()
    opts.profiling = int(profiling)
    ret = load().hb_sweep_ex(arr, n, devs, len(devices), out, st, ctypes.byref(opts))
    if n and any(v == -1 for v in st[:n]):  # an early failure (bad arguments) before any problem ran
        _check(ret if ret != OK else EINVAL, "hb_sweep_ex")
    res, o = [], 0
    for p in problems:
        res.append([RankResult.of(out[o + t]) for t in range(p.ntol)])
        o += p.ntol
    if with_times:
        return res, list(st[:n]), list(opts.device_seconds[:len(devices)])
    return res, list(st[:n])


def global_stats() -> dict:
    st = hb_stats()
    _check(load().hb_stats_get(None, ctypes.byref(st)), "hb_stats_get")
    return st.as_dict()


def reset_global_stats():
    load().hb_stats_reset(None)


def sweep_release():
    load().hb_sweep_release()
