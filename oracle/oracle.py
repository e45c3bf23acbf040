"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Python face of the oracle: ctypes over ``oracle/_build/libhb_oracle.so`` (the plain-C entry
restatement, see hb_oracle.h for file:line citations) plus the ε-rank restated with numpy's
LAPACK SVD.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or the timed CPU
baseline.  The product package ``paper_2209_05819_b200`` never imports it.

Rank semantics (the oracle's contract):
  * ε-rank = count of σ_k > tol·σ₁  — PAPER.md:141-145 (doc A definition; the tables report
    this count), SPEC.md:560-568,606-609 (``epsilon_rank`` reports count-above-threshold).
  * σ from LAPACK ``dgesdd`` (numpy.linalg.svd, compute_uv=False), i.e. a LAPACK-class full
    SVD as SPEC ``epsilon_rank`` prescribes ("computes full singular values").
  * gap = min(σ_p/thr − 1, 1 − σ_{p+1}/thr): the distance of the nearest σ to the threshold,
    reported with every rank so that boundary ties are visible (BASELINE.json north_star).
Geometry (SPEC.md:537-558 ``pair_geometry``, corrected per SURVEY.md A.1): target cube
[0,1]^d, source cube = target + o with o = (2,0,..,0) far-field, or d−d' leading ones for a
d'-dimensional shared surface; interior grid (i+1)/(n+1) for near-field tables, closed grid
i/(n−1) for far-field tables, i.i.d. uniform points from a seed for the BASELINE configs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libhb_oracle.so"

UNIFORM, GRID_INTERIOR, GRID_CLOSED = 0, 1, 2
KERNEL_IDS = {  # kernel.hpp:19-32 order, names kernel.hpp:112-129
    "one_over_r": 0, "log_r": 1, "helmholtz3d_re": 2, "helmholtz3d_im": 3,
    "hankel_h12_re": 4, "hankel_h12_im": 5, "r": 6, "sin_r": 7,
    "inv_sqrt_1_plus_r": 8, "exp_neg_r": 9, "exp_neg_r2": 10,
}
# kernel.hpp:46-61 catalog diagonal values
CATALOG_DIAG = {0: 0.0, 1: 0.0, 2: 0.0, 5: 0.0, 3: 1.0, 8: 1.0, 9: 1.0, 10: 1.0, 4: 0.0, 6: 0.0,
                7: 0.0}

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        L.hbo_points.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_double,
                                 ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                 ctypes.c_void_p]
        L.hbo_assemble.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_void_p,
                                   ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                   ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64]
        L.hbo_splitmix64.argtypes = [ctypes.c_uint64]
        L.hbo_splitmix64.restype = ctypes.c_uint64
        L.hbo_eval_radial.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_double, ctypes.POINTER(ctypes.c_int)]
        L.hbo_eval_radial.restype = ctypes.c_double
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: status {status}")
        self.status = status


def splitmix64(x: int) -> int:
    return int(lib().hbo_splitmix64(x & 0xFFFFFFFFFFFFFFFF))


def problem_seed(base: int, d: int, dprime: int | None, n: int) -> int:
    """Per-problem seed = hash(base_seed, d, d', N); dprime None = far."""
    dp = -1 if dprime is None else dprime
    key = (d << 48) | ((dp + 1) << 40) | n
    return splitmix64(base ^ splitmix64(key))


def offset(d: int, dprime: int | None) -> np.ndarray:
    o = np.zeros(d)
    if dprime is None:
        o[0] = 2.0
    else:
        o[: d - dprime] = 1.0
    return o


def points(d: int, lower, side: float, n: int, mode: int, seed: int, role: int) -> np.ndarray:
    lo = (ctypes.c_double * d)(*[float(v) for v in lower])
    out = np.empty((d, n), dtype=np.float64)
    st = lib().hbo_points(d, lo, side, n, mode, seed, role, out.ctypes.data)
    if st:
        raise OracleError(st, "hbo_points")
    return out


def pair_points(d: int, dprime: int | None, n: int, mode: int, seed: int):
    """(targets, sources) SoA arrays of shape (d, n)."""
    x = points(d, np.zeros(d), 1.0, n, mode, seed, 0)
    y = points(d, offset(d, dprime), 1.0, n, mode, seed, 1)
    return x, y


def assemble(kernel_id: int, x: np.ndarray, y: np.ndarray, has_diag: bool = True,
             diag: float | None = None, nthreads: int = 1, entry_cap: int = 0) -> np.ndarray:
    d, T = x.shape
    d2, N = y.shape
    if d != d2:
        raise OracleError(1, "dimension mismatch")
    if diag is None:
        diag = CATALOG_DIAG.get(kernel_id, 0.0)
    K = np.empty((T, N), dtype=np.float64, order="F")
    st = lib().hbo_assemble(kernel_id, int(has_diag), float(diag),
                            np.ascontiguousarray(x).ctypes.data, T,
                            np.ascontiguousarray(y).ctypes.data, N, d, K.ctypes.data, T,
                            nthreads, entry_cap)
    if st:
        raise OracleError(st, "hbo_assemble")
    return K


def eval_radial(kernel_id: int, r: float, has_diag: bool = True, diag: float | None = None):
    if diag is None:
        diag = CATALOG_DIAG.get(kernel_id, 0.0)
    st = ctypes.c_int(0)
    v = lib().hbo_eval_radial(kernel_id, int(has_diag), float(diag), float(r), ctypes.byref(st))
    if st.value:
        raise OracleError(st.value, "hbo_eval_radial")
    return v


def singular_values(K: np.ndarray) -> np.ndarray:
    if not np.all(np.isfinite(K)):
        raise OracleError(2, "non-finite entries")  # SPEC.md:564 numeric error
    return np.linalg.svd(K, compute_uv=False)


@dataclass
class RankRecord:
    rank: int
    sigma1: float
    sigma_r: float   # σ_p (0 if p == 0)
    sigma_r1: float  # σ_{p+1} (0 if p == min(m, n))
    gap: float


def epsilon_rank_from_sigma(s: np.ndarray, tol: float) -> RankRecord:
    s1 = float(s[0]) if len(s) else 0.0
    thr = tol * s1
    p = int(np.count_nonzero(s > thr))
    sp = float(s[p - 1]) if p > 0 else 0.0
    sp1 = float(s[p]) if p < len(s) else 0.0
    if thr > 0:
        up = sp / thr - 1.0 if p > 0 else np.inf
        lo = 1.0 - sp1 / thr if p < len(s) else np.inf
        gap = float(min(up, lo))
    else:
        gap = float("inf")
    return RankRecord(p, s1, sp, sp1, gap)


def epsilon_rank(K: np.ndarray, tol: float) -> RankRecord:
    return epsilon_rank_from_sigma(singular_values(K), tol)


def rank_problem(d: int, dprime: int | None, kernel: str, n: int, tols, mode: int = UNIFORM,
                 seed: int = 0, nthreads: int = None) -> list[RankRecord]:
    nthreads = nthreads or os.cpu_count() or 1
    x, y = pair_points(d, dprime, n, mode, seed)
    K = assemble(KERNEL_IDS[kernel], x, y, nthreads=nthreads)
    s = singular_values(K)
    return [epsilon_rank_from_sigma(s, t) for t in tols]


def rank_problem_complex(d: int, dprime: int | None, kernel_re: str, kernel_im: str, n: int, tols,
                         mode: int = UNIFORM, seed: int = 0, nthreads: int = None) -> list[RankRecord]:
    """ε-rank of K_re + i·K_im (the paper's complex F3 = e^{ir}/r and F4 = H_2^(1)(r) columns,
    PAPER.md:121-131, from the reference's real/imaginary kernel pairs kernel.hpp:22-27) with
    numpy's complex LAPACK SVD (zgesdd)."""
    nthreads = nthreads or os.cpu_count() or 1
    x, y = pair_points(d, dprime, n, mode, seed)
    A = assemble(KERNEL_IDS[kernel_re], x, y, nthreads=nthreads)
    B = assemble(KERNEL_IDS[kernel_im], x, y, nthreads=nthreads)
    s = singular_values(A + 1j * B)
    return [epsilon_rank_from_sigma(s, t) for t in tols]


COMPLEX_COLUMNS = {"F3": ("helmholtz3d_re", "helmholtz3d_im"), "F4": ("hankel_h12_re", "hankel_h12_im")}


# ---- ACA (aca.hpp:16-213) and the compiled reference (oracle/_ref) -----------------------------
REF_LIB = HERE / "_ref" / "libhb_ref.so"
_ref = None
_ACA_ARGS = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_int64,
             ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
             ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_int64, ctypes.c_int64,
             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
             ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32), ctypes.c_void_p,
             ctypes.c_void_p]


def ref_available() -> bool:
    """True when oracle/_ref/libhb_ref.so (the reference's own headers compiled here) exists."""
    return REF_LIB.exists()


def ref_lib():
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise OracleError(5, f"{REF_LIB} not built (needs /root/reference; see oracle/Makefile)")
        L = ctypes.CDLL(str(REF_LIB))
        L.hbr_aca_compress.argtypes = _ACA_ARGS
        L.hbr_assemble_dense.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                         ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_int64]
        L.hbr_eval_radial.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_double, ctypes.POINTER(ctypes.c_int)]
        L.hbr_eval_radial.restype = ctypes.c_double
        L.hbr_classify_pair.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.hbr_box_grid.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p]
        L.hbr_chebyshev_nodes.argtypes = [ctypes.c_int, ctypes.c_void_p]
        L.hbr_lagrange_weights.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
        L.hbr_interpolation_decay.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                              ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p,
                                              ctypes.c_int, ctypes.c_void_p]
        L.hbr_fit_decay_rate.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        L.hbr_v_d_constant.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
        L.hbr_hmatrix_matvec.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_void_p,
                                         ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_double,
                                         ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_int64,
                                         ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p]
        for f in ("hbr_j2", "hbr_y2"):
            getattr(L, f).argtypes = [ctypes.c_double]
            getattr(L, f).restype = ctypes.c_double
        _ref = L
    return _ref


def ref_assemble(kernel_id: int, x: np.ndarray, y: np.ndarray, has_diag: bool = True,
                 diag: float | None = None, entry_cap: int = 400_000_000) -> np.ndarray:
    """hodlr::assemble_dense (kernel.hpp:168-181) itself, compiled from /root/reference."""
    d, T = x.shape
    _, N = y.shape
    if diag is None:
        diag = CATALOG_DIAG.get(kernel_id, 0.0)
    K = np.empty((T, N), dtype=np.float64, order="F")
    st = ref_lib().hbr_assemble_dense(kernel_id, int(has_diag), float(diag),
                                      np.ascontiguousarray(x).ctypes.data, T,
                                      np.ascontiguousarray(y).ctypes.data, N, d, K.ctypes.data,
                                      entry_cap)
    if st:
        raise OracleError(st, "hbr_assemble_dense")
    return K


@dataclass
class ACAResult:
    rank: int
    met: bool
    sigma: np.ndarray  # global target ids of the row pivots
    tau: np.ndarray    # global source ids of the column pivots
    L: np.ndarray      # rank x rank unit lower
    U: np.ndarray      # rank x rank upper, pivots on the diagonal
    b: np.ndarray | None = None  # apply(q) if q was given


def aca_compress(kernel_id: int, x: np.ndarray, y: np.ndarray, eps: float, max_rank: int,
                 rb: int = 0, rows: int | None = None, cb: int = 0, cols: int | None = None,
                 q: np.ndarray | None = None, has_diag: bool = True, diag: float | None = None,
                 impl: str = "oracle") -> ACAResult:
    """hodlr::compress (+ apply) on BlockSpec(kernel, x, rb, rows, y, cb, cols).
    impl="oracle": the C restatement (hb_oracle.c); impl="ref": the reference's aca.hpp
    compiled in place (oracle/_ref)."""
    d, nt = x.shape
    _, ns = y.shape
    rows = nt - rb if rows is None else rows
    cols = ns - cb if cols is None else cols
    if diag is None:
        diag = CATALOG_DIAG.get(kernel_id, 0.0)
    cap = max(1, min(rows, cols, max_rank))
    sigma = np.zeros(cap, np.int64)
    tau = np.zeros(cap, np.int64)
    L = np.zeros(cap * cap)
    U = np.zeros(cap * cap)
    rk, met = ctypes.c_int32(0), ctypes.c_int32(0)
    qq = None if q is None else np.ascontiguousarray(q, dtype=np.float64)
    b = None if q is None else np.zeros(rows)
    f = ref_lib().hbr_aca_compress if impl == "ref" else lib().hbo_aca_compress
    if impl != "ref":
        f.argtypes = _ACA_ARGS
    xs, ys = np.ascontiguousarray(x), np.ascontiguousarray(y)
    st = f(kernel_id, int(has_diag), float(diag), xs.ctypes.data, nt, ys.ctypes.data, ns, d,
           rb, rows, cb, cols, float(eps), max_rank, cap, sigma.ctypes.data, tau.ctypes.data,
           L.ctypes.data, U.ctypes.data, ctypes.byref(rk), ctypes.byref(met),
           None if qq is None else qq.ctypes.data, None if b is None else b.ctypes.data)
    if st:
        raise OracleError(st, f"aca_compress[{impl}]")
    r = rk.value
    return ACAResult(r, bool(met.value), sigma[:r].copy(), tau[:r].copy(),
                     L[:r * r].reshape(r, r, order="F").copy(),
                     U[:r * r].reshape(r, r, order="F").copy(), b)


def ref_interpolation_decay(kernel_id: int, x: np.ndarray, lower, side: float, p_list,
                            has_diag: bool = True, diag: float | None = None) -> list:
    """hodlr::interpolation_decay (chebyshev.hpp:151-177) itself, compiled from /root/reference."""
    d, T = x.shape
    if diag is None:
        diag = CATALOG_DIAG.get(kernel_id, 0.0)
    lo = np.ascontiguousarray(lower, dtype=np.float64)
    ps = np.ascontiguousarray(p_list, dtype=np.int32)
    out = np.zeros(len(p_list))
    xs = np.ascontiguousarray(x)
    st = ref_lib().hbr_interpolation_decay(kernel_id, int(has_diag), float(diag), xs.ctypes.data, T, d,
                                           lo.ctypes.data, float(side), ps.ctypes.data, len(p_list),
                                           out.ctypes.data)
    if st:
        raise OracleError(st, "hbr_interpolation_decay")
    return list(zip(list(p_list), out.tolist()))


POLICIES = {"weakdd": 0, "strong": 1, "weakall": 2}  # cluster_tree.hpp:20 AdmissibilityPolicy


def ref_hmatrix_matvec(kernel_id: int, pts: np.ndarray, lower, side: float, policy: str, n_max: int,
                       eps: float, q: np.ndarray, max_rank: int = 1 << 14, has_diag: bool = True,
                       diag: float | None = None):
    """hodlr::HMatrix::initialize + matvec (hmatrix.hpp:50-179), compiled from /root/reference.
    pts (d, N); q (N,) or (N, nq).  Returns (b, report dict, perm tree -> original)."""
    d, N = pts.shape
    if diag is None:
        diag = CATALOG_DIAG.get(kernel_id, 0.0)
    qq = np.asfortranarray(q.reshape(N, -1), dtype=np.float64)
    b = np.zeros_like(qq)
    rep = np.zeros(6, np.int64)
    perm = np.zeros(N, np.int64)
    lo = np.ascontiguousarray(lower, dtype=np.float64)
    xs = np.ascontiguousarray(pts)
    st = ref_lib().hbr_hmatrix_matvec(kernel_id, int(has_diag), float(diag), xs.ctypes.data, N, d,
                                      lo.ctypes.data, float(side), POLICIES[policy], n_max, float(eps),
                                      max_rank, qq.ctypes.data, qq.shape[1], b.ctypes.data,
                                      rep.ctypes.data, perm.ctypes.data)
    if st:
        raise OracleError(st, "hbr_hmatrix_matvec")
    keys = ["max_block_rank", "num_low_rank_blocks", "num_dense_entries", "num_tolerance_failures",
            "memory_bytes", "depth"]
    return b.reshape(q.shape), dict(zip(keys, rep.tolist())), perm

