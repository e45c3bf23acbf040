"""CPU ORACLE — TEST INFRASTRUCTURE ONLY: the certified large-N ε-rank route.

A full LAPACK SVD (oracle.py, ``gesdd``) is O(N³) and impractical for N ≥ 16000 on a CPU; the
reference's own driver guards dense SVD at N ≤ 20000/8000/4096.  This module
restates the certified truncated route BASELINE.md §3 / SURVEY.md §7.1 prescribe:

  1. Truncated QR with column pivoting by LAPACK ``dgeqp3rk`` (LAPACK ≥ 3.12, from the OpenBLAS
     that scipy bundles; LP64 symbol ``scipy_dgeqp3rk_``):  A·P = Q·[R11 R12; 0 A22] with k
     columns factored; the trailing residual A22 is left in A(k+1:M, k+1:N).
  2. δ = ‖A22‖_F (exact, from the residual block), an upper bound on ‖A22‖₂.
  3. σ(R_k) of the k × N top rows of R by LAPACK ``dgesdd`` (numpy.linalg.svd).
  4. Weyl: AᵀA = R_kᵀR_k + [0 A22]ᵀ[0 A22] ⇒ σ_i(R_k) ≤ σ_i(A) ≤ sqrt(σ_i(R_k)² + δ²) for every i,
     including σ₁, so with thr_lo = tol·σ₁(R_k) and thr_hi = tol·sqrt(σ₁(R_k)² + δ²)
         rank_lo = #{σ(R_k) > thr_hi}  ≤  rank = #{σ(A) > tol·σ₁(A)}  ≤  rank_hi = #{sqrt(σ(R_k)²+δ²) > thr_lo}.
     When rank_lo == rank_hi the ε-rank is certified (in exact arithmetic, see 6).
  5. If the bracket is open the factorisation resumes on the residual (a second ``dgeqp3rk`` on
     A22, its column permutation applied to R12) with a tighter stopping tolerance.
  6. Rounding: Householder QR is backward stable, so the computed factors are exact for A + E with
     ‖E‖_F ≈ c·sqrt(N)·u·‖A‖_F.  ``fp_band`` = sqrt(N)·u·‖A‖_F / thr is recorded with each rank;
     a result whose gap is below it is flagged ``in_fp_band`` (certified only up to rounding).

Rank semantics are the oracle's (oracle.py): count of σ_k > tol·σ₁ (PAPER.md:141-145,
SPEC.md:560-568).  The pivoting rule does not matter for correctness: the bracket in 4 holds for
any column order; pivoting only decides how many columns k are needed to close it.
"""
from __future__ import annotations

import ctypes
import glob
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

_lapack = None


def _lib():
    global _lapack
    if _lapack is None:
        import scipy
        base = os.path.dirname(scipy.__file__)
        cands = sorted(glob.glob(os.path.join(base, "..", "scipy.libs", "libscipy_openblas*.so")))
        if not cands:
            raise RuntimeError("scipy's bundled OpenBLAS (dgeqp3rk) not found")
        L = ctypes.CDLL(cands[0])
        _lapack = L.scipy_dgeqp3rk_
    return _lapack


_I, _D = ctypes.c_int, ctypes.c_double


def dgeqp3rk(A: np.ndarray, row0: int, col0: int, kmax: int, abstol: float, reltol: float = 0.0):
    """In-place dgeqp3rk on the Fortran-ordered view A[row0:, col0:] (lda = A.shape[0]).
    Returns (k, maxc2nrmk, jpiv (0-based, relative to col0), tau)."""
    assert A.flags.f_contiguous and A.dtype == np.float64
    lda = A.shape[0]
    m, n = lda - row0, A.shape[1] - col0
    ptr = A.ctypes.data + 8 * (col0 * lda + row0)
    jpiv = np.zeros(n, np.int32)
    tau = np.zeros(max(1, min(m, n)))
    iwork = np.zeros(max(1, n), np.int32)
    k, mx, rmx, info = _I(0), _D(0), _D(0), _I(0)
    kmax = max(0, min(kmax, m, n))

    def call(work, lwork):
        _lib()(ctypes.byref(_I(m)), ctypes.byref(_I(n)), ctypes.byref(_I(0)), ctypes.byref(_I(kmax)),
               ctypes.byref(_D(abstol)), ctypes.byref(_D(reltol)), ctypes.c_void_p(ptr),
               ctypes.byref(_I(lda)), ctypes.byref(k), ctypes.byref(mx), ctypes.byref(rmx),
               jpiv.ctypes.data_as(ctypes.c_void_p), tau.ctypes.data_as(ctypes.c_void_p),
               work.ctypes.data_as(ctypes.c_void_p), ctypes.byref(_I(lwork)),
               iwork.ctypes.data_as(ctypes.c_void_p), ctypes.byref(info))

    wq = np.zeros(1)
    call(wq, -1)
    work = np.zeros(max(1, int(wq[0])))
    call(work, work.size)
    if info.value < 0:
        raise RuntimeError(f"dgeqp3rk: illegal argument {-info.value}")
    return k.value, mx.value, jpiv - 1, tau


def sigma1_lower(A: np.ndarray, iters: int = 12, seed: int = 1) -> float:
    """Lower bound on σ₁(A): ‖A v‖ for a unit v after a few power steps on AᵀA."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(A.shape[1])
    v /= np.linalg.norm(v)
    best = 0.0
    for _ in range(iters):
        w = A @ v
        best = max(best, float(np.linalg.norm(w)))
        v = A.T @ w
        nv = np.linalg.norm(v)
        if nv == 0:
            break
        v /= nv
    return best


@dataclass
class CertifiedRank:
    ranks: list            # certified ε-rank per tol (rank_lo when the bracket stays open)
    rank_lo: list
    rank_hi: list
    sigma1: float          # σ₁(R_k) (≤ σ₁(A) ≤ sqrt(σ₁(R_k)² + δ²))
    sigma_r: list          # σ_p(R_k)
    sigma_r1: list         # σ_{p+1}(R_k)
    gaps: list             # min(σ_p/thr − 1, 1 − σ_{p+1}/thr) from σ(R_k)
    k: int                 # columns factored
    delta_F: float         # ‖A22‖_F
    fp_band: list          # sqrt(N)·u·‖A‖_F / thr
    in_fp_band: list
    seconds: dict = field(default_factory=dict)


def certified_rank(A: np.ndarray, tols, eta: float = 0.25, max_rounds: int = 64,
                   sigma1_hint: float | None = None) -> CertifiedRank:
    """Certified ε-rank of A (destroyed: overwritten by the factorisation), Fortran order."""
    t0 = time.time()
    A = np.asfortranarray(A)
    m, n = A.shape
    tmin = min(tols)
    fro = float(np.linalg.norm(A))
    s1 = sigma1_hint or sigma1_lower(A)
    ts = {"sigma1_est": time.time() - t0}
    # first pass: stop when the max residual column norm is ≤ target / sqrt(N) · 4 (a Frobenius
    # guess); the exact δ_F decides afterwards, and a resumed pass tightens it
    target = eta * tmin * s1
    abstol = target
    k = 0
    delta = math.inf
    ts["qp3rk"] = ts["svd_Rk"] = 0.0
    for rnd in range(max_rounds):
        # advance until δ_F ≤ target; passes after the first move k/8 columns at a time, aimed
        # with ρ = δ_F / (max residual column norm), which varies slowly
        t1 = time.time()
        first = True
        while delta > target and k < min(m, n):
            kmax = min(m, n) - k if k == 0 else max(32, k // 8)
            kk, colmax, jpiv, _ = dgeqp3rk(A, k, k, kmax, abstol)
            if k > 0 and kk > 0:  # keep the stacked R consistent: permute R12's columns by P2
                A[:k, k:] = A[:k, k:][:, jpiv]
            k += kk
            delta = _fro(A, k) if k < min(m, n) else 0.0
            rho = delta / colmax if colmax > 0 else math.sqrt(n)
            abstol = min(abstol * (0.9 if first else 1.0), 0.8 * target / max(rho, 1.0))
            first = False
        ts["qp3rk"] += time.time() - t1
        t2 = time.time()
        Rk = np.triu(A[:k, :]) if k else np.zeros((0, n))
        s = np.linalg.svd(Rk, compute_uv=False) if k else np.zeros(0)
        del Rk
        ts["svd_Rk"] += time.time() - t2
        res = _bracket(s, delta, tols, n, fro)
        if all(lo == hi for lo, hi in zip(res[1], res[2])) or k >= min(m, n):
            break
        # open bracket: σ_{p+1} sits within the Weyl window; the window closes once
        # δ < sqrt(thr² − σ_{p+1}²) ≈ thr·sqrt(2·gap)
        need = []
        for tol, lo, hi, sp1 in zip(tols, res[1], res[2], res[4]):
            if lo != hi:
                thr = tol * float(s[0])
                need.append(math.sqrt(max(thr * thr - sp1 * sp1, (thr * 1e-6) ** 2)))
        target = min(target / 2.0, 0.7 * min(need))
    ranks, lo, hi, sr, sr1, gaps, band, inb = res
    return CertifiedRank(ranks, lo, hi, float(s[0]) if len(s) else 0.0, sr, sr1, gaps, k, delta,
                         band, inb, ts)


def _fro(A: np.ndarray, k: int, chunk: int = 2048) -> float:
    """‖A[k:, k:]‖_F column block by column block (no copy of the trailing block)."""
    acc = 0.0
    for j in range(k, A.shape[1], chunk):
        blk = A[k:, j:j + chunk]
        acc += float(np.einsum("ij,ij->", blk, blk))
    return math.sqrt(acc)


def _bracket(s, delta, tols, n, fro):
    s1 = float(s[0]) if len(s) else 0.0
    s1_hi = math.sqrt(s1 * s1 + delta * delta)
    out = ([], [], [], [], [], [], [], [])
    u = 2.0 ** -53
    for tol in tols:
        thr_lo, thr_hi = tol * s1, tol * s1_hi
        lo = int(np.count_nonzero(s > thr_hi))
        hi = int(np.count_nonzero(np.sqrt(s * s + delta * delta) > thr_lo))
        thr = thr_lo
        p = int(np.count_nonzero(s > thr))
        sp = float(s[p - 1]) if p > 0 else 0.0
        sp1 = float(s[p]) if p < len(s) else 0.0
        if thr > 0:
            gap = min(sp / thr - 1.0 if p > 0 else math.inf, 1.0 - sp1 / thr if p < len(s) else math.inf)
            band = math.sqrt(n) * u * fro / thr
        else:
            gap, band = math.inf, 0.0
        rank = lo if lo == hi else lo
        for lst, v in zip(out, (rank, lo, hi, sp, sp1, gap, band, bool(gap < band))):
            lst.append(v)
    return out
