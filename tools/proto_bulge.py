"""Prototype (numpy) of the two-stage bidiagonalisation used by the certification step:
stage 1 dense -> upper band (bandwidth nb) by alternating block QR / block LQ, stage 2 band ->
upper bidiagonal by Householder bulge chasing.  Checks singular values and records the index
windows each stage-2 task touches (to derive the inter-sweep lag of the GPU kernel)."""
import sys

import numpy as np


def house(x):
    """v (v[0]=1), tau, beta with (I - tau v v^T) x = beta e1."""
    alpha = x[0]
    s = float(np.dot(x[1:], x[1:]))
    v = np.zeros_like(x)
    v[0] = 1.0
    if s == 0.0:
        return v, 0.0, alpha
    beta = -np.copysign(np.sqrt(alpha * alpha + s), alpha)
    tau = (beta - alpha) / beta
    v[1:] = x[1:] / (alpha - beta)
    return v, tau, beta


def stage1(M, nb):
    A = M.copy()
    k = A.shape[0]
    for i in range(0, k, nb):
        # block QR of column panel
        b = min(nb, k - i)
        Q, R = np.linalg.qr(A[i:, i:i + b], mode="complete")
        A[i:, i:] = Q.T @ A[i:, i:]
        if i + b < k:
            b2 = min(nb, k - i - b)
            Q2, _ = np.linalg.qr(A[i:i + b, i + b:].T, mode="complete")
            A[i:, i + b:] = A[i:, i + b:] @ Q2
    return A


def tasks_of_sweep(s, k, nb):
    """Yield (kind, vec_index, span_lo, span_hi, app_lo, app_hi) for sweep s.
    R: reflector over columns [span_lo, span_hi] built from row vec_index; applied to rows
       [app_lo, app_hi].  L: reflector over rows [span_lo, span_hi] built from column vec_index;
       applied to columns [app_lo, app_hi]."""
    out = []
    q = 0
    while True:
        # right step
        c0 = s + 1 + q * nb
        if c0 > k - 1:
            break
        c1 = min(c0 + nb - 1, k - 1)
        row = s if q == 0 else s + 1 + (q - 1) * nb
        if c1 > c0 or q == 0:
            out.append(("R", row, c0, c1, row, min(k - 1, c1 + nb - 1, row + 2 * nb - 1)))
        # left step: rows [c0, c1], annihilate column c0 below row c0
        if c1 > c0:
            out.append(("L", c0, c0, c1, c0, min(k - 1, c1 + nb)))
        else:
            break
        q += 1
    return out


def stage2(Bm, nb, record=None):
    B = Bm.copy()
    k = B.shape[0]
    for s in range(k - 1):
        for t, (kind, idx, lo, hi, alo, ahi) in enumerate(tasks_of_sweep(s, k, nb)):
            if kind == "R":
                x = B[idx, lo:hi + 1].copy()
                v, tau, beta = house(x)
                blk = B[alo:ahi + 1, lo:hi + 1]
                w = blk @ v
                blk -= tau * np.outer(w, v)
                B[idx, lo + 1:hi + 1] = 0.0
                B[idx, lo] = beta
            else:
                x = B[lo:hi + 1, idx].copy()
                v, tau, beta = house(x)
                blk = B[lo:hi + 1, alo:ahi + 1]
                w = v @ blk
                blk -= tau * np.outer(v, w)
                B[lo + 1:hi + 1, idx] = 0.0
                B[lo, idx] = beta
            if record is not None:
                record.append((s, t, kind, lo, hi, alo, ahi))
            # invariant check: nothing outside offsets [-nb, 2nb]
        off = np.abs(np.triu(B, 2 * nb + 1)).max() if k > 2 * nb + 1 else 0
        low = np.abs(np.tril(B, -nb - 1)).max() if k > nb + 1 else 0
        assert off == 0 and low == 0, (s, off, low)
    return B


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    rng = np.random.default_rng(0)
    M = rng.standard_normal((k, k)) * np.logspace(0, -10, k)[None, :]
    sv = np.linalg.svd(M, compute_uv=False)
    Bd = stage1(M, nb)
    band_ok = np.abs(np.tril(Bd, -1)).max() < 1e-12 * sv[0] and np.abs(np.triu(Bd, nb + 1)).max() < 1e-12 * sv[0]
    Bd = np.triu(np.tril(Bd, nb))
    rec = []
    Bb = stage2(Bd, nb, rec)
    bid_ok = np.abs(Bb - np.diag(np.diag(Bb)) - np.diag(np.diag(Bb, 1), 1)).max()
    s2 = np.linalg.svd(np.diag(np.diag(Bb)) + np.diag(np.diag(Bb, 1), 1), compute_uv=False)
    print(f"k={k} nb={nb} band_ok={band_ok} offbidiag={bid_ok:.2e} "
          f"max rel sv err={np.max(np.abs(s2 - sv) / sv):.2e} (sv range {sv[-1]/sv[0]:.1e})")
    # lag analysis: task (s, t) vs tasks of sweep s-1 touching the same entries
    win = {}
    for (s, t, kind, lo, hi, alo, ahi) in rec:
        rows = (alo, ahi) if kind == "R" else (lo, hi)
        cols = (lo, hi) if kind == "R" else (alo, ahi)
        win[(s, t)] = (rows, cols)
    need = 0
    for (s, t), (r, c) in win.items():
        if s == 0:
            continue
        # last task of sweep s-1 whose window overlaps (s, t)
        last = -1
        tt = 0
        while (s - 1, tt) in win:
            r2, c2 = win[(s - 1, tt)]
            if r2[0] <= r[1] and r[0] <= r2[1] and c2[0] <= c[1] and c[0] <= c2[1]:
                last = tt
            tt += 1
        need = max(need, last - t)
    print(f"sweep s task t must wait for sweep s-1 task t+{need} (max over tasks)")


if __name__ == "__main__":
    main()
