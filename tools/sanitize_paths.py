"""One small problem through every kernel path, for compute-sanitizer (memcheck / racecheck /
synccheck).  Sizes are tiny on purpose: instrumented cooperative kernels are ~100x slower.
Usage: compute-sanitizer --tool memcheck python tools/sanitize_paths.py [sections...]
Sections: rank_small rank_cluster rank_band complex aca hodlr cheb gemm tma (default: all but tma;
`tma` needs HB_GEMM_TMA=1 to route the NN GEMM to the TMA kernel)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402

sections = sys.argv[1:] or ["rank_small", "rank_cluster", "rank_band", "complex", "aca", "hodlr",
                            "cheb", "gemm"]
ctx = hb.Context(0)


def run(name, f):
    if name not in sections:
        return
    t0 = time.time()
    out = f()
    print(f"[sanitize] {name}: {out} ({time.time() - t0:.1f}s)", flush=True)


def rank(d, dp, kern, n, tols=(1e-12,)):
    r = ctx.rank(hb.make_kernel(kern), hb.make_pair(d, dp, n, hb.UNIFORM, hb.problem_seed(0, d, dp, n)),
                 list(tols))
    return [(x.rank, x.rank_lo, x.rank_hi, x.k_factored) for x in r]


# k <= 144: single-CTA bidiagonalisation, smem sketch CPQR, cluster panel
run("rank_small", lambda: rank(2, 1, "log_r", 600))
# 144 < k <= ~600: 16-CTA cluster bidiagonalisation (DSMEM triangle)
run("rank_cluster", lambda: rank(3, 2, "one_over_r", 900))
# k > 600: two-stage (band reduction GEMMs + bulge chase), two tolerances from one factorisation
run("rank_band", lambda: rank(4, 3, "exp_neg_r", 1100, (1e-12, 1e-10)))


def complex_rank():
    pair = hb.make_pair(2, 1, 500, hb.UNIFORM, 7)
    r = ctx.rank_complex(hb.make_kernel("hankel_h12_re"), hb.make_kernel("hankel_h12_im"), pair, [1e-12])
    return [(x.rank, x.rank_lo, x.rank_hi) for x in r]


def aca():
    rng = np.random.default_rng(3)
    x = torch.tensor(rng.random((2, 700)), dtype=torch.float64, device="cuda")  # SoA d x n
    y = torch.tensor(rng.random((2, 700)) + np.array([[1.0], [0.0]]), dtype=torch.float64, device="cuda")
    blocks = [(0, 700, 0, 700), (0, 300, 100, 300), (5, 1, 0, 700)]
    fs = ctx.aca_compress(hb.make_kernel("log_r"), x.data_ptr(), 700, y.data_ptr(), 700, 2, blocks,
                          1e-10, 300)
    out = [f.rank for f in fs]
    q = torch.ones(700, dtype=torch.float64, device="cuda")
    b = torch.zeros(700, dtype=torch.float64, device="cuda")
    ctx.aca_apply(fs[0], hb.make_kernel("log_r"), x.data_ptr(), 700, y.data_ptr(), 700, 2,
                  q.data_ptr(), b.data_ptr())
    torch.cuda.synchronize()
    return out


def hodlr():
    rng = np.random.default_rng(5)
    x = rng.random((2, 1500))
    H = hb.HMatrix(ctx, hb.make_kernel("log_r"), x, hb.make_cube([0.0, 0.0]), "weakdd", 128, 1e-8)
    b = H.matvec(rng.standard_normal((1500, 2)))
    H.close()
    return float(np.abs(b).max())


def cheb():
    rng = np.random.default_rng(9)
    x = rng.random((2, 300)) + np.array([[2.0], [0.0]])
    return ctx.interpolation_decay(hb.make_kernel("log_r"), x, hb.make_cube([0.0, 0.0], 1.0), [2, 4, 6])[-1]


def gemm(shapes):
    g = torch.Generator(device="cuda").manual_seed(0)
    worst = 0.0
    for ta, M, N, K in shapes:
        A = torch.randn((M, K) if ta else (K, M), dtype=torch.float64, device="cuda", generator=g)
        B = torch.randn((N, K), dtype=torch.float64, device="cuda", generator=g)
        C = torch.randn((N, M), dtype=torch.float64, device="cuda", generator=g)  # column-major M x N
        Am = A if ta else A.t()  # math A (M x K)
        ref = (-1.0 * (Am @ B.t()) + C.t()).t().contiguous()
        lda = K if ta else M
        ctx.dgemm(bool(ta), M, N, K, -1.0, A.data_ptr(), lda, B.data_ptr(), K, 1.0, C.data_ptr(), M)
        torch.cuda.synchronize()
        worst = max(worst, float((C - ref).abs().max()))
    return worst


run("complex", complex_rank)
run("aca", aca)
run("hodlr", hodlr)
run("cheb", cheb)
run("gemm", lambda: gemm([(0, 300, 500, 120), (1, 120, 700, 900), (0, 129, 67, 33), (1, 64, 64, 4000)]))
# the TMA update kernel (HB_GEMM_TMA=1): full and ragged tiles, odd C offsets via M
run("tma", lambda: gemm([(0, 1024, 2048, 120), (0, 1000, 1000, 117), (0, 362, 4100, 128), (0, 512, 512, 96)]))
ctx.close()
print("[sanitize] done", flush=True)
