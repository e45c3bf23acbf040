"""Ad-hoc GPU bring-up checks (prints, does not assert). Usage: python tools/gpu_check.py [sections]"""
import sys
import time
import traceback

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402
from oracle import oracle as O  # noqa: E402

sections = sys.argv[1:] or ["gemm", "assemble", "rankmat", "paper", "random", "big"]
ctx = hb.Context(0)
L = hb.load()


def p(*a):
    print(*a, flush=True)


def sec(name):
    def deco(f):
        if name in sections:
            p(f"===== {name}")
            t0 = time.time()
            try:
                f()
            except Exception:
                traceback.print_exc()
            p(f"----- {name} {time.time() - t0:.1f}s")
        return f
    return deco


@sec("gemm")
def _():
    import ctypes
    L.hb_debug_dgemm.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int64,
                                 ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p,
                                 ctypes.c_int64]
    L.hb_debug_dgemm_async.argtypes = L.hb_debug_dgemm.argtypes + [ctypes.c_int32]
    g = torch.Generator(device="cuda").manual_seed(0)
    for (ta, M, N, K) in [(0, 128, 1000, 777), (1, 120, 3000, 5000), (0, 5000, 3000, 120),
                          (1, 64, 64, 20000), (0, 37, 53, 11), (1, 37, 53, 11), (0, 1000, 999, 64)]:
        A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda", generator=g)
        B = torch.randn((K, N), dtype=torch.float64, device="cuda", generator=g)
        C = torch.randn((M, N), dtype=torch.float64, device="cuda", generator=g)
        # column-major views: use transposed contiguous storage
        Af = A.t().contiguous().t() if True else A
        Acm = A.t().contiguous()  # storage of A column-major = A^T row-major
        Bcm = B.t().contiguous()
        Ccm = C.t().contiguous()
        ref = (1.5 * ((A.t() if ta else A) @ B) - 0.5 * C)
        lda = A.shape[0]
        torch.cuda.synchronize()
        st = L.hb_debug_dgemm(ctx._h, ta, M, N, K, 1.5, Acm.data_ptr(), lda, Bcm.data_ptr(), K, -0.5,
                              Ccm.data_ptr(), M)
        out = Ccm.t()
        err = (out - ref).abs().max().item() / ref.abs().max().item()
        p(f"gemm ta={ta} {M}x{N}x{K}: status={st} relerr={err:.2e}")
        del Af
    # timing
    for (ta, M, N, K) in [(0, 8192, 8192, 8192), (0, 32768, 32768, 120), (1, 120, 32768, 32768),
                          (0, 128, 65536, 65536), (0, 16384, 16384, 64)]:
        A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda")
        B = torch.randn((K, N), dtype=torch.float64, device="cuda")
        C = torch.zeros((N, M), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        s = torch.cuda.ExternalStream(ctx.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        L.hb_debug_dgemm_async(ctx._h, ta, M, N, K, 1.0, A.data_ptr(), A.shape[1] if False else (K if ta else M),
                               B.data_ptr(), K, 1.0, C.data_ptr(), M, 1)
        e0.record(s)
        reps = 3
        L.hb_debug_dgemm_async(ctx._h, ta, M, N, K, 1.0, A.data_ptr(), K if ta else M, B.data_ptr(), K, 1.0,
                               C.data_ptr(), M, reps)
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        p(f"gemm time ta={ta} {M}x{N}x{K}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.2f} TF/s")
        del A, B, C


@sec("assemble")
def _():
    for (d, dp, kname, n, mode) in [(1, 0, "log_r", 1000, 0), (2, 1, "log_r", 777, 0),
                                    (3, 2, "one_over_r", 1000, 1), (4, 3, "exp_neg_r", 1296, 1),
                                    (2, None, "r", 1600, 2), (3, 0, "sin_r", 513, 0),
                                    (4, 1, "inv_sqrt_1_plus_r", 300, 0), (3, None, "exp_neg_r2", 200, 0),
                                    (3, 2, "helmholtz3d_re", 400, 0), (3, 2, "helmholtz3d_im", 400, 0)]:
        seed = 1234 + n
        pair = hb.make_pair(d, dp, n, mode, seed)
        X = torch.empty((d, n), dtype=torch.float64, device="cuda")
        Y = torch.empty((d, n), dtype=torch.float64, device="cuda")
        ctx.generate_points(pair, X.data_ptr(), Y.data_ptr())
        ld = n + 3
        K = torch.empty((n, ld), dtype=torch.float64, device="cuda")  # column-major storage rows=cols
        torch.cuda.synchronize()
        ctx.assemble(hb.make_kernel(kname), X.data_ptr(), n, Y.data_ptr(), n, d, K.data_ptr(), ld)
        torch.cuda.synchronize()
        Kg = K.cpu().numpy()[:, :n].T  # (n, n) with Kg[i, j]
        x, y = O.pair_points(d, dp, n, mode, seed)
        pts_ok = np.array_equal(X.cpu().numpy(), x) and np.array_equal(Y.cpu().numpy(), y)
        Ko = O.assemble(O.KERNEL_IDS[kname], x, y, nthreads=8)
        rel = np.abs(Kg - Ko) / np.maximum(np.abs(Ko), 1e-300)
        rel[(Kg == Ko)] = 0
        p(f"assemble d={d} dp={dp} {kname} n={n} mode={mode}: points bit-exact={pts_ok} "
          f"max rel={rel.max():.2e} bitexact frac={(Kg == Ko).mean():.4f}")


@sec("rankmat")
def _():
    rng = np.random.default_rng(0)
    cases = []
    u = rng.standard_normal((300, 1)); v = rng.standard_normal((1, 200))
    cases.append(("rank1", u @ v, 1))
    cases.append(("I5", np.eye(5), 5))
    q1, _ = np.linalg.qr(rng.standard_normal((500, 500)))
    q2, _ = np.linalg.qr(rng.standard_normal((400, 400)))
    s = np.logspace(0, -16, 400)
    cases.append(("graded500x400", (q1[:, :400] * s) @ q2.T, None))
    cases.append(("gauss 1000x700", rng.standard_normal((1000, 700)), None))
    for name, M, want in cases:
        A = torch.tensor(np.asfortranarray(M).T.copy(), device="cuda")  # col-major storage
        m, n = M.shape
        torch.cuda.synchronize()
        r = ctx.rank_matrix(A.data_ptr(), m, n, m, [1e-12, 1e-6])
        sv = np.linalg.svd(M, compute_uv=False)
        o = [O.epsilon_rank_from_sigma(sv, t) for t in (1e-12, 1e-6)]
        p(f"{name}: gpu ranks {[x.rank for x in r]} (lo/hi {[(x.rank_lo, x.rank_hi) for x in r]}, k={r[0].k_factored}, "
          f"resid={r[0].resid:.2e}, s1={r[0].sigma1:.6e}) oracle {[x.rank for x in o]} s1={sv[0]:.6e} want={want}")
        sg = np.array(ctx.last_sigma(50))
        p(f"   sigma head gpu {sg[:4]} cpu {sv[:4]}")


@sec("paper")
def _():
    import json
    tabs = json.load(open("tests/golden/paper_tables.json"))
    bad = 0
    tot = 0
    for tab in tabs:
        row = tab["rows"][0]
        n = row["N"]
        mode = hb.GRID_CLOSED if tab["dprime"] is None else hb.GRID_INTERIOR
        for kname, want in zip(tab["kernels"], row["ranks"]):
            if kname is None:
                continue
            pair = hb.make_pair(tab["d"], tab["dprime"], n, mode, 0)
            t0 = time.time()
            r = ctx.rank(hb.make_kernel(kname), pair, [1e-12])[0]
            tot += 1
            ok = r.rank == want
            bad += not ok
            p(f"{tab['label']} N={n} {kname}: want {want} got {r.rank} (lo {r.rank_lo} hi {r.rank_hi} k {r.k_factored}) "
              f"gap {r.gap:.2e} {time.time()-t0:.3f}s {'' if ok else 'MISMATCH'}")
    p(f"paper first-row: {tot - bad}/{tot} exact")


@sec("random")
def _():
    for (d, dp, kname, n) in [(1, 0, "log_r", 1000), (2, 1, "log_r", 1000), (2, 0, "log_r", 2000),
                              (2, None, "log_r", 2000), (3, 2, "one_over_r", 1000), (3, 0, "one_over_r", 2000),
                              (4, 3, "exp_neg_r", 2000), (4, None, "exp_neg_r", 1000)]:
        seed = O.problem_seed(0, d, dp, n)
        recs = O.rank_problem(d, dp, kname, n, [1e-12, 1e-10], seed=seed)
        pair = hb.make_pair(d, dp, n, hb.UNIFORM, seed)
        r = ctx.rank(hb.make_kernel(kname), pair, [1e-12, 1e-10])
        p(f"d={d} dp={dp} {kname} N={n}: gpu {[x.rank for x in r]} oracle {[x.rank for x in recs]} "
          f"gaps gpu {[f'{x.gap:.1e}' for x in r]} oracle {[f'{x.gap:.1e}' for x in recs]} k={r[0].k_factored} "
          f"sec={[round(s, 4) for s in r[0].sec]}")


@sec("big")
def _():
    for (d, dp, kname, n) in [(2, 1, "log_r", 16000), (3, 2, "one_over_r", 16000), (4, 3, "exp_neg_r", 8000),
                              (1, None, "log_r", 65536), (1, None, "log_r", 65536), (2, 1, "log_r", 65536),
                              (4, 3, "exp_neg_r", 16000), (4, 3, "exp_neg_r", 32000)]:
        seed = O.problem_seed(0, d, dp, n)
        pair = hb.make_pair(d, dp, n, hb.UNIFORM, seed)
        t0 = time.time()
        ctx.set_profiling(True)
        L.hb_stats_reset(ctx._h)
        r = ctx.rank(hb.make_kernel(kname), pair, [1e-12])[0]
        st = ctx.stats()
        ctx.set_profiling(False)
        p("   phases ms: " + " ".join(f"{k}={v:.1f}" for k, v in st["phase_ms"].items()) +
          f" gemm={st['gemm_ms']:.1f}ms {st['gemm_flops']/max(st['gemm_ms'],1e-9)/1e9:.1f}TF")
        p(f"d={d} dp={dp} {kname} N={n}: rank {r.rank} lo/hi {r.rank_lo}/{r.rank_hi} k={r.k_factored} gap {r.gap:.2e} "
          f"resid {r.resid:.2e} sec={[round(s, 4) for s in r.sec]} wall {time.time()-t0:.2f}s "
          f"Gent/s={n*n/r.sec[3]/1e9:.2f}")
