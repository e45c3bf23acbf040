"""Run the same DMMA GEMM many times from identical inputs and require bit-identical outputs (a race
in the TMA ring shows up as run-to-run differences).  Usage: python tools/gemm_determinism.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402

ctx = hb.Context(0)
bad = 0
for (M, N, K, oa, oc) in [(20000, 19880, 120, 0, 0), (32768, 32768, 120, 0, 0), (65536, 8192, 117, 1, 1),
                          (4000, 3000, 128, 0, 1), (50000, 4000, 100, 1, 0)]:
    ld = M + 8
    g = torch.Generator(device="cuda").manual_seed(M)
    A = torch.randn(ld * K + 8, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(K * N + 8, dtype=torch.float64, device="cuda", generator=g)
    C0 = torch.randn(ld * N + 8, dtype=torch.float64, device="cuda", generator=g)
    ref = None
    for rep in range(12):
        C = C0.clone()
        torch.cuda.synchronize()
        ctx.dgemm(False, M, N, K, -1.0, A.data_ptr() + 8 * oa, ld, B.data_ptr(), K, 1.0,
                  C.data_ptr() + 8 * oc, ld)
        torch.cuda.synchronize()
        if ref is None:
            ref = C
        elif not torch.equal(C, ref):
            d = (C != ref).nonzero()
            print(f"M={M} N={N} K={K}: rep {rep} differs in {d.numel()} entries, first {d[:3].tolist()}",
                  flush=True)
            bad += 1
    print(f"M={M} N={N} K={K} off=({oa},{oc}): done", flush=True)
print("BAD" if bad else "deterministic")

# with the Frobenius epilogue (the trailing update's form)
bad2 = 0
for (M, N, K, oa, oc, r0) in [(16000, 15880, 120, 0, 0, 120), (15880, 15760, 120, 0, 1, 120), (9000, 7000, 117, 1, 1, 117)]:
    ld = M + 8
    g = torch.Generator(device="cuda").manual_seed(M)
    A = torch.randn(ld * K + 8, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(K * N + 8, dtype=torch.float64, device="cuda", generator=g)
    C0 = torch.randn(ld * N + 8, dtype=torch.float64, device="cuda", generator=g)
    ref, rf = None, None
    for rep in range(12):
        C = C0.clone()
        torch.cuda.synchronize()
        f = ctx.dgemm_fro(False, M, N, K, -1.0, A.data_ptr() + 8 * oa, ld, B.data_ptr(), K, 1.0,
                          C.data_ptr() + 8 * oc, ld, r0)
        torch.cuda.synchronize()
        Cm = C[oc:oc + ld * N].view(N, ld).t()[:M]
        want = float((Cm[r0:] ** 2).sum())
        if ref is None:
            ref, rf = C, f
            print(f"fro M={M}: {f:.15e} torch {want:.15e} rel {abs(f - want) / want:.1e}", flush=True)
        elif not torch.equal(C, ref) or f != rf:
            print(f"fro M={M}: rep {rep} differs: C equal {torch.equal(C, ref)} fro {f!r} vs {rf!r}", flush=True)
            bad2 += 1
print("FRO BAD" if bad2 else "fro deterministic")
