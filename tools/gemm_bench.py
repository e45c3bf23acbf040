"""Time the FP64 DMMA GEMM (include/hb_debug.h hook) on the rank-reveal shapes.
Usage: python tools/gemm_bench.py [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
SHAPES = [  # (transA, M, N, K, beta): name
    ((0, 8192, 8192, 8192, 1.0), "square 8192^3"),
    ((0, 32768, 32768, 120, 1.0), "trailing update A2 -= V W (K=b=120)"),
    ((1, 120, 32768, 32768, 0.0), "W = V^T A2 (TN reduce, M=b)"),
    ((0, 128, 65536, 65536, 0.0), "sketch Y = Omega A (M=128)"),
    ((0, 16384, 16384, 32, 1.0), "band-reduction update (K=32)"),
    ((1, 64, 32768, 32768, 0.0), "W = V^T A2 (TN reduce, M=b=64)"),
    ((0, 32768, 32768, 64, 1.0), "trailing update (K=b=64)"),
    ((0, 32768, 32768, 240, 1.0), "trailing update (K=2b=240)"),
    ((1, 240, 32768, 32768, 0.0), "W = V^T A2 (TN reduce, M=2b=240)"),
    ((0, 65536, 65536, 120, 1.0), "trailing update N=65536 (K=120)"),
    ((0, 65536, 65536, 240, 1.0), "trailing update N=65536 (K=240)"),
    ((0, 49999, 49999, 117, 1.0, 1), "trailing update, odd offsets (K=117)"),
    ((0, 20000, 19880, 120, 1.0, 1), "cert-QR update (K=120, odd offsets)"),
    ((0, 50000, 50000, 117, 1.0, 2), "trailing update, A/C offset, even ld (K=117)"),
    ((0, 65536, 65536, 104, 1.0), "trailing update N=65536 (K=104)"),
    ((0, 65536, 65536, 128, 1.0), "trailing update N=65536 (K=128)"),
]
ctx = hb.Context(0)
s = torch.cuda.ExternalStream(ctx.stream)
for shape, name in SHAPES:
    ta, M, N, K, beta = shape[:5]
    off = shape[5] if len(shape) > 5 else 0  # 1: A and C start 8 bytes past a 16-byte boundary
    ld = M + 8 if off else M
    if off == 2:  # even leading dimension, odd start
        off, ld = 1, M + 8 + (M & 1)
    A = torch.randn(((ld if not ta else K) * (K if not ta else M) + 8,), dtype=torch.float64, device="cuda")
    B = torch.randn((K * N + 8,), dtype=torch.float64, device="cuda")
    C = torch.randn((ld * N + 8,), dtype=torch.float64, device="cuda")
    lda = K if ta else ld
    pa, pc = A.data_ptr() + 8 * off, C.data_ptr() + 8 * off
    torch.cuda.synchronize()
    ctx.dgemm(bool(ta), M, N, K, 1.0, pa, lda, B.data_ptr(), K, beta, pc, ld, reps=1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    ctx.dgemm(bool(ta), M, N, K, 1.0, pa, lda, B.data_ptr(), K, beta, pc, ld, reps=reps)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name:45s} {M}x{N}x{K}: {ms:8.3f} ms {2 * M * N * K / ms / 1e9:7.2f} TF/s", flush=True)
    del A, B, C
