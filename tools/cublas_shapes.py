"""cuBLAS DGEMM (torch.matmul on float64) on the rank-reveal shapes, for comparison with
tools/gemm_bench.py (our DMMA kernel).  Usage: python tools/cublas_shapes.py"""
import torch

SHAPES = [(8192, 8192, 8192), (32768, 32768, 120), (32768, 32768, 64), (32768, 32768, 240),
          (16000, 16000, 120), (16384, 16384, 32)]
for M, N, K in SHAPES:
    A = torch.randn((M, K), dtype=torch.float64, device="cuda")
    B = torch.randn((K, N), dtype=torch.float64, device="cuda")
    C = torch.randn((M, N), dtype=torch.float64, device="cuda")
    C.addmm_(A, B, alpha=-1.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        C.addmm_(A, B, alpha=-1.0)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cuBLAS C -= A B {M}x{N}x{K}: {ms:8.3f} ms {2 * M * N * K / ms / 1e9:7.2f} TF/s", flush=True)
    del A, B, C
