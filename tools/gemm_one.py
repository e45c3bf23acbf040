"""One DMMA GEMM launch of a given shape (after a warm-up) for ncu captures.
Usage: python tools/gemm_one.py transA M N K beta [alpha]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402

ta, M, N, K = (int(x) for x in sys.argv[1:5])
beta = float(sys.argv[5])
alpha = float(sys.argv[6]) if len(sys.argv) > 6 else 1.0
ctx = hb.Context(0)
A = torch.randn((M * K,), dtype=torch.float64, device="cuda")
B = torch.randn((K * N,), dtype=torch.float64, device="cuda")
C = torch.randn((M * N,), dtype=torch.float64, device="cuda")
lda = K if ta else M
torch.cuda.synchronize()
for _ in range(2):
    ctx.dgemm(bool(ta), M, N, K, alpha, A.data_ptr(), lda, B.data_ptr(), K, beta, C.data_ptr(), M)
torch.cuda.synchronize()
print("ok")
