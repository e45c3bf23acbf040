"""One DMMA GEMM launch with chosen pointer offsets, checked against torch.
Usage: python tools/gemm_repro.py M N K offA offB offC [ldpad]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402

M, N, K, oa, ob, oc = (int(v) for v in sys.argv[1:7])
pad = int(sys.argv[7]) if len(sys.argv) > 7 else 8
ld = M + pad
ldb = K + (pad if ob else 0)
ldb += ldb & 1
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(ld * K + 8, dtype=torch.float64, device="cuda", generator=g)
B = torch.randn(ldb * N + 8, dtype=torch.float64, device="cuda", generator=g)
C = torch.randn(ld * N + 8, dtype=torch.float64, device="cuda", generator=g)
Am = A[oa:oa + ld * K].view(K, ld).t()[:M]
Bm = B[ob:ob + ldb * N].view(N, ldb).t()[:K]
Cm = C[oc:oc + ld * N].view(N, ld).t()[:M]
ref = Cm - Am @ Bm
ctx = hb.Context(0)
torch.cuda.synchronize()
ctx.dgemm(False, M, N, K, -1.0, A.data_ptr() + 8 * oa, ld, B.data_ptr() + 8 * ob, ldb, 1.0,
          C.data_ptr() + 8 * oc, ld)
torch.cuda.synchronize()
err = (Cm - ref).abs().max().item() / ref.abs().max().item()
print(f"M={M} N={N} K={K} off=({oa},{ob},{oc}) ld={ld} ldb={ldb}: rel err {err:.2e}", flush=True)
assert err < 1e-13
