"""Generate a cube pair and assemble K once (after a warm-up) for ncu captures of k1/k2.
Usage: python tools/assemble_one.py d dp kernel N"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402

d, dp, kern, n = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
dp = None if dp < 0 else dp
with hb.Context(0) as ctx:
    pair = hb.make_pair(d, dp, n, hb.UNIFORM, 7)
    X = torch.empty((d, n), dtype=torch.float64, device="cuda")
    Y = torch.empty((d, n), dtype=torch.float64, device="cuda")
    K = torch.empty((n, n), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(2):
        ctx.generate_points(pair, X.data_ptr(), Y.data_ptr())
        ctx.assemble(hb.make_kernel(kern), X.data_ptr(), n, Y.data_ptr(), n, d, K.data_ptr(), n)
    torch.cuda.synchronize()
    print("ok")
