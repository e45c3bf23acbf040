"""One device ACA compress (after a warm-up) for ncu captures.  Usage: python tools/aca_one.py d dp kernel N eps"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402
from oracle import oracle as O  # noqa: E402

d, dp, kern, n, eps = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), float(sys.argv[5])
x, y = O.pair_points(d, dp, n, 0, 3)
X, Y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
torch.cuda.synchronize()
with hb.Context(0) as ctx:
    K = hb.make_kernel(kern)
    for _ in range(2):
        f = ctx.aca_compress(K, X.data_ptr(), n, Y.data_ptr(), n, d, [(0, n, 0, n)], eps, n)[0]
    print("rank", f.rank)
