"""Time device ACA (hb_aca_compress) against the CPU oracle restatement on cube pairs.
Usage: python tools/aca_bench.py"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402
from oracle import oracle as O  # noqa: E402

CASES = [(2, 1, "log_r", 4000, 1e-12), (3, 2, "one_over_r", 8000, 1e-8), (2, 1, "log_r", 16000, 1e-12),
         (3, 2, "one_over_r", 16000, 1e-10), (4, 3, "exp_neg_r", 8000, 1e-8)]
with hb.Context(0) as ctx:
    for d, dp, k, n, eps in CASES:
        x, y = O.pair_points(d, dp, n, 0, 3)
        X, Y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        torch.cuda.synchronize()
        K = hb.make_kernel(k)
        f = ctx.aca_compress(K, X.data_ptr(), n, Y.data_ptr(), n, d, [(0, n, 0, n)], eps, n)[0]
        f.close()
        t = time.perf_counter()
        f = ctx.aca_compress(K, X.data_ptr(), n, Y.data_ptr(), n, d, [(0, n, 0, n)], eps, n)[0]
        tg = time.perf_counter() - t
        r = f.rank
        line = f"d={d} d'={dp} {k} N={n} eps={eps:g}: rank {r} gpu {tg * 1e3:.1f} ms"
        if n <= 8000:
            t = time.perf_counter()
            o = O.aca_compress(O.KERNEL_IDS[k], x, y, eps, n)
            tc = time.perf_counter() - t
            sig, tau, _, _ = f.arrays()
            line += (f" | cpu oracle {tc * 1e3:.0f} ms (1 core) rank {o.rank} "
                     f"pivots_equal={np.array_equal(sig, o.sigma) and np.array_equal(tau, o.tau)}")
        print(line, flush=True)
        f.close()
    # batched: 512 blocks of 256 x 256 (HODLR-leaf-like) in one call
    x, y = O.pair_points(3, 2, 256 * 512, 0, 9)
    X, Y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    torch.cuda.synchronize()
    blocks = [(256 * i, 256, 256 * i, 256) for i in range(512)]
    K = hb.make_kernel("one_over_r")
    fs = ctx.aca_compress(K, X.data_ptr(), 256 * 512, Y.data_ptr(), 256 * 512, 3, blocks, 1e-8, 256)
    t = time.perf_counter()
    fs = ctx.aca_compress(K, X.data_ptr(), 256 * 512, Y.data_ptr(), 256 * 512, 3, blocks, 1e-8, 256)
    tg = time.perf_counter() - t
    print(f"batched 512 blocks 256x256 1/r eps 1e-8: mean rank {np.mean([f.rank for f in fs]):.1f}, "
          f"gpu {tg * 1e3:.1f} ms", flush=True)
