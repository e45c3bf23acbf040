"""How many columns would a spectral stopping rule need vs the Frobenius one? Uses σ(R_k)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb
ctx = hb.Context(0)
for (d, dp, k, n) in [(4, 3, "exp_neg_r", 16000), (3, 2, "one_over_r", 16000), (2, 1, "log_r", 65536),
                      (4, 2, "one_over_r", 16000), (4, 1, "exp_neg_r", 16000), (4, 0, "one_over_r", 16000)]:
    r = ctx.rank(hb.make_kernel(k), hb.make_pair(d, dp, n, hb.UNIFORM, hb.problem_seed(0, d, dp, n)), [1e-12])[0]
    s = np.array(ctx.last_sigma())
    thr = 1e-12 * s[0]
    out = [f"d={d} dp={dp} {k} N={n}: p={r.rank} k={r.k_factored} k/p={r.k_factored/r.rank:.2f} resid/thr={r.resid/thr:.3f}"]
    for eta in (0.2, 0.05, 0.025, 0.01):
        kk = int(np.argmax(s <= eta * thr)) if np.any(s <= eta * thr) else len(s)
        out.append(f"spectral eta={eta}: k'={kk} ({kk/r.rank:.2f}p)")
    print("; ".join(out), flush=True)
