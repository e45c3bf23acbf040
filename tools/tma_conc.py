"""TMA update GEMM under concurrency: thread 1 repeats the same A2 -= V W (HB_GEMM_TMA=1) on its
own context and compares every result with the first; thread 2 runs a chosen background load on
another context.  Usage: HB_GEMM_TMA=1 python tools/tma_conc.py none|gemm|rank|aca [reps]"""
import sys
import threading

import torch

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402

mode = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
M = N = 16000
K, ld = 120, 16000
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(ld * K, dtype=torch.float64, device="cuda", generator=g)
B = torch.randn(K * N, dtype=torch.float64, device="cuda", generator=g)
C0 = torch.randn(ld * N, dtype=torch.float64, device="cuda", generator=g)
c1 = hb.Context(0)
c2 = hb.Context(0)
stop = threading.Event()


def background():
    if mode == "gemm":
        A2 = torch.randn(8000 * 8000, dtype=torch.float64, device="cuda")
        while not stop.is_set():
            c2.dgemm(False, 8000, 8000, 64, -1.0, A2.data_ptr(), 8000, A2.data_ptr(), 64, 1.0,
                     A2.data_ptr() + 8 * 8000 * 100, 8000)
    elif mode == "rank":
        k = hb.make_kernel("exp_neg_r")
        i = 0
        while not stop.is_set():
            n = [2000, 4000, 8000][i % 3]
            c2.rank(k, hb.make_pair(4, i % 4, n, hb.UNIFORM, i), [1e-12])
            i += 1
    elif mode == "tma":  # a second stream of TMA GEMMs (other shape, other buffers)
        n2 = 12000
        A2 = torch.randn(n2 * 120, dtype=torch.float64, device="cuda")
        B2 = torch.randn(120 * n2, dtype=torch.float64, device="cuda")
        C2 = torch.randn(n2 * n2, dtype=torch.float64, device="cuda")
        while not stop.is_set():
            c2.dgemm(False, n2, n2, 120, -1.0, A2.data_ptr(), n2, B2.data_ptr(), 120, 1.0,
                     C2.data_ptr(), n2)
    elif mode == "aca":
        X = torch.rand(2 * 4000, dtype=torch.float64, device="cuda")
        Y = X + 2.0
        while not stop.is_set():
            c2.aca_compress(hb.make_kernel("log_r"), X.data_ptr(), 4000, Y.data_ptr(), 4000, 2,
                            [(0, 4000, 0, 4000)], 1e-10, 300)


th = threading.Thread(target=background)
if mode != "none":
    th.start()
ref = None
bad = 0
for r in range(reps):
    C = C0.clone()
    torch.cuda.synchronize()
    c1.dgemm(False, M, N, K, -1.0, A.data_ptr(), ld, B.data_ptr(), K, 1.0, C.data_ptr(), ld)
    torch.cuda.synchronize()
    if ref is None:
        ref = C
    elif not torch.equal(C, ref):
        bad += 1
stop.set()
if mode != "none":
    th.join()
print(f"mode={mode}: {bad} of {reps - 1} repeats differ from the first", flush=True)
