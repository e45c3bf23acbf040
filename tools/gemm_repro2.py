"""Pipeline-shaped GEMM repro: A (M x K) inside an lda x K buffer whose rows >= M hold junk,
C in place inside a bigger ld.  Usage: python tools/gemm_repro2.py M N K lda [junk]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2209_05819_b200 as hb  # noqa: E402

M, N, K, lda = (int(v) for v in sys.argv[1:5])
junk = float(sys.argv[5]) if len(sys.argv) > 5 else 1e3
g = torch.Generator(device="cuda").manual_seed(3)
A = torch.randn((K, lda), dtype=torch.float64, device="cuda", generator=g)
A[:, M:] = junk
B = torch.randn((N, K), dtype=torch.float64, device="cuda", generator=g)
C = torch.randn((N, lda), dtype=torch.float64, device="cuda", generator=g)
ref = C[:, :M].t() - A[:, :M].t() @ B.t()
keep = C[:, M:].clone()
ctx = hb.Context(0)
for rep in range(3):
    Cw = C.clone()
    torch.cuda.synchronize()
    f = ctx.dgemm_fro(False, M, N, K, -1.0, A.data_ptr(), lda, B.data_ptr(), K, 1.0, Cw.data_ptr(), lda, K)
    torch.cuda.synchronize()
    err = (Cw[:, :M].t() - ref).abs().max().item() / ref.abs().max().item()
    bad = ((Cw[:, :M].t() - ref).abs() > 1e-12 * ref.abs().max()).nonzero()
    fw = float((ref[K:] ** 2).sum())
    print(f"M={M} N={N} K={K} lda={lda} rep {rep}: rel err {err:.2e}, bad {bad.shape[0]} first {bad[:4].tolist()}, "
          f"fro rel {abs(f - fw) / fw:.1e}, tail kept {torch.equal(Cw[:, M:], keep)}", flush=True)
Cw = C.clone()
torch.cuda.synchronize()
ctx.dgemm(False, M, N, K, -1.0, A.data_ptr(), lda, B.data_ptr(), K, 1.0, Cw.data_ptr(), lda)
torch.cuda.synchronize()
bad = ((Cw[:, :M].t() - ref).abs() > 1e-12 * ref.abs().max()).nonzero()
if bad.shape[0]:
    rows = sorted(set(bad[:, 0].tolist()))
    cols = bad[:, 1]
    print("bad rows", rows[:20], "n rows", len(rows))
    print("bad col%64 hist", torch.bincount(cols % 64, minlength=64).tolist())
    tiles = sorted(set((cols // 64).tolist()))
    print("bad tiles", tiles[:40], len(tiles), "tile%32", sorted(set(t % 32 for t in tiles)))
if bad.shape[0]:
    Am_, Bm_ = A[:, :M].t(), B.t()
    for (r, c) in bad[:6].tolist():
        got = Cw[c, r].item(); want = ref[r, c].item(); c0 = C[c, r].item()
        parts = [(Am_[r, k0:k0 + 40] @ Bm_[k0:k0 + 40, c]).item() for k0 in (0, 40, 80)]
        print(f"r={r} c={c}: got-want {got - want:+.6e}  C0 {c0:+.6e}  chunk products {[f'{p:+.6e}' for p in parts]}")
if bad.shape[0]:
    for (r, c) in bad[:4].tolist():
        used = C[c, r].item() + (Cw[c, r].item() - ref[r, c].item())
        row = C[:N, r]
        close = ((row - used).abs() < 1e-9 * max(1.0, abs(used))).nonzero().flatten().tolist()
        colrow = C[c, :M]
        close2 = ((colrow - used).abs() < 1e-9 * max(1.0, abs(used))).nonzero().flatten().tolist()
        print(f"r={r} c={c}: C value used {used:+.6e}; matches C[r, cols] at {close[:5]}; C[rows, c] at {close2[:5]}")
