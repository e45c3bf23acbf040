"""k1/k2 parity on the B200: points bit-identical to the oracle, r bit-identical (kernel "r"),
every catalog kernel within 1e-13 relative of the oracle (BASELINE.json north_star), and the
reference's error behaviour (kernel.hpp:149-181) through the C ABI."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL_REL = 1e-13  # north_star: assembled entries within 1e-13 relative of the reference


def dev_points(ctx, hb, pair):
    d = pair.target.d
    X = torch.empty((d, pair.n_target), dtype=torch.float64, device="cuda")
    Y = torch.empty((d, pair.n_source), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ctx.generate_points(pair, X.data_ptr(), Y.data_ptr())
    torch.cuda.ExternalStream(ctx.stream).synchronize()
    return X, Y


def dev_assemble(ctx, hb, kernel, X, Y, ld_pad=0):
    d, T = X.shape
    N = Y.shape[1]
    ld = T + ld_pad
    K = torch.full((N, ld), float("nan"), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ctx.assemble(kernel, X.data_ptr(), T, Y.data_ptr(), N, d, K.data_ptr(), ld)
    return K.cpu().numpy()[:, :T].T  # K[i, j]


@pytest.mark.parametrize("d,dp,n,mode", [(1, 0, 1000, 0), (2, 1, 1001, 0), (3, None, 7, 0),
                                         (4, 3, 1296, 1), (2, None, 1600, 2), (3, 2, 1000, 1),
                                         (1, None, 1, 0), (5, 2, 300, 0), (8, None, 64, 0)])
def test_points_bit_exact(ctx, hb, oracle, d, dp, n, mode):
    seed = 12345 + n
    pair = hb.make_pair(d, dp, n, mode, seed)
    X, Y = dev_points(ctx, hb, pair)
    x, y = oracle.pair_points(d, dp, n, mode, seed)
    assert np.array_equal(X.cpu().numpy(), x) and np.array_equal(Y.cpu().numpy(), y)


@pytest.mark.parametrize("d,dp,n,m", [(1, 0, 1000, 1000), (2, 1, 513, 777), (3, 2, 1000, 64),
                                      (4, 3, 300, 301), (6, None, 100, 90)])
def test_distance_bit_exact(ctx, hb, oracle, d, dp, n, m):
    """kernel 'r' returns r itself: the device distance must equal the oracle's bit for bit."""
    pair = hb.make_pair(d, dp, n, 0, 99, n_source=m)
    X, Y = dev_points(ctx, hb, pair)
    Kg = dev_assemble(ctx, hb, hb.make_kernel("r"), X, Y, ld_pad=3)
    x = oracle.points(d, [0.0] * d, 1.0, n, 0, 99, 0)
    y = oracle.points(d, hb.offset(d, dp), 1.0, m, 0, 99, 1)
    Ko = oracle.assemble(oracle.KERNEL_IDS["r"], x, y)
    assert np.array_equal(Kg, Ko)


KERNELS = ["one_over_r", "log_r", "helmholtz3d_re", "helmholtz3d_im", "hankel_h12_re",
           "hankel_h12_im", "r", "sin_r", "inv_sqrt_1_plus_r", "exp_neg_r", "exp_neg_r2"]


@pytest.mark.parametrize("kname", KERNELS)
@pytest.mark.parametrize("d,dp,n,mode", [(2, 1, 700, 0), (3, 0, 1000, 1), (4, None, 256, 2)])
def test_entries_within_tolerance(ctx, hb, oracle, kname, d, dp, n, mode):
    pair = hb.make_pair(d, dp, n, mode, 7)
    X, Y = dev_points(ctx, hb, pair)
    Kg = dev_assemble(ctx, hb, hb.make_kernel(kname), X, Y)
    x, y = oracle.pair_points(d, dp, n, mode, 7)
    Ko = oracle.assemble(oracle.KERNEL_IDS[kname], x, y)
    both_zero = (Kg == 0) & (Ko == 0)
    rel = np.abs(Kg - Ko) / np.where(both_zero, 1.0, np.abs(Ko))
    assert np.all(np.isfinite(Kg))
    assert rel.max() <= TOL_REL, f"max rel {rel.max():.3e}"


@pytest.mark.parametrize("kname", ["hankel_h12_re", "hankel_h12_im"])
def test_bessel_entries(ctx, hb, oracle, kname):
    """J2 / Y2 (bessel.hpp:129-144) in double-double on the device vs the oracle's __float128 /
    long double restatement (itself bit-identical to the reference's bessel.hpp, test_oracle.py):
    series branch (r <= 19) within 2 ulp + 1e-300, asymptotic branch (r > 19) within
    8e-16 * sqrt(2 / (pi r)) absolute — the reference evaluates cos / sin of x - (2nu+1)pi/4 in
    long double, the device from sincos(x) and the exact +-sqrt(2)/2."""
    n = 1500
    x = np.zeros((1, n))
    y = np.concatenate([np.geomspace(1e-6, 19.0, 1000), np.linspace(19.0 + 1e-9, 120.0, 500)])[None, :]
    X, Y = torch.from_numpy(x).cuda(), torch.from_numpy(np.ascontiguousarray(y)).cuda()
    torch.cuda.synchronize()
    Kg = dev_assemble(ctx, hb, hb.make_kernel(kname), X[:, :1].contiguous(), Y)[0]
    Ko = oracle.assemble(oracle.KERNEL_IDS[kname], x[:, :1], y)[0]
    r = y[0]
    ser = r <= 19.0
    ulp = np.spacing(np.abs(Ko))
    assert np.all(np.abs(Kg - Ko)[ser] <= 2 * ulp[ser] + 1e-300)
    assert np.all(np.abs(Kg - Ko)[~ser] <= 8e-16 * np.sqrt(2 / (np.pi * r[~ser])))


def test_diagonal_rule(ctx, hb, oracle):
    """Coincident points use the catalog diagonal (kernel.hpp:46-61, 150-152)."""
    pair = hb.make_pair(2, 1, 16, hb.GRID_INTERIOR, 0)
    X, _ = dev_points(ctx, hb, pair)
    for kname, want in [("log_r", 0.0), ("one_over_r", 0.0), ("exp_neg_r", 1.0), ("sin_r", 0.0)]:
        K = dev_assemble(ctx, hb, hb.make_kernel(kname), X, X)
        assert np.all(np.diag(K) == want)
    K = dev_assemble(ctx, hb, hb.make_kernel("exp_neg_r", diagonal=None), X, X)  # F(0) fallback
    assert np.all(np.diag(K) == 1.0)
    K = dev_assemble(ctx, hb, hb.make_kernel("one_over_r", diagonal=7.5), X, X)
    assert np.all(np.diag(K) == 7.5)


def test_assemble_errors(ctx, hb):
    pair = hb.make_pair(2, 1, 16, hb.GRID_INTERIOR, 0)
    X, _ = dev_points(ctx, hb, pair)
    with pytest.raises(hb.HBError) as e:
        dev_assemble(ctx, hb, hb.make_kernel("one_over_r", diagonal=None), X, X)
    assert e.value.status == 4  # ESINGULAR (kernel.hpp:152-153)
    with pytest.raises(hb.HBError) as e:
        dev_assemble(ctx, hb, hb.make_kernel("custom"), X, X)
    assert e.value.status == 5
    with pytest.raises(hb.HBError) as e:  # Y2 is singular at 0 (kernel.hpp:80), no diagonal given
        dev_assemble(ctx, hb, hb.make_kernel("hankel_h12_im", diagonal=None), X, X)
    assert e.value.status == 4
    K = torch.empty(16 * 16, dtype=torch.float64, device="cuda")
    with pytest.raises(hb.HBError) as e:
        ctx.assemble(hb.make_kernel("log_r"), X.data_ptr(), 16, X.data_ptr(), 16, 2, K.data_ptr(), 8)
    assert e.value.status == 1  # ldk < T
    with pytest.raises(hb.HBError) as e:
        ctx.assemble(hb.make_kernel("log_r"), X.data_ptr(), 0, X.data_ptr(), 16, 2, K.data_ptr(), 16)
    assert e.value.status == 1  # empty point set (kernel.hpp:171)


def test_pair_validation(ctx, hb):
    bad = hb.make_pair(2, 1, 100, hb.UNIFORM, 0)
    bad.source.side = 0.0
    with pytest.raises(hb.HBError) as e:
        ctx.rank(hb.make_kernel("log_r"), bad, [1e-12])
    assert e.value.status == 1  # HyperCube side > 0 (geometry.hpp:22)
    with pytest.raises(hb.HBError) as e:
        ctx.rank(hb.make_kernel("log_r"), hb.make_pair(2, 1, 99, hb.GRID_INTERIOR, 0), [1e-12])
    assert e.value.status == 1  # grid needs N = n^d
    with pytest.raises(hb.HBError) as e:
        ctx.rank(hb.make_kernel("log_r"), hb.make_pair(2, 1, 100, hb.UNIFORM, 0), [0.0])
    assert e.value.status == 1


def test_dgemm_hook_numerics(ctx, hb):
    g = torch.Generator(device="cuda").manual_seed(0)
    for ta, M, N, K in [(0, 128, 1000, 777), (1, 120, 3000, 5000), (0, 5000, 333, 120),
                        (1, 64, 64, 20000), (0, 37, 53, 11), (1, 37, 53, 11), (0, 1, 1, 1)]:
        A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda", generator=g)
        B = torch.randn((K, N), dtype=torch.float64, device="cuda", generator=g)
        C = torch.randn((M, N), dtype=torch.float64, device="cuda", generator=g)
        ref = 1.5 * ((A.t() if ta else A) @ B) - 0.5 * C
        Acm, Bcm, Ccm = A.t().contiguous(), B.t().contiguous(), C.t().contiguous()
        torch.cuda.synchronize()
        ctx.dgemm(bool(ta), M, N, K, 1.5, Acm.data_ptr(), A.shape[0], Bcm.data_ptr(), K, -0.5,
                  Ccm.data_ptr(), M)
        err = (Ccm.t() - ref).abs().max().item() / max(ref.abs().max().item(), 1e-300)
        assert err < 1e-14 * max(1.0, K ** 0.5), (ta, M, N, K, err)


@pytest.mark.parametrize("M,N,K,offs", [(20000, 19880, 120, (1, 0, 0)), (4000, 3000, 120, (0, 1, 0)),
                                        (4000, 3000, 117, (1, 1, 1)), (3001, 2999, 128, (1, 0, 1)),
                                        (513, 777, 100, (0, 1, 1)), (256, 256, 96, (1, 1, 0)),
                                        (1000, 300, 121, (0, 0, 1))])
def test_update_gemm_pointer_offsets(ctx, hb, M, N, K, offs):
    """Operands starting 8 bytes past a 16-byte boundary (odd column offsets inside K, V and W
    buffers): the TMA-fed kernel loads from the aligned boundary and reads at +1."""
    g = torch.Generator(device="cuda").manual_seed(M + K)
    oa, ob, oc = offs
    ld, ldb = M + 8, K + 8
    A = torch.randn(ld * K + 8, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(ldb * N + 8, dtype=torch.float64, device="cuda", generator=g)
    C = torch.randn(ld * N + 8, dtype=torch.float64, device="cuda", generator=g)
    Am = A[oa:oa + ld * K].view(K, ld).t()[:M]
    Bm = B[ob:ob + ldb * N].view(N, ldb).t()[:K]
    Cm = C[oc:oc + ld * N].view(N, ld).t()[:M]
    ref = Cm - Am @ Bm
    torch.cuda.synchronize()
    ctx.dgemm(False, M, N, K, -1.0, A.data_ptr() + 8 * oa, ld, B.data_ptr() + 8 * ob, ldb, 1.0,
              C.data_ptr() + 8 * oc, ld)
    torch.cuda.synchronize()
    err = (Cm - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-14 * max(1.0, K ** 0.5), err


@pytest.mark.parametrize("M,N,K,ldpad", [(5000, 333, 120, 0), (1000, 1000, 64, 0), (777, 4097, 117, 3),
                                         (4096, 257, 8, 1), (300, 300, 1, 0), (2048, 2048, 128, 0),
                                         (16001, 1500, 97, 5), (4000, 4000, 120, 0),
                                         (3000, 3500, 64, 1), (9000, 1100, 1, 0), (5003, 4001, 30, 2)])
def test_update_gemm_numerics(ctx, hb, M, N, K, ldpad):
    """The rank-b trailing-update shape C -= A B (K <= 128) of the DMMA GEMM against torch fp64:
    odd K, ragged M / N, odd leading dimensions (8-byte path), K not a multiple of the k-tile."""
    g = torch.Generator(device="cuda").manual_seed(K)
    lda, ldb, ldc = M + ldpad, K + ldpad, M + ldpad
    A = torch.randn((K, lda), dtype=torch.float64, device="cuda", generator=g)  # column-major M x K
    B = torch.randn((N, ldb), dtype=torch.float64, device="cuda", generator=g)  # column-major K x N
    C = torch.randn((N, ldc), dtype=torch.float64, device="cuda", generator=g)  # column-major M x N
    ref = C[:, :M].t() - A[:, :M].t() @ B[:, :K].t()
    keep = C[:, M:].clone()
    torch.cuda.synchronize()
    ctx.dgemm(False, M, N, K, -1.0, A.data_ptr(), lda, B.data_ptr(), ldb, 1.0, C.data_ptr(), ldc)
    torch.cuda.synchronize()
    err = (C[:, :M].t() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-14 * max(1.0, K ** 0.5), err
    assert torch.equal(C[:, M:], keep)  # padding rows untouched


def test_dprime_validated_against_cubes(ctx, hb):
    """d_prime must equal classify_pair of the cube pair when the cubes are boxes of one grid
    (geometry.hpp:109-118); a mismatch is an invalid_argument (EINVAL), not a silent relabel."""
    for d, dp, wrong in [(2, 1, 0), (3, None, 2), (4, 0, -1), (1, 0, -2)]:
        p = hb.make_pair(d, dp, 64, hb.UNIFORM, 0)
        p.d_prime = wrong
        with pytest.raises(hb.HBError) as e:
            ctx.rank(hb.make_kernel("exp_neg_r"), p, [1e-12])
        assert e.value.status == 1
    p = hb.make_pair(2, 1, 64, hb.UNIFORM, 0)
    p.d_prime = 5  # out of range for d = 2
    with pytest.raises(hb.HBError):
        ctx.rank(hb.make_kernel("exp_neg_r"), p, [1e-12])
    # cubes off the common grid: d_prime cannot be implied and any valid label is accepted
    p = hb.make_pair(2, 1, 64, hb.UNIFORM, 0)
    p.source.lower[0] = 1.25
    assert ctx.rank(hb.make_kernel("exp_neg_r"), p, [1e-12])[0].rank > 0


@pytest.mark.parametrize("d,dp,T,N,kname", [(2, 1, 500, 700, "log_r"), (3, None, 64, 1000, "one_over_r"),
                                            (4, 3, 333, 129, "exp_neg_r"), (1, 0, 1, 1, "sin_r")])
def test_assemble_dense_host_matches_oracle(ctx, hb, oracle, d, dp, T, N, kname):
    """hb_assemble_dense_host: the reference's assemble_dense(spec, targets, sources) on host
    PointSets (kernel.hpp:168-181), same layout, entries within 1e-13 of the oracle (pinned bit
    for bit against the compiled reference in tests/test_oracle.py)."""
    x = oracle.points(d, [0.0] * d, 1.0, T, 0, 7, 0)
    y = oracle.points(d, hb.offset(d, dp), 1.0, N, 0, 7, 1)
    K = ctx.assemble_dense_host(hb.make_kernel(kname), x, y)
    Ko = oracle.assemble(oracle.KERNEL_IDS[kname], x, y)
    assert K.shape == (T, N)
    np.testing.assert_allclose(K, Ko, rtol=TOL_REL, atol=0)


def test_assemble_dense_host_errors(ctx, hb):
    x = np.zeros((2, 10))
    with pytest.raises(hb.HBError) as e:  # length_error: T*N above the entry cap (kernel.hpp:174-175)
        ctx.assemble_dense_host(hb.make_kernel("log_r"), x, x + 1.0, entry_cap=50)
    assert e.value.status == 3
    with pytest.raises(hb.HBError) as e:  # empty point set (kernel.hpp:171)
        ctx.assemble_dense_host(hb.make_kernel("log_r"), np.zeros((2, 0)), x)
    assert e.value.status == 1
    with pytest.raises(hb.HBError) as e:  # point dimensions differ (kernel.hpp:172-173)
        ctx.assemble_dense_host(hb.make_kernel("log_r"), np.zeros((3, 4)), x)
    assert e.value.status == 1
    with pytest.raises(hb.HBError) as e:  # r == 0 on 1/r without a diagonal (kernel.hpp:152-153)
        ctx.assemble_dense_host(hb.make_kernel("one_over_r", diagonal=None), x, x)
    assert e.value.status == 4
