// Host driver of k3: sketch-pivoted blocked QR + certification (one problem, one stream).
//
// Replaces SPEC `epsilon_rank` — the count of σ_k > tol·σ₁ of a dense block —
// with a factorisation whose cost scales with the ε-rank p instead of N³:
//   1. Y = Ω A (ℓ = 128 Gaussian rows).
//   2. per block of b <= 120 columns: sketch CPQR picks pivots -> swap -> Householder panel ->
//      T -> A2 ← (I − V Tᵀ Vᵀ) A2 with the exact ||A22||_F² in the GEMM epilogue -> Y downdate.
//   3. stop when δ = ||A22||_F <= η·tol·σ̂₁ (σ̂₁: power-iteration lower bound on σ₁).
//   4. certify: σ(R_k) from QR(R_kᵀ) -> bidiagonal -> bisection; then
//        rank_lo = #σ(R_k) > thr <= true rank <= rank_hi = #σ(R_k) > sqrt(thr² − δ²)
//      (σ_i(R_k) <= σ_i(A) <= sqrt(σ_i(R_k)² + δ²) by Weyl, since AᵀA = R_kᵀR_k + EᵀE, ||E|| = δ).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "context.h"

namespace hb {

namespace {

template <typename P>
void coop(void (*kern)(P), int grid, size_t smem, cudaStream_t st, P prm, int threads = 256) {
  void* args[] = {&prm};
  ensure_dyn_smem((const void*)kern, smem);
  {
    TraceSync ts(true);
    HB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(threads), args, smem, st));
  }
  launch_counter().fetch_add(1);
  if (sync_debug_enabled()) debug_sync_after_launch("coop", grid);
}

int clampi(int64_t v, int lo, int hi) { return (int)std::max<int64_t>(lo, std::min<int64_t>(hi, v)); }

void sync_to_host(hb_context* c, const void* dsrc, void* hdst, size_t bytes) {
  HB_CUDA(cudaMemcpyAsync(c->pinned, dsrc, bytes, cudaMemcpyDeviceToHost, c->stream));
  TraceSync ts;
  HB_CUDA(cudaStreamSynchronize(c->stream));
  std::memcpy(hdst, c->pinned, bytes);
}

GridBarrier barrier(hb_context* c) { return GridBarrier{c->bar, c->bar + 32}; }  // separate 128 B lines

struct Gemm {
  hb_context* c;
  void operator()(const GemmArgs& g) {
    double* sk = ws<double>(c, B_SPLITK, kSplitKElems);
    size_t e0 = 0;
    if (c->profiling) e0 = prof_event(c);
    launch_dgemm(g, sk, kSplitKElems, c->num_sms, c->stream);
    if (c->profiling)
      c->marks.push_back({PH_GEMM, e0, prof_event(c), 2.0 * (double)g.M * (double)g.N * (double)g.K});
  }
  static constexpr int64_t kSplitKElems = 24ll << 20;  // 192 MB of split-K partials
};

// Householder panel + compact-WY T.  Panel mp x b at P (ld); V (ld ldv) and T (ld b) out.
void apply_block_reflector(hb_context* c, const double* V, int64_t ldv, const double* T, int b,
                           double* A2, int64_t ld, int64_t mp, int64_t n2, double* fro_dev);

// T of the compact-WY form for the b explicit reflectors in V (S = VᵀV by DMMA GEMM).
void build_T(hb_context* c, const double* V, int64_t ldv, int64_t mp, int b, const double* tau,
             double* T, int bufid) {
  double* S = ws<double>(c, bufid, kBlockMax * kBlockMax);
  GemmArgs g{};
  g.M = b; g.N = b; g.K = mp; g.alpha = 1.0; g.A = V; g.lda = ldv; g.transA = true;
  g.B = V; g.ldb = ldv; g.beta = 0.0; g.C = S; g.ldc = b;
  Gemm{c}(g);
  const size_t tsm = ((size_t)b * (b + 1) + (size_t)b * (b - 1) / 2) * sizeof(double);
  ensure_dyn_smem((const void*)build_T_kernel, tsm);
  build_T_kernel<<<1, 256, tsm, c->stream>>>(S, b, tau, b, T, b);
  HB_LAUNCH_CHECK();
}

// Lower bound on σ₁ of the rows x n matrix X (ld): Gram G = X Xᵀ by one DMMA GEMM on the
// transposed copy, then a one-CTA power iteration on G (rows <= 128).  upper_trap: X holds the
// first rows of R (entries below the diagonal of the leading block are Householder vectors and
// count as zero).  Replaces a grid-wide power iteration whose per-column dot products were
// latency-serialised (~200 µs per call).
double sigma1_lower_bound(hb_context* c, const double* X, int64_t ld, int rows, int64_t n,
                          bool upper_trap, double* dev_out) {
  cudaStream_t st = c->stream;
  double* Xt = ws<double>(c, B_PX, (size_t)n * rows);
  dim3 tb(32, 8), tg((unsigned)ceil_div(n, 32), (unsigned)ceil_div(rows, 32));
  if (upper_trap) transpose_upper_kernel<<<tg, tb, 0, st>>>(X, ld, rows, n, Xt, n);
  else transpose_kernel<<<tg, tb, 0, st>>>(X, ld, rows, n, Xt, n);
  HB_LAUNCH_CHECK();
  double* G = ws<double>(c, B_PY, (size_t)kSketchRows * kSketchRows);
  GemmArgs g{};
  g.M = rows; g.N = rows; g.K = n; g.alpha = 1.0; g.A = Xt; g.lda = n; g.transA = true;
  g.B = Xt; g.ldb = n; g.beta = 0.0; g.C = G; g.ldc = rows;
  Gemm{c}(g);
  const size_t smem = (size_t)rows * rows * sizeof(double);
  ensure_dyn_smem((const void*)gram_sigma1_kernel, smem);
  // 16 iterations: σ̂₁ only sets the stopping target η·tol·σ̂₁ (a Rayleigh quotient is a lower
  // bound at any iteration; the certification measures σ₁ itself)
  gram_sigma1_kernel<<<1, 256, smem, st>>>(G, rows, 16, dev_out);
  HB_LAUNCH_CHECK();
  return 0.0;
}

// Householder QR of the mp x b panel at P (ld): R and V in place, explicit V (ld ldv), τ, and T
// (ld b) of Q = I − V T Vᵀ.  The shared-memory-resident kernel handles up to ~200 KB of panel
// rows per CTA; wider panels are factored as column sub-panels joined by a block-reflector
// GEMM update (left-looking within the panel).
void panel_and_T(hb_context* c, double* P, int64_t ld, int64_t mp, int b, double* V, int64_t ldv,
                 double* tau, double* T) {
  cudaStream_t st = c->stream;
  double* slots = ws<double>(c, B_SLOTS, (size_t)c->num_sms * (kBlockMax + 1) * 2 + 64);
  double* scal2 = ws<double>(c, B_PSCAL, 2 * kBlockMax + 8);
  // as few CTAs as shared memory allows (~150 KB of panel per CTA): fewer partials to reduce and
  // cheaper grid barriers per column
  auto panel_ctas = [&](int64_t rows, int cols) {
    return clampi(ceil_div(rows * cols * 8, 150 * 1024), 1, c->coop_sms);
  };
  const int G = panel_ctas(mp, b);
  const int64_t chunk = ceil_div(mp, G);
  // whole panel in one cluster's distributed shared memory: DSMEM exchange + hardware cluster
  // barrier per column instead of L2 partials + a grid barrier (HB_PANEL_CLUSTER=0 disables)
  static const bool cluster_on = [] {
    const char* e = getenv("HB_PANEL_CLUSTER");
    return !(e && atoi(e) == 0);
  }();
  if (cluster_on && b > 0) {
    const int cmax = panel_cluster_max();
    int Gc = (int)std::max<int64_t>(2, ceil_div(mp * b * 8, 150 * 1024));
    if (cmax > 0 && Gc <= cmax) {
      while (Gc < cmax && panel_cluster_smem(ceil_div(mp, Gc), b, Gc) > kPanelClusterSmem) ++Gc;
      if (Gc > 8 && cmax == 16) Gc = 16;  // cluster sizes 2..8 portable, 16 opt-in
      const int64_t chc = ceil_div(mp, Gc);
      if (panel_cluster_smem(chc, b, Gc) <= kPanelClusterSmem) {
        PanelParams pp{};
        pp.P = P; pp.ld = ld; pp.mp = mp; pp.b = b; pp.chunk = chc;
        pp.tau = tau; pp.V = V; pp.ldv = ldv;
        launch_panel_cluster(pp, Gc, st);
        build_T(c, V, ldv, mp, b, tau, T, B_S);
        return;
      }
    }
  }
  const int64_t budget = (200 * 1024) / 8;  // doubles of shared memory per CTA
  int bsub = (int)std::min<int64_t>(b, budget / (chunk + 3));
  if (bsub >= 8 && bsub < b) bsub &= ~7;
  if (bsub < 8 && bsub < b) {
    // very tall panel: global-memory fallback kernel
    PanelParams pp{};
    pp.P = P; pp.ld = ld; pp.mp = mp; pp.b = b;
    const int Gf = clampi(ceil_div(mp, 256), 1, c->coop_sms);
    pp.chunk = ceil_div(mp, Gf);
    pp.tau = tau; pp.V = V; pp.ldv = ldv;
    pp.nslot = slots; pp.wslot = slots + c->num_sms;
    pp.bar = barrier(c);
    const size_t smem = (size_t)(pp.chunk + b) * sizeof(double);
    HB_REQUIRE(smem <= 200 * 1024, HB_ECAP, "panel: too many rows per CTA");
    coop(panel_qr_kernel, Gf, smem, st, pp);
    build_T(c, V, ldv, mp, b, tau, T, B_S);
    return;
  }
  double* Tsub = ws<double>(c, B_TSUB, kBlockMax * kBlockMax);
  for (int c0 = 0; c0 < b; c0 += bsub) {
    const int bs = std::min(bsub, b - c0);
    const int64_t mps = mp - c0;
    if (c0 > 0) HB_CUDA(cudaMemset2DAsync(V + c0 * ldv, ldv * 8, 0, c0 * 8, bs, st));
    if (mps <= 0) {  // wide LQ panel ran out of rows: no more reflectors
      HB_CUDA(cudaMemsetAsync(tau + c0, 0, (b - c0) * sizeof(double), st));
      HB_CUDA(cudaMemset2DAsync(V + c0 * ldv, ldv * 8, 0, mp * 8, b - c0, st));
      break;
    }
    PanelParams pp{};
    pp.P = P + c0 + c0 * ld; pp.ld = ld; pp.mp = mps; pp.b = bs;
    const int Gs = panel_ctas(mps, bs);
    pp.chunk = ceil_div(mps, Gs);
    pp.tau = tau + c0; pp.V = V + c0 + c0 * ldv; pp.ldv = ldv;
    pp.nslot = nullptr; pp.wslot = slots; pp.scal = scal2;  // [2][Gs][bs] partials, [2][bs] rows
    pp.bar = barrier(c);
    const size_t smem = ((size_t)bs * (pp.chunk + 1) + 2 * bs) * sizeof(double);
    coop(panel_qr_smem_kernel, Gs, smem, st, pp, kPanelThreads);
    if (c0 + bs < b) {
      build_T(c, V + c0 + c0 * ldv, ldv, mps, bs, tau + c0, Tsub, B_S);
      apply_block_reflector(c, V + c0 + c0 * ldv, ldv, Tsub, bs, P + c0 + (c0 + bs) * ld, ld, mps,
                            b - c0 - bs, nullptr);
    }
  }
  build_T(c, V, ldv, mp, b, tau, T, B_S);
}

// A2 (mp x n2, ld) ← (I − V Tᵀ Vᵀ) A2; if fro != nullptr the exact sum of squares of rows >= b of
// the updated A2 is accumulated into *fro_dev (device scalar).
void apply_block_reflector(hb_context* c, const double* V, int64_t ldv, const double* T, int b,
                           double* A2, int64_t ld, int64_t mp, int64_t n2, double* fro_dev) {
  if (n2 <= 0) return;
  // W, W2 with an even leading dimension (multiple of 8): 16-byte column strides keep the update
  // GEMM on the TMA-fed kernel for any block width b
  const int64_t ldw = round_up(b, 8);
  double* W = ws<double>(c, B_W, (size_t)ldw * n2);
  double* W2 = ws<double>(c, B_W2, (size_t)ldw * n2);
  Gemm gemm{c};
  GemmArgs g{};
  g.M = b; g.N = n2; g.K = mp; g.alpha = 1.0; g.A = V; g.lda = ldv; g.transA = true;
  g.B = A2; g.ldb = ld; g.beta = 0.0; g.C = W; g.ldc = ldw;
  gemm(g);
  GemmArgs g2{};
  g2.M = b; g2.N = n2; g2.K = b; g2.alpha = 1.0; g2.A = T; g2.lda = b; g2.transA = true;
  g2.B = W; g2.ldb = ldw; g2.beta = 0.0; g2.C = W2; g2.ldc = ldw;
  gemm(g2);
  GemmArgs g3{};
  g3.M = mp; g3.N = n2; g3.K = b; g3.alpha = -1.0; g3.A = V; g3.lda = ldv; g3.transA = false;
  g3.B = W2; g3.ldb = ldw; g3.beta = 1.0; g3.C = A2; g3.ldc = ld;
  double* parts = nullptr;
  int64_t cnt = 0;
  if (fro_dev) {
    cnt = gemm_fro_count(mp, n2, b, c->num_sms);
    parts = ws<double>(c, B_FRO, (size_t)cnt);
    g3.fro_partials = parts;
    g3.fro_row0 = b;
  }
  gemm(g3);
  if (fro_dev) {
    sum_kernel<<<1, 1024, 0, c->stream>>>(parts, cnt, fro_dev);
    HB_LAUNCH_CHECK();
  }
}

// σ_max of the first `rows` rows (rows <= kBlockMax) of a column-major matrix with ld, n
// columns, by the grid-cooperative power iteration (lower bound, converges from below).
double sigma_max_rows(hb_context* c, const double* R, int64_t ld, int rows, int64_t n, int iters,
                      double* yout = nullptr) {
  double* out = ws<double>(c, B_PN, 16);
  PowerParams pw{};
  pw.R = R; pw.ld = ld; pw.b = rows; pw.n = n; pw.iters = iters; pw.mask = 0; pw.yout = yout;
  pw.slots = ws<double>(c, B_SIG1, (size_t)2 * c->num_sms * (kBlockMax + 1));
  pw.out = out + 8; pw.bar = barrier(c);
  coop(power_sigma1_kernel, clampi(ceil_div(n, 256), 1, c->coop_sms), 0, c->stream, pw);
  double h = 0.0;
  sync_to_host(c, out + 8, &h, sizeof(double));
  return h;
}

// Block power method on the residual A22 (m2 x n2): r = 8 independent Gaussian start vectors,
// q = 10 iterations of x <- A22ᵀ A22 x, each column normalised separately (no re-orthogonali-
// sation, so each is an independent power iteration).  Returns the largest ‖A22 x‖ seen, a
// lower bound on ‖A22‖₂.  Kuczyński–Woźniakowski: for one uniformly random start,
// P[λ_est < (1−ε)λ_max] <= 0.824·sqrt(n)·(1−ε)^(q−1/2); with ε = 3/4 (σ_est < σ_max/2),
// q = 10, n <= 65536 this is < 4.3e-4 per vector, < 1e-27 for all 8 — so 2·σ_est bounds ‖A22‖₂
// except with that probability.
double residual_sigma_max(hb_context* c, const double* A22, int64_t lda, int64_t m2, int64_t n2) {
  constexpr int r = 8, q = 10;
  cudaStream_t st = c->stream;
  double* X = ws<double>(c, B_PX, (size_t)n2 * r);
  double* Yv = ws<double>(c, B_PY, (size_t)m2 * r);
  double* nb = ws<double>(c, B_PN, 16);
  launch_gaussian(X, n2, r, n2, 0x5DEECE66Dull ^ (uint64_t)n2, st);
  HB_CUDA(cudaMemsetAsync(nb + r, 0, r * sizeof(double), st));
  colnorm_normalize_kernel<<<r, 1024, 0, st>>>(X, n2, n2, nb, nullptr);
  HB_LAUNCH_CHECK();
  Gemm gemm{c};
  for (int it = 0; it < q; ++it) {
    GemmArgs g{};
    g.M = m2; g.N = r; g.K = n2; g.alpha = 1.0; g.A = A22; g.lda = lda; g.transA = false;
    g.B = X; g.ldb = n2; g.beta = 0.0; g.C = Yv; g.ldc = m2;
    gemm(g);
    colnorm_normalize_kernel<<<r, 1024, 0, st>>>(Yv, m2, m2, nb, nb + r);  // ‖A22 x‖
    HB_LAUNCH_CHECK();
    GemmArgs g2{};
    g2.M = n2; g2.N = r; g2.K = m2; g2.alpha = 1.0; g2.A = A22; g2.lda = lda; g2.transA = true;
    g2.B = Yv; g2.ldb = m2; g2.beta = 0.0; g2.C = X; g2.ldc = n2;
    gemm(g2);
    colnorm_normalize_kernel<<<r, 1024, 0, st>>>(X, n2, n2, nb, nb + r);   // ‖A22ᵀ y‖
    HB_LAUNCH_CHECK();
  }
  max_kernel<<<1, 32, 0, st>>>(nb + r, r, nb);
  HB_LAUNCH_CHECK();
  double h = 0.0;
  sync_to_host(c, nb, &h, sizeof(double));
  return h;
}

// Cheap screen for the spectral stopping test: the dominant right singular direction z of the
// sketch Y2 = G·A22 (power iteration on its first rows) approximates that of A22; ‖A22 ẑ‖ is a
// lower bound on ‖A22‖₂ (one pass over A22).
double residual_sigma_screen(hb_context* c, const double* Y2, int64_t ldy, int rows, const double* A22,
                             int64_t lda, int64_t m2, int64_t n2) {
  cudaStream_t st = c->stream;
  double* z = ws<double>(c, B_PX, (size_t)n2 * 8);
  double* yv = ws<double>(c, B_PY, (size_t)m2 * 8);
  double* nb = ws<double>(c, B_PN, 16);
  sigma_max_rows(c, Y2, ldy, rows, n2, 12, z);
  colnorm_normalize_kernel<<<1, 1024, 0, st>>>(z, n2, n2, nb, nullptr);
  HB_LAUNCH_CHECK();
  GemmArgs g{};
  g.M = m2; g.N = 1; g.K = n2; g.alpha = 1.0; g.A = A22; g.lda = lda; g.transA = false;
  g.B = z; g.ldb = n2; g.beta = 0.0; g.C = yv; g.ldc = m2;
  Gemm{c}(g);
  colnorm_normalize_kernel<<<1, 1024, 0, st>>>(yv, m2, m2, nb + 1, nullptr);
  HB_LAUNCH_CHECK();
  double h[2];
  sync_to_host(c, nb, h, sizeof(h));
  return h[1];
}

void sketch(hb_context* c, const double* A, int64_t lda, int64_t m, int64_t n, double* Y,
            uint64_t seed) {
  double* Om = ws<double>(c, B_OMEGA, (size_t)kSketchRows * std::max<int64_t>(m, 1));
  launch_gaussian(Om, kSketchRows, m, kSketchRows, seed, c->stream);
  GemmArgs g{};
  g.M = kSketchRows; g.N = n; g.K = m; g.alpha = 1.0; g.A = Om; g.lda = kSketchRows;
  g.transA = false; g.B = A; g.ldb = lda; g.beta = 0.0; g.C = Y; g.ldc = kSketchRows;
  Gemm{c}(g);
}

// Two-stage Golub–Kahan bidiagonalisation of the k x k upper triangle Mk (destroyed):
// stage 1 dense -> upper band (bandwidth kBand) with DMMA GEMM updates, stage 2 bulge chasing.
constexpr int kBand = 64;  // band width of stage 1 (64: full DMMA tiles, half the panel steps of 32)

void two_stage_bidiag(hb_context* c, double* Mk, int64_t ldm, int64_t k, double* d, double* e,
                      double* V, int64_t ldv, double* tau, double* T) {
  cudaStream_t st = c->stream;
  if (k <= kSmallBidiag) {  // one CTA, whole triangle in shared memory
    const size_t smem = ((size_t)k * (k + 1) + 3 * (size_t)k) * sizeof(double);
    ensure_dyn_smem((const void*)bidiag_small_kernel, smem);
    bidiag_small_kernel<<<1, kSmallBidiagThreads, smem, st>>>(Mk, ldm, (int)k, d, e);
    HB_LAUNCH_CHECK();
    return;
  }
  if (const int G = bidiag_cluster_size((int)k)) {  // one cluster, triangle in DSMEM
    launch_bidiag_cluster(Mk, ldm, (int)k, d, e, G, st);
    return;
  }
  const int64_t ldp = round_up(k, 8);
  double* P2 = ws<double>(c, B_ST1_P, (size_t)ldp * kBand);
  double* X = ws<double>(c, B_ST1_X, (size_t)ldp * kBand);
  double* X2 = ws<double>(c, B_ST1_X2, (size_t)ldp * kBand);
  double* Vt = ws<double>(c, B_ST1_VT, (size_t)kBand * ldp);
  Gemm gemm{c};
  for (int64_t i = 0; i < k; i += kBand) {
    const int b = (int)std::min<int64_t>(kBand, k - i);
    panel_and_T(c, Mk + i + i * ldm, ldm, k - i, b, V, ldv, tau, T);
    if (i + b >= k) break;
    const int64_t nc = k - i - b;
    apply_block_reflector(c, V, ldv, T, b, Mk + i + (i + b) * ldm, ldm, k - i, nc, nullptr);
    // block LQ of the row panel Mk[i:i+b, i+b:k] = QR of its transpose
    dim3 tb(32, 8);
    transpose_kernel<<<dim3((unsigned)ceil_div(nc, 32), (unsigned)ceil_div(b, 32)), tb, 0, st>>>(
        Mk + i + (i + b) * ldm, ldm, b, nc, P2, ldp);
    HB_LAUNCH_CHECK();
    panel_and_T(c, P2, ldp, nc, b, V, ldv, tau, T);
    const int nl = (int)std::min<int64_t>(b, nc);
    write_lower_from_R<<<nl, kBand, 0, st>>>(P2, ldp, b, nl, Mk + i + (i + b) * ldm, ldm);
    HB_LAUNCH_CHECK();
    // trailing rows from the right: M2 <- M2 (I - V T V^T), M2 = Mk[i+b:k, i+b:k]
    double* M2 = Mk + (i + b) + (i + b) * ldm;
    GemmArgs g1{};
    g1.M = nc; g1.N = b; g1.K = nc; g1.alpha = 1.0; g1.A = M2; g1.lda = ldm; g1.B = V; g1.ldb = ldv;
    g1.beta = 0.0; g1.C = X; g1.ldc = ldp;
    gemm(g1);
    GemmArgs g2{};
    g2.M = nc; g2.N = b; g2.K = b; g2.alpha = 1.0; g2.A = X; g2.lda = ldp; g2.B = T; g2.ldb = b;
    g2.beta = 0.0; g2.C = X2; g2.ldc = ldp;
    gemm(g2);
    transpose_kernel<<<dim3((unsigned)ceil_div(b, 32), (unsigned)ceil_div(nc, 32)), tb, 0, st>>>(
        V, ldv, nc, b, Vt, b);
    HB_LAUNCH_CHECK();
    GemmArgs g3{};
    g3.M = nc; g3.N = nc; g3.K = b; g3.alpha = -1.0; g3.A = X2; g3.lda = ldp; g3.B = Vt; g3.ldb = b;
    g3.beta = 1.0; g3.C = M2; g3.ldc = ldm;
    gemm(g3);
  }
  // stage 2: band -> bidiagonal
  Phase ph_chase(c, HB_PH_CHASE);
  const int W = 3 * kBand + 1;
  double* Bd = ws<double>(c, B_CERT_B2, (size_t)k * W);
  band_extract_kernel<<<(unsigned)ceil_div(k * W, 256), 256, 0, st>>>(Mk, ldm, k, kBand, Bd);
  HB_LAUNCH_CHECK();
  if (k > 1) {
    int* prog = ws<int>(c, B_PROG, (size_t)k);
    HB_CUDA(cudaMemsetAsync(prog, 0, sizeof(int) * k, st));
    static const int per_sm = [] {
      int v = 0;
      HB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, bulge_chase_kernel, 256, 0));
      return v;
    }();
    const int G = clampi(k - 1, 1, std::max(1, std::min(per_sm, 8)) * c->coop_sms);
    int kb = kBand;
    int64_t kk = k;
    void* args[] = {&Bd, &kk, &kb, &prog};
    HB_CUDA(cudaLaunchCooperativeKernel((const void*)bulge_chase_kernel, dim3(G), dim3(256), args, 0, st));
    launch_counter().fetch_add(1);
    if (sync_debug_enabled()) debug_sync_after_launch("bulge_chase", G);
  }
  band_bidiag_out<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(Bd, k, kBand, d, e);
  HB_LAUNCH_CHECK();
}

}  // namespace

void rank_matrix_inplace(hb_context* c, double* A, int64_t m, int64_t n, int64_t lda,
                         const double* tols, int ntol, hb_rank_result* out, float* fact_ms,
                         float* cert_ms) {
  cudaStream_t st = c->stream;
  const int ell = kSketchRows;
  const int64_t kmax = std::min(m, n);
  double tol_min = tols[0];
  for (int t = 1; t < ntol; ++t) tol_min = std::min(tol_min, tols[t]);

  HB_CUDA(cudaEventRecord(c->ev[1], st));
  double* Y = ws<double>(c, B_YSK, (size_t)ell * n);
  double* Ys = ws<double>(c, B_YS, (size_t)ell * n);
  double* nrm = ws<double>(c, B_NRM, (size_t)n);
  const int64_t ldv = round_up(std::max(m, n), 8);
  double* V = ws<double>(c, B_V, (size_t)ldv * kBlockMax);
  double* T = ws<double>(c, B_T, kBlockMax * kBlockMax);
  double* Z = ws<double>(c, B_Z, (size_t)ell * kBlockMax);
  double* tau = ws<double>(c, B_TAU, kBlockMax);
  int* piv = ws<int>(c, B_PIV, kBlockMax);
  int* swaps = ws<int>(c, B_SWAPS, kBlockMax);
  double* rdiag = ws<double>(c, B_RDIAG, kBlockMax);
  double* est = ws<double>(c, B_EST, kBlockMax + 1);
  int* beff = ws<int>(c, B_BEFF, 4);
  int64_t* perm = ws<int64_t>(c, B_PERM, (size_t)n);
  double* scal = ws<double>(c, B_FROSUM, 8);  // [0] fro², [1] σ̂₁
  double* sk_slots = ws<double>(c, B_SCAL, (size_t)c->num_sms * 12 + 16);  // [2][G <= 2 SMs][3]
  double* sk_cand = ws<double>(c, B_SKCAND, (size_t)2 * c->num_sms * kSketchRows);  // [2][G][ℓ]
  iota_kernel<<<(unsigned)ceil_div(std::max<int64_t>(n, 1), 256), 256, 0, c->stream>>>(perm, n);
  HB_LAUNCH_CHECK();

  {  // ‖A‖_F² -> scal[2], for the rounding band of the certificate (read with the first block)
    double* parts = ws<double>(c, B_FRO, 592);
    sumsq_kernel<<<592, 256, 0, st>>>(A, m, n, lda, parts);
    sum_kernel<<<1, 1024, 0, st>>>(parts, 592, scal + 2);
    HB_LAUNCH_CHECK();
  }
  double fro_a2 = -1.0;
  uint64_t sketch_seed = 0x243F6A8885A308D3ull;
  if (kmax > 0) {
    Phase ph(c, HB_PH_SKETCH);
    sketch(c, A, lda, m, n, Y, sketch_seed);
  }

  int64_t j = 0;
  int b = std::min(32, c->block_max);
  double sigma1_est = 0.0, delta = 0.0, fro_at_sketch = INFINITY;
  if (kmax > 0 && c->block_max >= 64) {
    // σ̂₁ for the first block's stopping test from the sketch: ‖Ω A‖₂ ≈ sqrt(ℓ)·σ₁ (half of it,
    // for margin).  Not a bound — an overestimate can only stop a block early, which the exact
    // residual test after the update (and, at worst, a re-certification round) catches — but
    // it lets the first block run at the full width instead of 32 -> 64 -> 120 ramp-up blocks.
    Phase ph(c, HB_PH_SIGMA1);
    sigma1_lower_bound(c, Y, ell, ell, n, false, scal + 1);
    double sy = 0.0;
    sync_to_host(c, scal + 1, &sy, sizeof(double));
    if (sy > 0.0 && std::isfinite(sy)) {
      sigma1_est = 0.5 * sy / std::sqrt((double)ell);
      b = c->block_max;
    }
  }
  bool first = true;
  int zero_retries = 0;
  // Factor until ||A22||_F <= eta·tol·σ̂₁, certify, and only if some bracket stays open
  // (a σ(R_k) inside the window (sqrt(thr² − δ²), thr]) resume the factorisation with a 5x
  // smaller eta and certify again.  The bracket is rigorous for any δ; eta trades columns
  // (work) against the chance of a re-certification.
  double eta_cur = c->eta;
  double delta2 = INFINITY;  // probabilistic bound 2·σ̂(A22) when the spectral test stopped us
  int cert_kind[HB_MAX_TOLS] = {0, 0, 0, 0};
  SigmaAnswer ans[2 * HB_MAX_TOLS];
  int64_t k = 0;
  // certifications done and open-bracket predictor skips, counted apart so a skip never uses up
  // one of the re-certification attempts (up to 4 certifications, up to 3 skips)
  int certs = 0, skips = 0;
  double last_slope = 0.0;  // log-decay of |R_jj| per index near the threshold (0: unknown)
  for (;;) {
    while (j < kmax) {
      const int b_req = (int)std::min<int64_t>({(int64_t)b, kmax - j, (int64_t)kBlockMax});
      const int64_t n_tr = n - j, mp = m - j;
      SketchParams sp{};
      sp.Y = Y + j * ell; sp.Ys = Ys; sp.nrm = nrm; sp.ell = ell; sp.ldy = ell; sp.n_tr = n_tr;
      sp.b_req = b_req; sp.b_min = std::min(8, b_req);
      const double stop_res = 0.5 * eta_cur * tol_min * sigma1_est;
      sp.stop_fro2 = sigma1_est > 0.0 ? stop_res * stop_res : -1.0;
      sp.slots = sk_slots; sp.piv = piv; sp.swaps = swaps; sp.rdiag = rdiag; sp.out_est = est;
      sp.out_b = beff; sp.bar = barrier(c);
      {
        Phase ph(c, HB_PH_PIVOT);
        // shared-memory variant when every CTA's ℓ x cpc sketch block fits (~200 KB)
        const int Gm = clampi(ceil_div(n_tr, 64), 1, c->coop_sms);
        const int64_t cpcm = ceil_div(n_tr, Gm);
        const size_t smem_m = ((size_t)cpcm * ell + cpcm) * sizeof(double);
        if (ell == kSketchRows && smem_m <= 200 * 1024) {
          sp.cand = sk_cand;
          coop(sketch_cpqr_smem_kernel, Gm, smem_m, st, sp, kSketchThreads);
        } else {
          const int Gs = clampi(ceil_div(n_tr, 64), 1, 2 * c->coop_sms);
          coop(sketch_cpqr_kernel, Gs, (size_t)ceil_div(n_tr, Gs) * sizeof(double), st, sp);
        }
      }
      int bh = 0;
      sync_to_host(c, beff, &bh, sizeof(int));
      if (bh == 0) {
        // the sketch of the trailing matrix vanished: re-sketch once, else the trailing block is 0
        if (zero_retries++ < 1) {
          Phase ph(c, HB_PH_SKETCH);
          sketch_seed = splitmix64(sketch_seed);
          double* Om = ws<double>(c, B_OMEGA, (size_t)ell * std::max<int64_t>(mp, 1));
          launch_gaussian(Om, ell, mp, ell, sketch_seed, st);
          GemmArgs g{};
          g.M = ell; g.N = n_tr; g.K = mp; g.alpha = 1.0; g.A = Om; g.lda = ell;
          g.B = A + j + j * lda; g.ldb = lda; g.beta = 0.0; g.C = Y + j * ell; g.ldc = ell;
          Gemm{c}(g);
          continue;
        }
        break;
      }
      zero_retries = 0;
      {
        Phase ph(c, HB_PH_PIVOT);
        permute_kernel<<<(unsigned)ceil_div(m + ell + 1, 256), 256, 0, st>>>(A, lda, m, Y, ell, ell,
                                                                               perm, j, swaps, beff);
        HB_LAUNCH_CHECK();
      }
      double* P = A + j + j * lda;
      {
        Phase ph(c, HB_PH_PANEL);
        panel_and_T(c, P, lda, mp, bh, V, ldv, tau, T);
      }
      const int64_t n2 = n - j - bh;
      Phase ph_up(c, HB_PH_UPDATE);
      if (n2 > 0 && mp > bh) {
        apply_block_reflector(c, V, ldv, T, bh, A + j + (j + bh) * lda, lda, mp, n2, scal);
      } else {
        if (n2 > 0) apply_block_reflector(c, V, ldv, T, bh, A + j + (j + bh) * lda, lda, mp, n2, nullptr);
        HB_CUDA(cudaMemsetAsync(scal, 0, sizeof(double), st));
      }
      ph_up.close();
      if (first) {
        Phase ph(c, HB_PH_SIGMA1);
        sigma1_lower_bound(c, A, lda, bh, n, true, scal + 1);
      }
      if (n2 > 0) {
        Phase ph(c, HB_PH_DOWNDATE);
        const int nb8 = (bh + 7) / 8;
        const size_t rsm = ((size_t)32 * nb8 * (nb8 + 1) + (size_t)bh * ell) * sizeof(double);
        ensure_dyn_smem((const void*)sketch_trsm_kernel, rsm);
        sketch_trsm_kernel<<<1, ell, rsm, st>>>(Y + j * ell, ell, ell, P, lda, bh, Z, ell);
        HB_LAUNCH_CHECK();
        GemmArgs g{};
        g.M = ell; g.N = n2; g.K = bh; g.alpha = -1.0; g.A = Z; g.lda = ell;
        g.B = A + j + (j + bh) * lda; g.ldb = lda; g.beta = 1.0; g.C = Y + (j + bh) * ell; g.ldc = ell;
        Gemm{c}(g);
      }
      j += bh;
      double hs[3];
      sync_to_host(c, scal, hs, sizeof(hs));
      delta = std::sqrt(std::max(hs[0], 0.0));
      if (fro_a2 < 0.0) fro_a2 = hs[2];
      if (first) {
        sigma1_est = hs[1];
        first = false;
      }
      if (j >= kmax) break;
      const double target = eta_cur * tol_min * sigma1_est;
      if (delta <= target) {
        delta2 = INFINITY;
        break;
      }
      static const double screen_gate = [] {  // HB_SCREEN_GATE: screen once delta <= gate·target
        const char* e = getenv("HB_SCREEN_GATE");
        const double v = e ? atof(e) : 64.0;
        return v > 1.0 ? v : 64.0;
      }();
      if (c->spectral && sigma1_est > 0.0 && delta <= screen_gate * target) {
        // screen: ‖A22 ẑ‖ with ẑ the sketch's dominant right direction (a lower bound on
        // ‖A22‖₂); only when it is well below target run the certifying block power method
        Phase ph(c, HB_PH_SIGMA1);
        const double s2 = residual_sigma_screen(c, Y + j * ell, ell, std::min(ell, kBlockMax),
                                                A + j + j * lda, lda, m - j, n - j);
        static const bool dbg = getenv("HB_DEBUG_STOP") != nullptr;
        if (dbg)
          fprintf(stderr, "[stop] j=%lld dF/t=%.3g screen/t=%.3g\n", (long long)j, delta / target,
                  s2 / target);
        if (s2 <= target / 2.5) {
          const double sig = residual_sigma_max(c, A + j + j * lda, lda, m - j, n - j);
          if (dbg) fprintf(stderr, "[stop]   power/t=%.3g\n", sig / target);
          if (2.0 * sig <= target) {
            delta2 = 2.0 * sig;
            break;
          }
        }
      }
      if (!(fro_at_sketch < INFINITY)) fro_at_sketch = delta;
      // Fresh sketch once ‖A22‖ fell by this factor since the last one: the downdated sketch then
      // carries ~1e-16/resketch relative error, still far below what pivot choice needs (c1 and
      // c2 measured with 1e-8 / 1e-10 / 1e-12 / 1e-16: identical k everywhere, 3-5 % faster than
      // 1e-8 from the skipped second Ω·A pass).  HB_RESKETCH overrides.
      static const double resketch = [] {
        const char* e = getenv("HB_RESKETCH");
        const double v = e ? atof(e) : 1e-11;
        return v > 0.0 ? v : 1e-11;
      }();
      if (delta < resketch * fro_at_sketch) {
        Phase ph(c, HB_PH_SKETCH);
        // the downdated sketch has lost ~11 digits to cancellation: draw a fresh one
        sketch_seed = splitmix64(sketch_seed);
        const int64_t mr = m - j;
        double* Om = ws<double>(c, B_OMEGA, (size_t)ell * std::max<int64_t>(mr, 1));
        launch_gaussian(Om, ell, mr, ell, sketch_seed, st);
        GemmArgs g{};
        g.M = ell; g.N = n - j; g.K = mr; g.alpha = 1.0; g.A = Om; g.lda = ell;
        g.B = A + j + j * lda; g.ldb = lda; g.beta = 0.0; g.C = Y + j * ell; g.ldc = ell;
        Gemm{c}(g);
        fro_at_sketch = delta;
      }
      b = std::min(2 * b, c->block_max);
    }
    if (j >= kmax) {
      delta = 0.0;
      delta2 = INFINITY;
    }
    // Skip a certification that would likely leave the bracket open: the window
    // (sqrt(thr² − δ²), thr] has log-width ~η²/2, and where the spectrum is dense near thr
    // (slowly decaying 4-D spectra: ~470 σ per unit of log σ) it holds ~0.6 σ on average at
    // η = 0.05.  The local density comes from the R diagonal (|R_jj| tracks σ_j's decay for a
    // pivoted QR); when more than 0.1 σ are expected, η drops to the value that expects 0.1
    // (>= η/5) before the first certification.  A wrong guess costs time only — the
    // certification below stays rigorous.
    if (j < kmax && skips < 3 && certs < 3 && delta2 == INFINITY && sigma1_est > 0.0) {
      static const bool predict = [] {
        const char* e = getenv("HB_PREDICT_OPEN");
        return !(e && atoi(e) == 0);
      }();
      if (predict && j >= 256) {
        double* dg = ws<double>(c, B_RDIAG2, (size_t)j);
        HB_CUDA(cudaMemcpy2DAsync(dg, sizeof(double), A, (lda + 1) * sizeof(double), sizeof(double),
                                  (size_t)j, cudaMemcpyDeviceToDevice, st));
        std::vector<double> hd((size_t)j);
        HB_CUDA(cudaMemcpyAsync(hd.data(), dg, sizeof(double) * j, cudaMemcpyDeviceToHost, st));
        {
          TraceSync ts;
          HB_CUDA(cudaStreamSynchronize(st));
        }
        const double thr = tol_min * sigma1_est;
        int64_t ph = -1;
        for (int64_t i = 0; i < j; ++i)
          if (std::fabs(hd[(size_t)i]) < thr) { ph = i; break; }
        const int64_t mw = std::min<int64_t>({64, ph / 4, (j - 1 - ph) / 2});
        if (ph > 0 && mw >= 8) {
          const double lo = std::fabs(hd[(size_t)(ph - mw)]), hi = std::fabs(hd[(size_t)(ph + mw)]);
          const double slope = (lo > 0.0 && hi > 0.0) ? std::log(lo / hi) / (2.0 * mw) : 0.0;  // per index
          const double expected = slope > 0.0 ? 0.5 * eta_cur * eta_cur / slope : 0.0;
          static const bool dbg = getenv("HB_DEBUG_STOP") != nullptr;
          if (dbg) fprintf(stderr, "[predict] j=%lld p~%lld slope=%.3g expected=%.3g eta=%.3g\n", (long long)j,
                           (long long)ph, slope, expected, eta_cur);
          last_slope = slope;
          if (expected > 0.1) {
            // the η at which ~0.1 σ are expected in the window (never below η/5): factor on to
            // it and certify once there
            const double eta_new = std::max(0.2 * eta_cur, std::sqrt(2.0 * 0.1 * slope));
            if (eta_new < 0.9 * eta_cur) {
              eta_cur = eta_new;
              ++skips;
              continue;
            }
          }
        }
      }
    }
    k = j;
    HB_CUDA(cudaEventRecord(c->ev[2], st));

    // ---- certification: σ(R_k) ------------------------------------------------------------
    // queries [0, ntol): δ = ‖A22‖_F (deterministic); [ntol, 2 ntol): δ = 2σ̂(A22) (counts only)
    SigmaQuery hq[2 * HB_MAX_TOLS];
    const int nq = delta2 < INFINITY ? 2 * ntol : ntol;
    for (int t = 0; t < ntol; ++t) {
      hq[t] = SigmaQuery{tols[t], delta, 0, 0};
      hq[ntol + t] = SigmaQuery{tols[t], delta2 < INFINITY ? delta2 : delta, 1, 0};
    }
    std::memset(ans, 0, sizeof(ans));
    if (k > 0) {
      const int64_t ldb = round_up(n, 8);
      double* Bc = ws<double>(c, B_CERT_B, (size_t)ldb * k);
      dim3 tb(32, 8), tg((unsigned)ceil_div(n, 32), (unsigned)ceil_div(k, 32));
      Phase ph_qr(c, HB_PH_CERT_QR);
      transpose_upper_kernel<<<tg, tb, 0, st>>>(A, lda, k, n, Bc, ldb);
      HB_LAUNCH_CHECK();
      const int bq_max = kBlockMax;
      for (int64_t jj = 0; jj < k; jj += bq_max) {
        const int bq = (int)std::min<int64_t>(bq_max, k - jj);
        double* P = Bc + jj + jj * ldb;
        panel_and_T(c, P, ldb, n - jj, bq, V, ldv, tau, T);
        if (jj + bq < k)
          apply_block_reflector(c, V, ldv, T, bq, Bc + jj + (jj + bq) * ldb, ldb, n - jj,
                                k - jj - bq, nullptr);
      }
      const int64_t ldm = round_up(k, 8);
      double* Mk = ws<double>(c, B_CERT_M, (size_t)ldm * k);
      copy_upper_kernel<<<(unsigned)ceil_div(k * k, 256), 256, 0, st>>>(Bc, ldb, k, Mk, ldm);
      HB_LAUNCH_CHECK();
      ph_qr.close();
      Phase ph_bd(c, HB_PH_BIDIAG);
      double* d = ws<double>(c, B_D, (size_t)k + 1);
      double* e = ws<double>(c, B_E, (size_t)k + 1);
      two_stage_bidiag(c, Mk, ldm, k, d, e, V, ldv, tau, T);
      ph_bd.close();
      Phase ph_bs(c, HB_PH_BISECT);
      SigmaQuery* dq = ws<SigmaQuery>(c, B_QUERY, 2 * HB_MAX_TOLS);
      SigmaAnswer* da = ws<SigmaAnswer>(c, B_ANSWER, 2 * HB_MAX_TOLS);
      HB_CUDA(cudaMemcpyAsync(dq, hq, sizeof(SigmaQuery) * nq, cudaMemcpyHostToDevice, st));
      const size_t tg_bytes = (size_t)(2 * k) * sizeof(double);
      const int tg_smem = tg_bytes <= 200 * 1024 ? 1 : 0;
      double* tg_glob = tg_smem ? nullptr : ws<double>(c, B_TG, (size_t)2 * k);
      if (tg_smem) ensure_dyn_smem((const void*)sigma_queries_kernel, tg_bytes);
      sigma_queries_kernel<<<1, 512, tg_smem ? tg_bytes : 0, st>>>(d, e, k, dq, nq, da, tg_glob, tg_smem);
      HB_LAUNCH_CHECK();
      sync_to_host(c, da, ans, sizeof(SigmaAnswer) * nq);
    }
    bool open = false;
    for (int t = 0; t < ntol; ++t) {
      cert_kind[t] = 0;
      if (ans[t].rank_lo == ans[t].rank_hi) cert_kind[t] = 1;
      else if (nq > ntol && ans[ntol + t].rank_hi == ans[t].rank_lo) cert_kind[t] = 2;
      open |= cert_kind[t] == 0;
    }
    ++certs;
    if (!open || j >= kmax || certs >= 4) break;
    // open bracket: with a density estimate, the η expecting ~0.02 σ in the window (in [η/5, η/2]);
    // without one, η/5
    eta_cur = last_slope > 0.0 ? std::min(0.5 * eta_cur, std::max(0.2 * eta_cur, std::sqrt(2.0 * 0.02 * last_slope)))
                               : 0.2 * eta_cur;
  }
  HB_CUDA(cudaEventRecord(c->ev[3], st));
  {
    TraceSync ts;
    HB_CUDA(cudaEventSynchronize(c->ev[3]));
  }
  float f_ms = 0.f, c_ms = 0.f;
  HB_CUDA(cudaEventElapsedTime(&f_ms, c->ev[1], c->ev[2]));
  HB_CUDA(cudaEventElapsedTime(&c_ms, c->ev[2], c->ev[3]));
  if (c->profiling) {
    prof_resolve(c);
    c->stats.problems += 1;
  }
  if (fact_ms) *fact_ms = f_ms;
  if (cert_ms) *cert_ms = c_ms;
  c->last_k = k;
  c->last_sigma1 = k > 0 ? ans[0].sigma1 : 0.0;
  for (int t = 0; t < ntol; ++t) {
    hb_rank_result& r = out[t];
    std::memset(&r, 0, sizeof(r));
    r.rank = ans[t].rank_lo;
    r.rank_lo = ans[t].rank_lo;
    r.rank_hi = ans[t].rank_hi;
    r.k_factored = (int32_t)k;
    r.sigma1 = ans[t].sigma1;
    r.sigma_r = ans[t].sigma_p;
    r.sigma_r1 = ans[t].sigma_p1;
    const double thr = tols[t] * ans[t].sigma1;
    double gap = INFINITY;
    if (thr > 0.0) {
      if (r.rank > 0) gap = std::min(gap, r.sigma_r / thr - 1.0);
      if (r.rank < kmax) gap = std::min(gap, 1.0 - r.sigma_r1 / thr);
    }
    r.gap = gap;
    r.certificate = cert_kind[t];
    // Householder QR is backward stable: the computed factors are exact for A + E with
    // ‖E‖ ≈ sqrt(N)·u·‖A‖_F; relative to the threshold that is the band a count could move by
    if (fro_a2 < 0.0) {  // no block ran (tiny problem): read ‖A‖_F² now
      double h3[3];
      sync_to_host(c, scal, h3, sizeof(h3));
      fro_a2 = h3[2];
    }
    r.fp_band = thr > 0.0 ? std::sqrt((double)std::max(m, n)) * 0x1p-53 * std::sqrt(std::max(fro_a2, 0.0)) / thr
                          : 0.0;
    r.resid = cert_kind[t] == 2 ? delta2 : delta;
    if (cert_kind[t] == 2) r.rank_hi = ans[ntol + t].rank_hi;
    r.sec[1] = f_ms * 1e-3;
    r.sec[2] = c_ms * 1e-3;
  }
}

size_t prof_event(hb_context* c) {
  if (c->evused == c->evpool.size()) {
    cudaEvent_t e;
    HB_CUDA(cudaEventCreate(&e));
    c->evpool.push_back(e);
  }
  const size_t i = c->evused++;
  HB_CUDA(cudaEventRecord(c->evpool[i], c->stream));
  return i;
}

void prof_resolve(hb_context* c) {
  if (!c->profiling && c->marks.empty()) return;
  for (const auto& mk : c->marks) {
    float ms = 0.f;
    if (mk.e0 >= c->evused || mk.e1 >= c->evused) continue;
    cudaEventSynchronize(c->evpool[mk.e1]);
    if (cudaEventElapsedTime(&ms, c->evpool[mk.e0], c->evpool[mk.e1]) != cudaSuccess) {
      (void)cudaGetLastError();  // a profiling hiccup must not poison the next launch check
      continue;
    }
    if (mk.phase == PH_GEMM) {
      c->stats.gemm_ms += ms;
      c->stats.gemm_flops += mk.flops;
      c->stats.gemm_launches += 1;
    } else if (mk.phase >= 0 && mk.phase < HB_NPHASE) {
      c->stats.phase_ms[mk.phase] += ms;
    }
  }
  c->marks.clear();
  c->evused = 0;
}

void debug_sync_after_launch(const char* file, int line) {
  fprintf(stderr, "[hb sync] %s:%d ...", file, line);
  fflush(stderr);
  const cudaError_t e = cudaDeviceSynchronize();
  fprintf(stderr, " %s\n", cudaGetErrorString(e));
}

void context_init(hb_context* c, int device) {
  c->device = device;
  HB_CUDA(cudaSetDevice(device));
  HB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  HB_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  c->coop_sms = c->num_sms;
  {
    size_t free_b = 0;
    HB_CUDA(cudaMemGetInfo(&free_b, &c->total_mem));
  }
  if (const char* e = getenv("HB_SPECTRAL")) c->spectral = atoi(e) != 0;  // experiments / sweeps
  cudaMemPool_t pool;
  HB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;
  HB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  HB_CUDA(cudaMalloc(&c->bar, 64 * sizeof(unsigned int)));
  // stream-ordered and waited for: a legacy-stream cudaMemset is not ordered before work on the
  // non-blocking context stream, and a grid barrier starting from garbage never releases
  HB_CUDA(cudaMemsetAsync(c->bar, 0, 64 * sizeof(unsigned int), c->stream));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  HB_CUDA(cudaMallocHost(&c->pinned, 4096));
  for (auto& e : c->ev) HB_CUDA(cudaEventCreate(&e));
  c->bufs.resize(B_COUNT);
}

// Re-create the context stream with another CUDA priority (workspace stays allocated: it was
// allocated stream-ordered, and the old stream is drained first).
void context_set_priority(hb_context* c, int prio) {
  if (c->priority == prio) return;
  HB_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = nullptr;
  HB_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  HB_CUDA(cudaStreamDestroy(c->stream));
  c->stream = s;
  c->priority = prio;
}

void context_trim(hb_context* c, size_t keep_bytes) {
  HB_CUDA(cudaSetDevice(c->device));
  for (auto& b : c->bufs)
    if (b.p && b.cap > keep_bytes) {
      HB_CUDA(cudaFreeAsync(b.p, c->stream));
      b.p = nullptr;
      b.cap = 0;
    }
}

void context_free(hb_context* c) {
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& b : c->bufs)
    if (b.p) cudaFreeAsync(b.p, c->stream);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->bar) cudaFree(c->bar);
  if (c->pinned) cudaFreeHost(c->pinned);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->evpool) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
}

}  // namespace hb
