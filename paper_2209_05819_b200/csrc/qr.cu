// k3: sketch-pivoted blocked Householder QR building blocks (sm_100a).
//
// This replaces SPEC `epsilon_rank` ("computes full singular values") with a
// rank-revealing factorisation that only touches O(N^2 k) flops: HQRRP-style block pivoting.
//   * Ω (ℓ x m, Gaussian, counter-based) sketches the trailing matrix: Y = Ω A (DMMA GEMM).
//   * sketch_cpqr: column-pivoted Householder QR of the small ℓ x n sketch picks b pivots —
//     warp-shuffle norm/argmax search, one grid barrier per pivot, norms recomputed exactly
//     from the updated sketch column (the downdate is free because the column is in flight).
//   * permute: the b chosen columns move to the front (LAPACK swap semantics) in A, Y, perm.
//   * panel_qr: unpivoted Householder QR of the tall m x b panel (grid-cooperative, two grid
//     barriers per column); emits the explicit V and τ; T of the compact-WY form Q = I − V T Vᵀ
//     comes from S = VᵀV (DMMA GEMM) and the forward recurrence of LAPACK dlarft.
//   * the trailing update A2 ← (I − V Tᵀ Vᵀ) A2 and the sketch downdate Y2 −= Y1 R11⁻¹ R12
//     are DMMA GEMMs (dgemm.cu); Z = Y1 R11⁻¹ is a small triangular solve here.
//   * power_sigma1: power iteration on the first b rows of R — a lower bound on σ₁ used for the
//     stopping threshold before the certification computes σ₁ exactly.
#include "common.cuh"
#include "kernels.h"
#include "qr.h"

namespace hb {

// ------------------------------------------------------------------------------------------
// Gaussian Ω: entry (i, c) = Box–Muller of two counter hashes; deterministic in (seed, i, c).
// ------------------------------------------------------------------------------------------
__global__ void gaussian_kernel(double* __restrict__ om, int64_t rows, int64_t cols, int64_t ld,
                                uint64_t seed) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const int64_t i = idx % rows, c = idx / rows;
  const uint64_t h = splitmix64(seed ^ splitmix64((uint64_t)c * 0x100000001B3ull + (uint64_t)i));
  const uint64_t h2 = splitmix64(h);
  const double u1 = ((double)(h >> 11) + 0.5) * 0x1p-53;
  const double u2 = (double)(h2 >> 11) * 0x1p-53;
  om[i + c * ld] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

void launch_gaussian(double* om, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                     cudaStream_t st) {
  const int64_t tot = rows * cols;
  if (tot == 0) return;
  gaussian_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, st>>>(om, rows, cols, ld, seed);
  HB_LAUNCH_CHECK();
}

// ------------------------------------------------------------------------------------------
// sketch_cpqr: b pivots from the ℓ x n_tr sketch.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ bool better(double na, int ia, double nb, int ib) {
  return na > nb || (na == nb && ia < ib);
}

__global__ void __launch_bounds__(256) sketch_cpqr_kernel(SketchParams p) {
  GridSync gbar(p.bar);
  extern __shared__ double nrm_s[];  // norms of this CTA's columns (-1 = chosen)
  const int G = gridDim.x, g = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ell = p.ell;
  const int64_t cpc = ceil_div(p.n_tr, G);
  const int64_t c0 = g * cpc, c1 = min(p.n_tr, c0 + cpc);
  __shared__ double v[kSketchRows];
  __shared__ double wbest[8], wsum[8];
  __shared__ int wbi[8];
  __shared__ double sh_tau;
  __shared__ int sh_piv, sh_stop;
  constexpr int RPL = kSketchRows / 32;  // sketch rows per lane

  // init: copy Y -> Ys, exact column norms
  double best = -1.0, sum = 0.0;
  int bi = INT_MAX;
  for (int64_t q = c0 + warp; q < c1; q += 8) {
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const int i = lane + 32 * t;
      if (i < ell) {
        const double y = p.Y[i + q * p.ldy];
        p.Ys[i + q * p.ldy] = y;
        s += y * y;
      }
    }
    s = warp_sum(s);
    if (lane == 0) nrm_s[q - c0] = s;
    if (better(s, (int)q, best, bi)) { best = s; bi = (int)q; }
    sum += s;
  }
  auto publish = [&](int slot) {
    if (lane == 0) { wbest[warp] = best; wbi[warp] = bi; wsum[warp] = sum; }
    __syncthreads();
    if (tid == 0) {
      double b0 = -1.0, s0 = 0.0;
      int i0 = INT_MAX;
      for (int w = 0; w < 8; ++w) {
        if (better(wbest[w], wbi[w], b0, i0)) { b0 = wbest[w]; i0 = wbi[w]; }
        s0 += wsum[w];
      }
      double* sl = p.slots + ((size_t)slot * G + g) * 3;
      sl[0] = b0; sl[1] = (double)i0; sl[2] = s0;
    }
  };
  publish(0);
  gbar.sync();

  int c = 0;
  for (; c < p.b_req; ++c) {
    // global argmax + total remaining sketch mass (block-parallel, fixed order -> identical in
    // every CTA)
    {
      const double* sl = p.slots + (size_t)(c & 1) * G * 3;
      double b0 = -1.0, s0 = 0.0;
      int i0 = INT_MAX;
      for (int h = tid; h < G; h += 256) {
        if (better(sl[3 * h], (int)sl[3 * h + 1], b0, i0)) { b0 = sl[3 * h]; i0 = (int)sl[3 * h + 1]; }
        s0 += sl[3 * h + 2];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, b0, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i0, o);
        if (better(ob, oi, b0, i0)) { b0 = ob; i0 = oi; }
      }
      s0 = warp_sum(s0);
      if (lane == 0) { wbest[warp] = b0; wbi[warp] = i0; wsum[warp] = s0; }
      __syncthreads();
      if (tid == 0) {
        double bb = -1.0, ss = 0.0;
        int ii = INT_MAX;
        for (int w = 0; w < 8; ++w) {
          if (better(wbest[w], wbi[w], bb, ii)) { bb = wbest[w]; ii = wbi[w]; }
          ss += wsum[w];
        }
        const double est = c < ell ? ss / (double)(ell - c) : 0.0;
        if (g == 0) p.out_est[c] = est;
        int stop = 0;
        if (!(bb > 0.0) || c >= ell) stop = 1;
        else if (c >= p.b_min && (c % 8) == 0 && est <= p.stop_fro2) stop = 1;
        sh_stop = stop;
        sh_piv = ii;
      }
    }
    __syncthreads();
    if (sh_stop) break;
    const int piv = sh_piv;
    // Householder vector of the pivot column (rows c..ell-1), computed redundantly per CTA
    if (warp == 0) {
      double s = 0.0;
      for (int i = c + 1 + lane; i < ell; i += 32) {
        const double y = p.Ys[i + (int64_t)piv * p.ldy];
        v[i] = y;
        s += y * y;
      }
      s = warp_sum(s);
      const double alpha = p.Ys[c + (int64_t)piv * p.ldy];
      double tau = 0.0, scal = 0.0, beta = alpha;
      if (s > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + s), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      for (int i = c + 1 + lane; i < ell; i += 32) v[i] *= scal;
      if (lane == 0) {
        v[c] = 1.0;
        sh_tau = tau;
        if (g == 0) { p.piv[c] = piv; p.rdiag[c] = fabs(beta); }
      }
    }
    __syncthreads();
    const double tau = sh_tau;
    double vr[RPL];
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const int i = lane + 32 * t;
      vr[t] = (i >= c && i < ell) ? v[i] : 0.0;
    }
    best = -1.0; sum = 0.0; bi = INT_MAX;
    // two columns per warp iteration: all their loads are issued before the first reduction
    for (int64_t qa = c0 + warp; qa < c1; qa += 16) {
      const int64_t qb = qa + 8;
      const bool va = qa != piv && nrm_s[qa - c0] >= 0.0;
      const bool vb = qb < c1 && qb != piv && nrm_s[qb - c0] >= 0.0;
      double* ca = p.Ys + qa * p.ldy;
      double* cb = p.Ys + qb * p.ldy;
      double ya[RPL], yb[RPL];
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int i = lane + 32 * t;
        const bool act = i >= c && i < ell;
        ya[t] = (va && act) ? ca[i] : 0.0;
        yb[t] = (vb && act) ? cb[i] : 0.0;
      }
      double wa = 0.0, wb = 0.0;
#pragma unroll
      for (int t = 0; t < RPL; ++t) { wa += vr[t] * ya[t]; wb += vr[t] * yb[t]; }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        wa += __shfl_xor_sync(0xffffffffu, wa, o);
        wb += __shfl_xor_sync(0xffffffffu, wb, o);
      }
      wa *= tau; wb *= tau;
      double sa = 0.0, sb = 0.0;
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int i = lane + 32 * t;
        const bool act = i >= c && i < ell;
        const double xa = ya[t] - wa * vr[t], xb = yb[t] - wb * vr[t];
        if (act) {
          if (va) ca[i] = xa;
          if (vb) cb[i] = xb;
          if (i > c) { sa += xa * xa; sb += xb * xb; }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
      }
      if (va) {
        if (lane == 0) nrm_s[qa - c0] = sa;
        if (better(sa, (int)qa, best, bi)) { best = sa; bi = (int)qa; }
        sum += sa;
      } else if (qa == piv && lane == 0) {
        nrm_s[qa - c0] = -1.0;
      }
      if (vb) {
        if (lane == 0) nrm_s[qb - c0] = sb;
        if (better(sb, (int)qb, best, bi)) { best = sb; bi = (int)qb; }
        sum += sb;
      } else if (qb < c1 && qb == piv && lane == 0) {
        nrm_s[qb - c0] = -1.0;
      }
    }
    __syncthreads();
    publish((c + 1) & 1);
    gbar.sync();
  }
  if (g == 0 && tid == 0) {
    // LAPACK-style swap list: swaps[i] = current position of the i-th pivot when it is
    // exchanged with position i.
    int pos[kBlockMax];
    for (int i = 0; i < c; ++i) pos[i] = p.piv[i];
    for (int i = 0; i < c; ++i) {
      const int src = pos[i];
      p.swaps[i] = src;
      if (src != i)
        for (int t = i + 1; t < c; ++t)
          if (pos[t] == i) pos[t] = src;
    }
    *p.out_b = c;
  }
}

// Shared-memory variant of sketch_cpqr.  Each CTA keeps its ℓ x cpc block of the sketch in
// shared memory.  Per pivot: every CTA publishes (best norm, index, remaining mass) and the
// column of its best candidate; after ONE grid barrier all CTAs reduce the slots in the same
// fixed order (identical decisions everywhere), read the winner's column from its candidate slot,
// form the Householder vector redundantly, update their own columns and recompute their norms
// exactly.
__global__ void __launch_bounds__(kSketchThreads) sketch_cpqr_smem_kernel(SketchParams p) {
  GridSync gbar(p.bar);
  constexpr int NW = kSketchThreads / 32;
  constexpr int RPL = kSketchRows / 32;
  extern __shared__ double ssm[];
  const int G = gridDim.x, g = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ell = p.ell;
  const int64_t cpc = ceil_div(p.n_tr, G);
  const int64_t c0 = g * cpc, c1 = min(p.n_tr, c0 + cpc);
  const int ncol = (int)max((int64_t)0, c1 - c0);
  double* Ysm = ssm;                          // [cpc][ell]
  double* nrm_s = ssm + (size_t)cpc * ell;    // [cpc] (-1 = chosen)
  __shared__ double v[kSketchRows];
  __shared__ double wbest[NW], wsum[NW];
  __shared__ int wbi[NW];
  __shared__ double sh_tau;
  __shared__ int sh_win;
  __shared__ int wh[NW];
  int piv_r = 0, win_r = 0, stop_r = 0;

  double best = -1.0, sum = 0.0;
  int bi = INT_MAX;
  for (int q = warp; q < ncol; q += NW) {
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const int i = lane + 32 * t;
      double y = 0.0;
      if (i < ell) y = p.Y[i + (c0 + q) * p.ldy];
      Ysm[q * ell + i] = y;
      s += y * y;
    }
    s = warp_sum(s);
    if (lane == 0) nrm_s[q] = s;
    if (better(s, (int)(c0 + q), best, bi)) { best = s; bi = (int)(c0 + q); }
    sum += s;
  }
  // CTA-level (best, index, mass) -> slot; the best candidate's column -> candidate slot
  auto publish = [&](int par) {
    if (lane == 0) { wbest[warp] = best; wbi[warp] = bi; wsum[warp] = sum; }
    __syncthreads();
    if (tid == 0) {
      double b0 = -1.0, s0 = 0.0;
      int i0 = INT_MAX;
      for (int w = 0; w < NW; ++w) {
        if (better(wbest[w], wbi[w], b0, i0)) { b0 = wbest[w]; i0 = wbi[w]; }
        s0 += wsum[w];
      }
      double* sl = p.slots + ((size_t)par * G + g) * 3;
      sl[0] = b0; sl[1] = (double)i0; sl[2] = s0;
      sh_win = i0;
    }
    __syncthreads();
    const int w = sh_win;
    if (w != INT_MAX && tid < ell) p.cand[((size_t)par * G + g) * ell + tid] = Ysm[(w - c0) * ell + tid];
  };
  publish(0);
  gbar.sync();

  int c = 0;
  for (; c < p.b_req; ++c) {
    const int par = c & 1;
    {
      const double* sl = p.slots + (size_t)par * G * 3;
      double b0 = -1.0, s0 = 0.0;
      int i0 = INT_MAX, h0 = -1;
      for (int h = tid; h < G; h += kSketchThreads) {
        const double bv = __ldcg(sl + 3 * h);
        const int iv = (int)__ldcg(sl + 3 * h + 1);
        if (better(bv, iv, b0, i0)) { b0 = bv; i0 = iv; h0 = h; }
        s0 += __ldcg(sl + 3 * h + 2);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, b0, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i0, o);
        const int oh = __shfl_xor_sync(0xffffffffu, h0, o);
        if (better(ob, oi, b0, i0)) { b0 = ob; i0 = oi; h0 = oh; }
      }
      s0 = warp_sum(s0);
      if (lane == 0) { wbest[warp] = b0; wbi[warp] = i0; wsum[warp] = s0; wh[warp] = h0; }
      __syncthreads();
      // every thread combines the NW warp results itself (same order: identical decisions), so
      // no second barrier is needed to broadcast them
      double bb = -1.0, ss = 0.0;
      int ii = INT_MAX, hh = -1;
      for (int w = 0; w < NW; ++w) {
        if (better(wbest[w], wbi[w], bb, ii)) { bb = wbest[w]; ii = wbi[w]; hh = wh[w]; }
        ss += wsum[w];
      }
      const double est = c < ell ? ss / (double)(ell - c) : 0.0;
      if (g == 0 && tid == 0) p.out_est[c] = est;
      int stop = 0;
      if (!(bb > 0.0) || c >= ell) stop = 1;
      else if (c >= p.b_min && (c % 8) == 0 && est <= p.stop_fro2) stop = 1;
      piv_r = ii;
      win_r = hh;
      stop_r = stop;
    }
    if (stop_r) break;
    const int piv = piv_r;
    // Householder vector of the winner's column (rows c..ell-1), redundantly in every CTA
    if (warp == 0) {
      const double* col = p.cand + ((size_t)par * G + win_r) * ell;
      double yv[RPL];
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int i = lane + 32 * t;
        yv[t] = i < ell ? __ldcg(col + i) : 0.0;
        if (i > c && i < ell) s += yv[t] * yv[t];
      }
      s = warp_sum(s);
      const int tc = c >> 5;
      const double yc = tc == 0 ? yv[0] : (tc == 1 ? yv[1] : (tc == 2 ? yv[2] : yv[3]));
      const double alpha = __shfl_sync(0xffffffffu, yc, c & 31);
      double tau = 0.0, scal = 0.0, beta = alpha;
      if (s > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + s), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int i = lane + 32 * t;
        if (i < kSketchRows) v[i] = i < c ? 0.0 : (i == c ? 1.0 : (i < ell ? yv[t] * scal : 0.0));
      }
      if (lane == 0) {
        sh_tau = tau;
        if (g == 0) { p.piv[c] = piv; p.rdiag[c] = fabs(beta); }
      }
    }
    __syncthreads();
    const double tau = sh_tau;
    double vr[RPL];
#pragma unroll
    for (int t = 0; t < RPL; ++t) vr[t] = v[lane + 32 * t];
    if (piv >= c0 && piv < c1 && tid == 0) nrm_s[piv - c0] = -1.0;
    __syncthreads();
    best = -1.0; sum = 0.0; bi = INT_MAX;
    for (int qa = warp; qa < ncol; qa += 2 * NW) {
      const int qb = qa + NW;
      const bool va = nrm_s[qa] >= 0.0;
      const bool vb = qb < ncol && nrm_s[qb] >= 0.0;
      double* ca = Ysm + (size_t)qa * ell;
      double* cb = Ysm + (size_t)qb * ell;
      double ya[RPL], yb[RPL];
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int i = lane + 32 * t;
        ya[t] = va ? ca[i] : 0.0;
        yb[t] = vb ? cb[i] : 0.0;
      }
      double wa = 0.0, wb = 0.0;
#pragma unroll
      for (int t = 0; t < RPL; ++t) { wa = fma(vr[t], ya[t], wa); wb = fma(vr[t], yb[t], wb); }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        wa += __shfl_xor_sync(0xffffffffu, wa, o);
        wb += __shfl_xor_sync(0xffffffffu, wb, o);
      }
      wa *= tau; wb *= tau;
      double sa = 0.0, sb = 0.0;
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int i = lane + 32 * t;
        const double xa = fma(-wa, vr[t], ya[t]), xb = fma(-wb, vr[t], yb[t]);
        if (va) ca[i] = xa;
        if (vb) cb[i] = xb;
        if (i > c) { sa = fma(xa, xa, sa); sb = fma(xb, xb, sb); }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
      }
      if (va) {
        if (lane == 0) nrm_s[qa] = sa;
        if (better(sa, (int)(c0 + qa), best, bi)) { best = sa; bi = (int)(c0 + qa); }
        sum += sa;
      }
      if (vb) {
        if (lane == 0) nrm_s[qb] = sb;
        if (better(sb, (int)(c0 + qb), best, bi)) { best = sb; bi = (int)(c0 + qb); }
        sum += sb;
      }
    }
    __syncthreads();
    publish(par ^ 1);
    gbar.sync();
  }
  if (g == 0 && tid == 0) {
    int pos[kBlockMax];
    for (int i = 0; i < c; ++i) pos[i] = p.piv[i];
    for (int i = 0; i < c; ++i) {
      const int src = pos[i];
      p.swaps[i] = src;
      if (src != i)
        for (int t = i + 1; t < c; ++t)
          if (pos[t] == i) pos[t] = src;
    }
    *p.out_b = c;
  }
}

// ------------------------------------------------------------------------------------------
// permute: apply the swap list to A (all m rows), Y (ℓ rows) and perm (one row).
// ------------------------------------------------------------------------------------------
__global__ void permute_kernel(double* __restrict__ A, int64_t lda, int64_t m, double* __restrict__ Y,
                               int64_t ldy, int ell, int64_t* __restrict__ perm, int64_t j,
                               const int* __restrict__ swaps, const int* __restrict__ bptr) {
  __shared__ int sw[kBlockMax];
  const int b = *bptr;
  for (int i = threadIdx.x; i < b; i += blockDim.x) sw[i] = swaps[i];
  __syncthreads();
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r < m) {
    double* row = A + r + j * lda;
    for (int i = 0; i < b; ++i) {
      const int s = sw[i];
      if (s != i) {
        const double t = row[(int64_t)i * lda];
        row[(int64_t)i * lda] = row[(int64_t)s * lda];
        row[(int64_t)s * lda] = t;
      }
    }
  } else if (r < m + ell) {
    double* row = Y + (r - m) + j * ldy;
    for (int i = 0; i < b; ++i) {
      const int s = sw[i];
      if (s != i) {
        const double t = row[(int64_t)i * ldy];
        row[(int64_t)i * ldy] = row[(int64_t)s * ldy];
        row[(int64_t)s * ldy] = t;
      }
    }
  } else if (r == m + ell) {
    int64_t* row = perm + j;
    for (int i = 0; i < b; ++i) {
      const int s = sw[i];
      if (s != i) {
        const int64_t t = row[i];
        row[i] = row[s];
        row[s] = t;
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// panel_qr: Householder QR of the mp x b panel at P (column-major, ld).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) panel_qr_kernel(PanelParams p) {
  GridSync gbar(p.bar);
  extern __shared__ double psm[];  // vs[chunk] | ws[b]
  const int G = gridDim.x, g = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = p.b;
  const int64_t chunk = p.chunk;
  const int64_t r0 = g * chunk, r1 = min(p.mp, r0 + chunk);
  double* vs = psm;
  double* ws = psm + chunk;
  __shared__ double sh[4];
  __shared__ double red[32];
  double* P = p.P;
  const int64_t ld = p.ld;

  // column 0 partial norm (rows > 0)
  if (warp == 0) {
    double s = 0.0;
    for (int64_t i = max(r0, (int64_t)1) + lane; i < r1; i += 32) {
      const double x = P[i];
      s += x * x;
    }
    s = warp_sum(s);
    if (lane == 0) p.nslot[g] = s;
  }
  gbar.sync();

  // reflectors for the first min(b, mp) columns (a wide panel, mp < b, occurs in the block LQ of
  // the band reduction); the remaining columns are only transformed
  const int nref = (int)min((int64_t)b, p.mp);
  for (int c = 0; c < nref; ++c) {
    {
      const double s = block_sum_strided(p.nslot, G, 1, red);
      if (tid == 0) {
      const double alpha = P[c + (int64_t)c * ld];
      double tau = 0.0, scal = 0.0, beta = alpha;
      if (s > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + s), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      sh[0] = tau; sh[1] = scal; sh[2] = beta;
      }
    }
    __syncthreads();
    const double tau = sh[0], scal = sh[1];
    double* colc = P + (int64_t)c * ld;
    for (int64_t i = r0 + tid; i < r1; i += 256) {
      double vi = 0.0;
      if (i > c) {
        vi = colc[i] * scal;
        colc[i] = vi;
      } else if (i == c) {
        vi = 1.0;
      }
      vs[i - r0] = vi;
    }
    __syncthreads();
    const int64_t lo = max(r0, (int64_t)c);
    // partial w_q = sum_i v_i P[i, q]  (q > c)
    for (int q = c + 1 + warp; q < b; q += 8) {
      const double* colq = P + (int64_t)q * ld;
      double s = 0.0;
      for (int64_t i = lo + lane; i < r1; i += 32) s += vs[i - r0] * colq[i];
      s = warp_sum(s);
      if (lane == 0) p.wslot[(size_t)g * b + q] = s;
    }
    gbar.sync();
    for (int q = c + 1 + warp; q < b; q += 8) {
      const double s = warp_sum_strided(p.wslot + q, G, b);
      if (lane == 0) ws[q] = s * tau;
    }
    __syncthreads();
    for (int q = c + 1 + warp; q < b; q += 8) {
      double* colq = P + (int64_t)q * ld;
      const double wq = ws[q];
      double s = 0.0;
      for (int64_t i = lo + lane; i < r1; i += 32) {
        const double x = colq[i] - vs[i - r0] * wq;
        colq[i] = x;
        if (q == c + 1 && i > c + 1) s += x * x;
      }
      if (q == c + 1) {
        s = warp_sum(s);
        if (lane == 0) p.nslot[g] = s;
      }
    }
    if (c + 1 >= b && tid == 0) p.nslot[g] = 0.0;
    if (c >= r0 && c < r1 && tid == 0) colc[c] = sh[2];
    if (g == 0 && tid == 0) p.tau[c] = tau;
    gbar.sync();
  }
  // explicit V (unit diagonal, zeros above; zero columns beyond the last reflector)
  for (int q = warp; q < b; q += 8) {
    const double* colq = P + (int64_t)q * ld;
    double* vq = p.V + (int64_t)q * p.ldv;
    for (int64_t i = r0 + lane; i < r1; i += 32)
      vq[i] = q >= nref ? 0.0 : (i > q ? colq[i] : (i == q ? 1.0 : 0.0));
  }
  if (g == 0)
    for (int q = nref + tid; q < b; q += 256) p.tau[q] = 0.0;
}

// T of the compact-WY form from S = VᵀV and τ (LAPACK dlarft, forward/columnwise), built by
// recursive merging instead of the column recurrence T[0:c, c] = −τ_c·T[0:c,0:c]·S[0:c, c]
// (whose b dependent steps made this a ~250 µs latency chain at b = 120):
//   leaves: 8-column diagonal blocks by the recurrence (one warp each);
//   level w: adjacent blocks [a, m) and [m, e) merge with T12 = −T1·S12·T2, all merges of a level
//   in parallel (W = S12·T2 is parked, transposed, in T's unused lower-left block).
// S's strict upper triangle (packed) and T live in shared memory.
__global__ void build_T_kernel(const double* __restrict__ S, int64_t lds, const double* __restrict__ tau,
                               int b, double* __restrict__ T, int64_t ldt) {
  extern __shared__ double smT[];
  const int ldT = b + 1;
  double* Ts = smT;                        // b x b, column-major, ld b+1
  double* Sp = smT + (size_t)b * ldT;      // packed strict upper: (r, c), r < c at c(c-1)/2 + r
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  auto sp = [&](int r, int c) { return Sp[c * (c - 1) / 2 + r]; };
  for (int e = tid; e < b * ldT; e += nt) Ts[e] = 0.0;
  {
    constexpr int U = 8;
    const int tot = b * b;
    for (int e0 = tid; e0 < tot; e0 += nt * U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * nt;
        const int r = e % b, c = e / b;
        v[u] = (e < tot && r < c) ? S[r + (int64_t)c * lds] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * nt;
        const int r = e % b, c = e / b;
        if (e < tot && r < c) Sp[c * (c - 1) / 2 + r] = v[u];
      }
    }
  }
  __syncthreads();
  // leaves
  for (int L = warp; L * 8 < b; L += nw) {
    const int a = L * 8, n8 = min(8, b - a);
    for (int c = 0; c < n8; ++c) {
      const double tc = tau[a + c];
      if (lane < c) {
        double s = 0.0;
        for (int k = lane; k < c; ++k) s += Ts[(a + lane) + (a + k) * ldT] * sp(a + k, a + c);
        Ts[(a + lane) + (a + c) * ldT] = -tc * s;
      } else if (lane == c) {
        Ts[(a + c) + (a + c) * ldT] = tc;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int w = 8; w < b; w *= 2) {
    const int nm = (b + 2 * w - 1) / (2 * w);
    const int per = w * w;
    // W[r][j] = Σ_{k<=j} S12[r][k]·T2[k][j]  -> Ts[(m+j) + (a+r)·ldT]
    for (int e = tid; e < nm * per; e += nt) {
      const int i = e / per, rem = e % per, r = rem % w, j = rem / w;
      const int a = 2 * w * i, m = min(a + w, b), ee = min(a + 2 * w, b);
      if (a + r >= m || m + j >= ee) continue;
      double s = 0.0;
      for (int k = 0; k <= j; ++k) s += sp(a + r, m + k) * Ts[(m + k) + (m + j) * ldT];
      Ts[(m + j) + (a + r) * ldT] = s;
    }
    __syncthreads();
    // T12[r][j] = −Σ_{k>=r} T1[r][k]·W[k][j]
    for (int e = tid; e < nm * per; e += nt) {
      const int i = e / per, rem = e % per, r = rem % w, j = rem / w;
      const int a = 2 * w * i, m = min(a + w, b), ee = min(a + 2 * w, b);
      if (a + r >= m || m + j >= ee) continue;
      double s = 0.0;
      for (int k = r; k < m - a; ++k) s += Ts[(a + r) + (a + k) * ldT] * Ts[(m + j) + (a + k) * ldT];
      Ts[(a + r) + (m + j) * ldT] = -s;
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += nt) {
    const int r = e % b, c = e / b;
    T[r + (int64_t)c * ldt] = r <= c ? Ts[r + c * ldT] : 0.0;
  }
}

// Z (ell x b) = Y1 R11^{-1}: one thread per sketch row, 8 columns at a time (8 independent FMA
// chains per thread).  R11 is staged in shared memory as row-major 8-column strips
// (strip B holds R[0:8B+8, 8B:8B+8] at offset 32·B·(B+1)), Z as Zs[c·ell + t].
__global__ void sketch_trsm_kernel(const double* __restrict__ Y1, int64_t ldy, int ell,
                                   const double* __restrict__ R, int64_t ldr, int b,
                                   double* __restrict__ Z, int64_t ldz) {
  extern __shared__ double smZ[];
  const int nb8 = (b + 7) / 8;
  double* Rs = smZ;                                  // 32·nb8·(nb8+1) doubles
  double* Zs = smZ + (size_t)32 * nb8 * (nb8 + 1);   // b x ell
  const int t = threadIdx.x, nt = blockDim.x;
  for (int B = 0; B < nb8; ++B) {
    double* strip = Rs + 32 * B * (B + 1);
    const int rows = 8 * B + 8;
    for (int e = t; e < rows * 8; e += nt) {
      const int i = e >> 3, jj = e & 7, c = 8 * B + jj;
      double v;
      if (c >= b) v = (i == c) ? 1.0 : 0.0;          // padding column: identity
      else v = (i <= c) ? R[i + (int64_t)c * ldr] : 0.0;
      strip[e] = v;
    }
  }
  __syncthreads();
  if (t >= ell) return;
  for (int B = 0; B < nb8; ++B) {
    const int a = 8 * B;
    const double* strip = Rs + 32 * B * (B + 1);
    double acc[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) acc[jj] = (a + jj < b) ? Y1[t + (int64_t)(a + jj) * ldy] : 0.0;
    for (int i = 0; i < a; ++i) {
      const double z = Zs[i * ell + t];
      const double2* r2 = reinterpret_cast<const double2*>(strip + i * 8);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 rv = r2[h];
        acc[2 * h] = fma(-z, rv.x, acc[2 * h]);
        acc[2 * h + 1] = fma(-z, rv.y, acc[2 * h + 1]);
      }
    }
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const double d = strip[(a + jj) * 8 + jj];
      const double z = d != 0.0 ? acc[jj] / d : 0.0;
#pragma unroll
      for (int j2 = jj + 1; j2 < 8; ++j2) acc[j2] = fma(-z, strip[(a + jj) * 8 + j2], acc[j2]);
      if (a + jj < b) {
        Zs[(a + jj) * ell + t] = z;
        Z[t + (int64_t)(a + jj) * ldz] = z;
      }
    }
  }
}

// σ₁ lower bound: power iteration on R_b = rows 0..b-1 of the factor (upper trapezoidal; the
// strictly-lower part of the first b columns holds V and is masked).
__global__ void __launch_bounds__(256) power_sigma1_kernel(PowerParams p) {
  GridSync gbar(p.bar);
  const int G = gridDim.x, g = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = p.b;
  const int64_t cpc = ceil_div(p.n, G);
  const int64_t c0 = g * cpc, c1 = min(p.n, c0 + cpc);
  __shared__ double x[kBlockMax], acc[8][kBlockMax];
  __shared__ double ysum[8];
  __shared__ double sh_norm;
  double best = 0.0;
  for (int it = 0; it <= p.iters; ++it) {
    // x from previous partials (it == 0: ones)
    {
      const double* prev = p.slots + (size_t)((it - 1) & 1) * G * (b + 1);
      for (int i = warp; i <= b; i += 8) {
        const double s = it == 0 ? (i < b ? 1.0 : 0.0) : warp_sum_strided(prev + i, G, b + 1);
        if (lane == 0) {
          if (i < b) x[i] = s;
          else ysum[0] = s;
        }
      }
      __syncthreads();
      if (tid == 0 && it > 0) best = fmax(best, sqrt(ysum[0]));  // ||R^T x_hat|| of the previous iterate
      __syncthreads();
    }
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int i = 0; i < b; ++i) s += x[i] * x[i];
      sh_norm = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
    }
    __syncthreads();
    if (tid < b) x[tid] *= sh_norm;
    for (int i = tid; i < 8 * kBlockMax; i += 256) (&acc[0][0])[i] = 0.0;
    __syncthreads();
    if (it == p.iters) break;
    double yy = 0.0;
    for (int64_t c = c0 + warp; c < c1; c += 8) {
      const double* col = p.R + c * p.ld;
      const int rmax = (p.mask && c < b) ? (int)c + 1 : b;
      double s = 0.0;
      for (int i = lane; i < rmax; i += 32) s += col[i] * x[i];
      s = warp_sum(s);
      yy += s * s;
      if (p.yout && it == p.iters - 1 && lane == 0) p.yout[c] = s;
      for (int i = lane; i < rmax; i += 32) acc[warp][i] += col[i] * s;
    }
    if (lane == 0) ysum[warp] = yy;
    __syncthreads();
    double* sl = p.slots + (size_t)(it & 1) * G * (b + 1) + (size_t)g * (b + 1);
    if (tid < b) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += acc[w][tid];
      sl[tid] = s;
    }
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += ysum[w];
      sl[b] = s;
    }
    gbar.sync();
  }
  if (g == 0 && tid == 0) *p.out = best;
}

__global__ void sum_kernel(const double* __restrict__ parts, int64_t n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += parts[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

// B (n x k) = upper-trapezoidal rows 0..k-1 of A (m x n), transposed; zero below the diagonal.
__global__ void transpose_upper_kernel(const double* __restrict__ A, int64_t lda, int64_t k,
                                       int64_t n, double* __restrict__ B, int64_t ldb) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t c = c0 + r, i = i0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < k && c < n && c >= i) ? A[i + c * lda] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, c = c0 + threadIdx.x;
    if (i < k && c < n) B[c + i * ldb] = tile[threadIdx.x][r];
  }
}

// λ_max lower bound of the symmetric positive semidefinite b x b Gram matrix G (ld b) by power
// iteration in one CTA: every Rayleigh quotient xᵀGx / xᵀx is <= λ_max, so sqrt of the largest
// one seen is a lower bound on σ₁ of the matrix whose Gram G is (up to rounding).
__global__ void __launch_bounds__(256) gram_sigma1_kernel(const double* __restrict__ G, int b, int iters,
                                                          double* __restrict__ out) {
  extern __shared__ double gs[];  // b x b
  __shared__ double x[kSketchRows], y[kSketchRows], part[2][kSketchRows], red[3][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < b * b; e += blockDim.x) gs[e] = G[e];
  for (int i = tid; i < b; i += blockDim.x) x[i] = 1.0;
  __syncthreads();
  // thread (i, h): half h of row i's dot product (b <= 128 rows x 2 halves = 256 threads), so
  // the dependent FMA chain is b/2 long; the three reductions share one pass
  const int i = tid % kSketchRows, h = tid / kSketchRows;
  const int j0 = h * ((b + 1) / 2), j1 = h ? b : (b + 1) / 2;
  double best = 0.0;
  for (int it = 0; it < iters; ++it) {
    if (i < b) {
      double s = 0.0;
      for (int j = j0; j < j1; ++j) s = fma(gs[i + j * b], x[j], s);  // G symmetric: row i = column i
      part[h][i] = s;
    }
    __syncthreads();
    double xx = 0.0, xy = 0.0, yy = 0.0;
    if (h == 0 && i < b) {
      const double s = part[0][i] + part[1][i];
      y[i] = s;
      xx = x[i] * x[i];
      xy = x[i] * s;
      yy = s * s;
    }
    xx = warp_sum(xx);
    xy = warp_sum(xy);
    yy = warp_sum(yy);
    if (lane == 0) { red[0][warp] = xx; red[1][warp] = xy; red[2][warp] = yy; }
    __syncthreads();
    xx = 0.0; xy = 0.0; yy = 0.0;
    for (int w = 0; w < 8; ++w) { xx += red[0][w]; xy += red[1][w]; yy += red[2][w]; }
    if (xx > 0.0) best = fmax(best, xy / xx);
    const double sc = yy > 0.0 ? 1.0 / sqrt(yy) : 0.0;
    if (h == 0 && i < b) x[i] = y[i] * sc;
    __syncthreads();
  }
  if (tid == 0) *out = sqrt(fmax(best, 0.0));
}

// C (k x k) = upper triangle of B[0:k, 0:k].
__global__ void copy_upper_kernel(const double* __restrict__ B, int64_t ldb, int64_t k,
                                  double* __restrict__ C, int64_t ldc) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= k * k) return;
  const int64_t i = idx % k, c = idx / k;
  C[i + c * ldc] = i <= c ? B[i + c * ldb] : 0.0;
}

}  // namespace hb

namespace hb {
__global__ void iota_kernel(int64_t* __restrict__ p, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}
// Sum of squares of a column-major m x n matrix: block b sums a fixed grid-strided subset into
// parts[b] (fixed order, deterministic); sum_kernel folds the partials.
__global__ void sumsq_kernel(const double* __restrict__ A, int64_t m, int64_t n, int64_t ld,
                             double* __restrict__ parts) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < m * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const double v = A[idx % m + (idx / m) * ld];
    s += v * v;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) parts[blockIdx.x] = s;
}

__global__ void nonfinite_kernel(const double* __restrict__ A, int64_t m, int64_t n, int64_t ld,
                                 unsigned int* flags) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= m * n) return;
  const int64_t i = idx % m, c = idx / m;
  if (!isfinite(A[i + c * ld])) atomicOr(flags, 2u);
}
}  // namespace hb

namespace hb {
// Spectral-norm check of the residual (block power method without re-orthogonalisation, so
// every column is an independent power iteration): normalise each column of X (rows x cols)
// and record its pre-normalisation norm in norms[c] (max over the run = lower bound on σ₁).
__global__ void colnorm_normalize_kernel(double* __restrict__ X, int64_t ld, int64_t rows,
                                         double* __restrict__ norms, double* __restrict__ best) {
  __shared__ double red[32];
  const int c = blockIdx.x;
  double* x = X + (int64_t)c * ld;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) s += x[i] * x[i];
  s = block_sum(s, red);
  const double nrm = sqrt(s);
  const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) x[i] *= inv;
  if (threadIdx.x == 0) {
    norms[c] = nrm;
    if (best) best[c] = fmax(best[c], nrm);
  }
}
__global__ void max_kernel(const double* __restrict__ v, int n, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < n; ++i) m = fmax(m, v[i]);
    *out = m;
  }
}
}  // namespace hb
