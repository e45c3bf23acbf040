// Certification kernels: Golub–Kahan bidiagonalisation of the k x k triangle R' (from the QR of
// R_kᵀ) and Sturm-count bisection on the Golub–Kahan tridiagonal (TGK) of the bidiagonal.
//
// The ε-rank definition needs singular values; the rank
// test count(σ > tol·σ₁) and the boundary gap only need σ₁, σ_p, σ_{p+1} and two counts, which
// bisection on the bidiagonal delivers to high relative accuracy without computing the rest.
//
#include "common.cuh"
#include "kernels.h"
#include "qr.h"

namespace hb {

// ---- bisection on the TGK matrix of the upper bidiagonal (d, e) ----------------------------
// count_less(x) = #singular values < x (x > 0): Sturm count of TGK − xI over the off-diagonal
// sequence d0, e0, d1, e1, ..., d_{k-1}; TGK has eigenvalues ±σ_i.
__device__ int64_t count_less(const double* __restrict__ d, const double* __restrict__ e, int64_t k,
                              double x, double pivmin) {
  double q = -x;
  int64_t neg = q < 0.0;
  for (int64_t t = 1; t < 2 * k; ++t) {
    const double a = (t & 1) ? d[(t - 1) >> 1] : e[(t - 2) >> 1];
    if (fabs(q) < pivmin) q = -pivmin;
    q = -x - (a * a) / q;
    neg += q < 0.0;
  }
  return neg - k;
}

// j-th largest singular value (1-based) by 32-way multisection within [lo, hi] (warp-wide).
__device__ double kth_largest(const double* d, const double* e, int64_t k, int64_t j, double lo,
                              double hi, double pivmin, double rel = 4e-16) {
  const int lane = threadIdx.x & 31;
  const int64_t need = k - j + 1;  // σ_(j) = inf{x : count_less(x) >= need}
  // geometric multisection while the bracket spans more than a factor 4 (σ's near the
  // threshold can sit many decades below σ₁), then linear multisection to relative `rel`
  if (!(lo > 0.0)) lo = hi * 1e-300;
  for (int it = 0; it < 12 && hi > 4.0 * lo; ++it) {
    const double lr = log(hi / lo);
    const double x = lo * exp(lr * (double)(lane + 1) / 33.0);
    const bool pred = count_less(d, e, k, x, pivmin) >= need;
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    const int first = mask ? __ffs(mask) - 1 : 32;
    const double nlo = first == 0 ? lo : lo * exp(lr * (double)first / 33.0);
    const double nhi = first == 32 ? hi : lo * exp(lr * (double)(first + 1) / 33.0);
    lo = __shfl_sync(0xffffffffu, nlo, 0);
    hi = __shfl_sync(0xffffffffu, nhi, 0);
  }
  for (int it = 0; it < 40; ++it) {
    if (!(hi - lo > rel * hi)) break;
    const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
    const bool pred = count_less(d, e, k, x, pivmin) >= need;
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    const int first = mask ? __ffs(mask) - 1 : 32;
    const double nlo = first == 0 ? lo : lo + (hi - lo) * (double)first / 33.0;
    const double nhi = first == 32 ? hi : lo + (hi - lo) * (double)(first + 1) / 33.0;
    lo = __shfl_sync(0xffffffffu, nlo, 0);
    hi = __shfl_sync(0xffffffffu, nhi, 0);
  }
  return 0.5 * (lo + hi);
}

__device__ double tgk_bounds(const double* d, const double* e, int64_t k, double* pivmin) {
  double ub = 0.0, amax2 = 0.0;
  double prev = 0.0;
  for (int64_t t = 1; t < 2 * k; ++t) {
    const double a = fabs((t & 1) ? d[(t - 1) >> 1] : e[(t - 2) >> 1]);
    ub = fmax(ub, prev + a);
    prev = a;
    amax2 = fmax(amax2, a * a);
  }
  ub = fmax(ub, prev);
  *pivmin = 1e-290 * fmax(1.0, amax2);
  return ub * (1.0 + 1e-14) + 1e-300;
}

// ---- block-wide Sturm-count multisection -------------------------------------------------
// count on the squared TGK off-diagonals tg[u] = a_u², u = 0..2k-2 (a = d0, e0, d1, e1, ...):
// the same recurrence and rounding as count_less above.
__device__ __forceinline__ int64_t count_less_sq(const double* __restrict__ tg, int64_t k, double x,
                                                 double pivmin) {
  double q = -x;
  int64_t neg = q < 0.0;
  const int64_t n2 = 2 * k - 1;
  for (int64_t u = 0; u < n2; ++u) {
    if (fabs(q) < pivmin) q = -pivmin;
    q = -x - tg[u] / q;
    neg += q < 0.0;
  }
  return neg - k;
}

__device__ __forceinline__ void group_bar(int id, int nthreads) {
  if (id == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// j-th largest singular value by (32·nw)-way multisection shared by the nw warps of a group
// (warp gw of the group, named barrier bar_id; bar_id < 0: single warp, no barrier).  Every
// thread of the group ends with the same bracket (identical masks and arithmetic).
__device__ double kth_group(const double* tg, int64_t k, int64_t j, double lo, double hi,
                            double pivmin, double rel, int gw, int nw, unsigned* masks, int bar_id) {
  const int lane = threadIdx.x & 31;
  const int npts = 32 * nw;
  const double inv = 1.0 / (double)(npts + 1);
  const int64_t need = k - j + 1;
  int par = 0;
  auto first_true = [&](bool pred) {
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    if (nw == 1) return m ? __ffs(m) - 1 : 32;
    if (lane == 0) masks[par * nw + gw] = m;
    group_bar(bar_id, 32 * nw);
    int f = npts;
    for (int w = 0; w < nw; ++w) {
      const unsigned mm = masks[par * nw + w];
      if (mm) { f = 32 * w + __ffs(mm) - 1; break; }
    }
    par ^= 1;
    return f;
  };
  if (!(lo > 0.0)) lo = hi * 1e-300;
  for (int it = 0; it < 12 && hi > 4.0 * lo; ++it) {
    const double lr = log(hi / lo);
    const int idx = 32 * gw + lane;
    const double x = lo * exp(lr * (double)(idx + 1) * inv);
    const int f = first_true(count_less_sq(tg, k, x, pivmin) >= need);
    const double nlo = f == 0 ? lo : lo * exp(lr * (double)f * inv);
    const double nhi = f == npts ? hi : lo * exp(lr * (double)(f + 1) * inv);
    lo = nlo; hi = nhi;
  }
  for (int it = 0; it < 40; ++it) {
    if (!(hi - lo > rel * hi)) break;
    const int idx = 32 * gw + lane;
    const double w = hi - lo;
    const double x = lo + w * (double)(idx + 1) * inv;
    const int f = first_true(count_less_sq(tg, k, x, pivmin) >= need);
    const double nlo = f == 0 ? lo : lo + w * (double)f * inv;
    const double nhi = f == npts ? hi : lo + w * (double)(f + 1) * inv;
    lo = nlo; hi = nhi;
  }
  return 0.5 * (lo + hi);
}

// σ₁ and, per query, rank_lo / rank_hi counts and σ_p, σ_{p+1} — all 16 warps of the block:
// σ₁ by a 512-point multisection from the bracket [max |entry|, Gershgorin bound] (no geometric
// phase), then 2·nq bisections with 16/(2·nq) warps each.  The squared off-diagonals live in
// shared memory when they fit (tg_smem), else in the global scratch tg_glob.
__global__ void __launch_bounds__(512) sigma_queries_kernel(const double* __restrict__ d,
                                                            const double* __restrict__ e, int64_t k,
                                                            const SigmaQuery* __restrict__ q, int nq,
                                                            SigmaAnswer* __restrict__ out,
                                                            double* __restrict__ tg_glob, int tg_smem) {
  extern __shared__ double tgs[];
  __shared__ unsigned masks[2 * 16];
  __shared__ unsigned gmasks[8][2 * 8];
  __shared__ double redmax[2][16];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* tg = tg_smem ? tgs : tg_glob;
  const int64_t n2 = 2 * k - 1;
  double amax = 0.0, ub = 0.0;
  for (int64_t u = tid; u < n2; u += blockDim.x) {
    const double a = fabs((u & 1) ? e[(u - 1) >> 1] : d[u >> 1]);
    tg[u] = a * a;
    const double an = u + 1 < n2 ? fabs(((u + 1) & 1) ? e[u >> 1] : d[(u + 1) >> 1]) : 0.0;
    amax = fmax(amax, a);
    ub = fmax(ub, a + an);
    if (u == 0) ub = fmax(ub, a);
  }
  for (int o = 16; o > 0; o >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    ub = fmax(ub, __shfl_xor_sync(0xffffffffu, ub, o));
  }
  if (lane == 0) { redmax[0][warp] = amax; redmax[1][warp] = ub; }
  __syncthreads();
  amax = 0.0; ub = 0.0;
  for (int w = 0; w < 16; ++w) { amax = fmax(amax, redmax[0][w]); ub = fmax(ub, redmax[1][w]); }
  const double pivmin = 1e-290 * fmax(1.0, amax * amax);
  ub = ub * (1.0 + 1e-14) + 1e-300;
  if (k <= 0) {
    if (tid < nq) { out[tid].sigma1 = 0.0; out[tid].sigma_p = 0.0; out[tid].sigma_p1 = 0.0; out[tid].rank_lo = 0; out[tid].rank_hi = 0; }
    return;
  }
  // σ₁: the largest entry is a lower bound, the Gershgorin bound an upper one
  const double s1 = kth_group(tg, k, 1, amax * (1.0 - 1e-15), ub, pivmin, 4e-16, warp, 16, masks, 0);
  // queries: 2·nq tasks, W warps each
  const int ntask = 2 * nq;
  int W = 16 / ntask;
  W = W >= 8 ? 8 : (W >= 4 ? 4 : (W >= 2 ? 2 : 1));
  const int task = warp / W, gw = warp % W;
  if (task >= ntask) return;
  const int qi = task >> 1, half = task & 1;
  const double thr = q[qi].tol * s1;
  const double xp = nextafter(thr, 1e308);
  const int64_t p = k - count_less_sq(tg, k, xp, pivmin);
  const int bar_id = W > 1 ? 1 + task : -1;
  if (half == 0) {
    const double thr2 = thr * thr - q[qi].delta * q[qi].delta;
    const double thr_hi = thr2 > 0.0 ? sqrt(thr2) : 0.0;
    const int64_t phi = thr_hi > 0.0 ? k - count_less_sq(tg, k, nextafter(thr_hi, 1e308), pivmin) : k;
    double sp = 0.0;
    if (!q[qi].counts_only && p >= 1) sp = kth_group(tg, k, p, thr, ub, pivmin, 1e-13, gw, W, gmasks[task], bar_id);
    if (gw == 0 && lane == 0) {
      out[qi].sigma1 = s1;
      out[qi].sigma_p = sp;
      out[qi].rank_lo = (int)p;
      out[qi].rank_hi = (int)phi;
    }
  } else {
    double sp1 = 0.0;
    if (!q[qi].counts_only && p + 1 <= k) sp1 = kth_group(tg, k, p + 1, 0.0, xp, pivmin, 1e-13, gw, W, gmasks[task], bar_id);
    if (gw == 0 && lane == 0) out[qi].sigma_p1 = sp1;
  }
}

// All singular values (descending), one warp per value — test/diagnostic path.
__global__ void sigma_all_kernel(const double* __restrict__ d, const double* __restrict__ e,
                                 int64_t k, double sigma_max, double* __restrict__ out) {
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  if (wid >= k) return;
  double pivmin = 1e-290;
  const double ub = sigma_max * (1.0 + 1e-12) + 1e-300;
  out[wid] = kth_largest(d, e, k, wid + 1, 0.0, ub, pivmin);
}

}  // namespace hb

// ================================================================================================
// Two-stage bidiagonalisation (certification of large k).
// Stage 1 (host-driven, rank.cu): dense k x k -> upper band of bandwidth nb by alternating block
// QR (column panel, from the left) and block LQ (row panel, from the right), all trailing updates
// as DMMA GEMMs.  Stage 2 (bulge_chase_kernel): band -> upper bidiagonal by Householder bulge
// chasing (one sweep per row; tasks R/L alternate, each annihilating one row/column segment of
// length <= nb and pushing the bulge nb further down).  The algorithm and the inter-sweep lag
// (sweep s task t may start once sweep s-1 finished task t+3) were pinned with the numpy
// prototype tools/proto_bulge.py.  Band storage: row-major, offsets -nb..2nb around the
// diagonal (W = 3nb + 1 per row); all nonzeros stay within offsets [-(nb-1), 2nb-1].
// ================================================================================================
namespace hb {

__global__ void transpose_kernel(const double* __restrict__ src, int64_t lds, int64_t rows,
                                 int64_t cols, double* __restrict__ dst, int64_t ldd) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t c = c0 + y, r = r0 + threadIdx.x;
    tile[y][threadIdx.x] = (r < rows && c < cols) ? src[r + c * lds] : 0.0;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + y, c = c0 + threadIdx.x;  // dst(c, r) = src(r, c)
    if (r < rows && c < cols) dst[c + r * ldd] = tile[threadIdx.x][y];
  }
}

// M[i + r, j0 + c] = R[c, r] for c <= r (r < b, c < nc): the LQ factor L = R_Pᵀ of a row panel.
__global__ void write_lower_from_R(const double* __restrict__ R, int64_t ldr, int b, int nc,
                                   double* __restrict__ M, int64_t ldm) {
  const int r = threadIdx.x, c = blockIdx.x;
  if (r < b && c < nc && c <= r) M[r + (int64_t)c * ldm] = R[c + (int64_t)r * ldr];
}

// Band (offsets 0..nb of the upper-band matrix M) -> compact storage Bd (offsets -nb..2nb, zeroed
// elsewhere).
__global__ void band_extract_kernel(const double* __restrict__ M, int64_t ldm, int64_t k, int nb,
                                    double* __restrict__ Bd) {
  const int W = 3 * nb + 1;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= k * W) return;
  const int64_t r = idx / W;
  const int o = (int)(idx % W) - nb;
  const int64_t c = r + o;
  Bd[idx] = (o >= 0 && o <= nb && c < k) ? M[r + c * ldm] : 0.0;
}

__global__ void band_bidiag_out(const double* __restrict__ Bd, int64_t k, int nb,
                                double* __restrict__ d, double* __restrict__ e) {
  const int W = 3 * nb + 1;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= k) return;
  d[i] = Bd[i * W + nb];
  e[i] = i + 1 < k ? Bd[i * W + nb + 1] : 0.0;
}

struct ChaseTask {
  bool right;   // R: reflector over columns, applied to rows; L: over rows, applied to columns
  int64_t idx;  // row (R) / column (L) whose segment is annihilated
  int64_t lo, hi;    // reflector span (columns for R, rows for L)
  int64_t alo, ahi;  // application range (rows for R, columns for L)
};

// t-th task of sweep s (tools/proto_bulge.py tasks_of_sweep); returns false past the end.
__device__ bool chase_task(int64_t s, int t, int64_t k, int nb, ChaseTask* tk) {
  const int q = t >> 1;
  const int64_t c0 = s + 1 + (int64_t)q * nb;
  if (c0 > k - 1) return false;
  const int64_t c1 = min(c0 + nb - 1, k - 1);
  if ((t & 1) == 0) {
    if (!(c1 > c0 || q == 0)) return false;
    tk->right = true;
    tk->idx = q == 0 ? s : s + 1 + (int64_t)(q - 1) * nb;
    tk->lo = c0; tk->hi = c1;
    tk->alo = tk->idx; tk->ahi = min(min(k - 1, c1 + nb - 1), tk->idx + 2 * (int64_t)nb - 1);
    return true;
  }
  if (!(c1 > c0)) return false;
  tk->right = false;
  tk->idx = c0;
  tk->lo = c0; tk->hi = c1;
  tk->alo = c0; tk->ahi = min(k - 1, c1 + nb);
  return true;
}

__device__ int chase_ntasks(int64_t s, int64_t k, int nb) {
  int t = 0;
  ChaseTask tk;
  while (chase_task(s, t, k, nb, &tk)) ++t;
  return t;
}

__device__ __forceinline__ int64_t band_off(int64_t r, int64_t c, int nb, int W) {
  return r * W + (c - r + nb);
}
__device__ __forceinline__ bool band_in(int64_t r, int64_t c, int nb) {
  const int64_t o = c - r;
  return o >= -nb && o <= 2 * nb;
}

// One CTA (8 warps) per sweep slot; reflectors up to 64 long (nb <= 64).
__global__ void __launch_bounds__(256) bulge_chase_kernel(double* __restrict__ Bd, int64_t k, int nb,
                                                          int* __restrict__ prog) {
  const int W = 3 * nb + 1;
  const int G = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = 8;
  __shared__ double v[64];
  __shared__ double wpart[2][128];
  __shared__ double sh[4];
  for (int64_t s = blockIdx.x; s < k - 1; s += G) {
    const int prev_n = s > 0 ? chase_ntasks(s - 1, k, nb) : 0;
    ChaseTask tk;
    int t = 0;
    for (; chase_task(s, t, k, nb, &tk); ++t) {
      if (s > 0) {
        // thread 0 acquires the previous sweep's progress; the CTA barrier then orders every
        // thread's (L2, __ldcg) loads after it — no per-thread fence (a MEMBAR.SC.GPU in all 256
        // threads was 84 % of the kernel's stall samples)
        const int need = min(t + 4, prev_n);
        if (tid == 0)
          while ((int)ld_acquire_gpu(reinterpret_cast<const unsigned int*>(prog + s - 1)) < need) __nanosleep(32);
        __syncthreads();
      }
      const int len = (int)(tk.hi - tk.lo + 1);
      // The reflector's segment is the first row (R task: row idx = alo) / first column (L task:
      // column idx = alo) of the block the task updates, so one L2 round trip loads both: the
      // block goes to registers, the segment is taken from them (R) or staged in shared memory (L).
      auto reflector = [&](double x0, double x1) {  // warp 0: x0 / x1 = elements lane / lane + 32
        const double alpha = __shfl_sync(0xffffffffu, x0, 0);
        double ss = (lane > 0 ? x0 * x0 : 0.0) + x1 * x1;
        ss = warp_sum(ss);
        double tau = 0.0, scal = 0.0, beta = alpha;
        if (ss > 0.0) {
          beta = -copysign(sqrt(alpha * alpha + ss), alpha);
          tau = (beta - alpha) / beta;
          scal = 1.0 / (alpha - beta);
        }
        v[lane] = lane == 0 ? 1.0 : (lane < len ? x0 * scal : 0.0);
        v[lane + 32] = lane + 32 < len ? x1 * scal : 0.0;
        if (lane == 0) { sh[0] = tau; sh[1] = beta; }
      };
      if (tk.right) {
        // rows r in [alo, ahi] (<= 127): s_r = sum_c M[r, lo + c] v_c; M[r, .] -= tau s_r v.
        // A warp owns up to 16 rows; all loads are issued before the reductions.
        constexpr int RMAX = 16;
        double m0[RMAX], m1[RMAX], sr[RMAX];
#pragma unroll
        for (int j = 0; j < RMAX; ++j) {
          const int64_t r = tk.alo + warp + (int64_t)j * NW;
          const int64_t c0 = tk.lo + lane, c1 = c0 + 32;
          const bool ok0 = r <= tk.ahi && lane < len && band_in(r, c0, nb);
          const bool ok1 = r <= tk.ahi && lane + 32 < len && band_in(r, c1, nb);
          m0[j] = ok0 ? __ldcg(Bd + band_off(r, c0, nb, W)) : 0.0;
          m1[j] = ok1 ? __ldcg(Bd + band_off(r, c1, nb, W)) : 0.0;
        }
        if (warp == 0) reflector(m0[0], m1[0]);  // row alo == idx: the segment
        __syncthreads();
        const double tau = sh[0];
        if (tau != 0.0) {
          const double v0 = v[lane], v1 = v[lane + 32];
#pragma unroll
          for (int j = 0; j < RMAX; ++j) sr[j] = m0[j] * v0 + m1[j] * v1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int j = 0; j < RMAX; ++j) sr[j] += __shfl_xor_sync(0xffffffffu, sr[j], o);
#pragma unroll
          for (int j = 0; j < RMAX; ++j) {
            const int64_t r = tk.alo + warp + (int64_t)j * NW;
            const int64_t c0 = tk.lo + lane, c1 = c0 + 32;
            if (r <= tk.ahi && lane < len && band_in(r, c0, nb))
              __stcg(Bd + band_off(r, c0, nb, W), m0[j] - tau * sr[j] * v0);
            if (r <= tk.ahi && lane + 32 < len && band_in(r, c1, nb))
              __stcg(Bd + band_off(r, c1, nb, W), m1[j] - tau * sr[j] * v1);
          }
        }
      } else {
        // columns c in [alo, ahi] (<= 128): thread (cc, half) holds 32 rows of column cc;
        // w_c = sum_r v_r M[lo + r, c] combined over the two halves; M[., c] -= tau v w_c.
        const int ncols = (int)(tk.ahi - tk.alo + 1);
        const int cc = tid & 127, half = tid >> 7;
        const int64_t c = tk.alo + cc;
        double x[32];
        if (cc < ncols) {
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            const int rr = half * 32 + r;
            const bool ok = rr < len && band_in(tk.lo + rr, c, nb);
            x[r] = ok ? __ldcg(Bd + band_off(tk.lo + rr, c, nb, W)) : 0.0;
          }
        }
        if (cc == 0) {  // column alo == idx: the segment
#pragma unroll
          for (int r = 0; r < 32; ++r) wpart[0][half * 32 + r] = x[r];
        }
        __syncthreads();
        if (warp == 0) reflector(wpart[0][lane], wpart[0][lane + 32]);
        __syncthreads();
        const double tau = sh[0];
        if (tau != 0.0) {
          double w = 0.0;
          if (cc < ncols) {
#pragma unroll
            for (int r = 0; r < 32; ++r) w += v[half * 32 + r] * x[r];
          }
          __syncthreads();  // wpart[0] held the segment
          if (cc < ncols) wpart[half][cc] = w;
          __syncthreads();
          if (cc < ncols) {
            w = (wpart[0][cc] + wpart[1][cc]) * tau;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
              const int rr = half * 32 + r;
              if (rr < len && band_in(tk.lo + rr, c, nb))
                __stcg(Bd + band_off(tk.lo + rr, c, nb, W), x[r] - v[rr] * w);
            }
          }
        }
      }
      __syncthreads();
      // exact zeros / beta on the annihilated segment
      if (warp == 0) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int el = lane + 32 * h;
          if (el < len) {
            const int64_t r = tk.right ? tk.idx : tk.lo + el;
            const int64_t c = tk.right ? tk.lo + el : tk.idx;
            __stcg(Bd + band_off(r, c, nb, W), el == 0 ? sh[1] : 0.0);
          }
        }
      }
      __syncthreads();  // every thread's (L2, __stcg) stores of this task precede the release
      if (tid == 0) st_release_gpu(reinterpret_cast<unsigned int*>(prog + s), (unsigned int)(t + 1));
    }
    if (tid == 0)  // sweep finished (>= any need)
      st_release_gpu(reinterpret_cast<unsigned int*>(prog + s), (unsigned int)(t + 1000000));
  }
}

}  // namespace hb

namespace hb {
// Small certification (k <= kSmallBidiag): one CTA holds the whole k x k triangle in shared
// memory and runs the one-stage Golub–Kahan bidiagonalisation there (no grid barriers, one
// launch).  Column-major with odd leading dimension k+1 so column sweeps (w = uᵀM) and row sweeps
// (z = M v) are both bank-conflict free.
__global__ void __launch_bounds__(kSmallBidiagThreads) bidiag_small_kernel(const double* __restrict__ Mk,
                                                                         int64_t ldm, int k,
                                                                         double* __restrict__ d,
                                                                         double* __restrict__ e) {
  constexpr int NT = kSmallBidiagThreads, NW = NT / 32, NG = NT / 4;
  extern __shared__ double S[];  // [k][k+1] + u[k] + v[k] + w[k]
  const int ld = k + 1;
  double* u = S + (size_t)k * ld;
  double* vv = u + k;
  double* w = vv + k;
  __shared__ double sh[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = lane & 3, grp = tid >> 2;  // 4 lanes per dot product
  for (int idx = tid; idx < k * k; idx += NT) {
    const int r = idx % k, c = idx / k;
    S[c * ld + r] = Mk[r + (int64_t)c * ldm];
  }
  __syncthreads();
  for (int i = 0; i < k; ++i) {
    // ---- left reflector from column i (rows i..k-1) ----
    if (warp == 0) {
      double s = 0.0;
      for (int r = i + 1 + lane; r < k; r += 32) s += S[i * ld + r] * S[i * ld + r];
      s = warp_sum(s);
      const double alpha = S[i * ld + i];
      double tau = 0.0, scal = 0.0, beta = alpha;
      if (s > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + s), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      for (int r = i + 1 + lane; r < k; r += 32) u[r] = S[i * ld + r] * scal;
      if (lane == 0) { u[i] = 1.0; sh[0] = tau; d[i] = beta; }
    }
    __syncthreads();
    const double tu = sh[0];
    // w[q] = tu · Σ_{r >= i} u[r] S[r, q]  (q > i), four lanes per column, fixed order
    for (int q0 = i + 1; q0 < k; q0 += NG) {
      const int q = q0 + grp;
      double s = 0.0;
      if (q < k)
        for (int r = i + sub; r < k; r += 4) s += u[r] * S[q * ld + r];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (q < k && sub == 0) w[q] = s * tu;
    }
    __syncthreads();
    for (int q = i + 1 + warp; q < k; q += NW) {
      const double wq = w[q];
      double* Sq = S + q * ld;
      for (int r = i + lane; r < k; r += 32) Sq[r] -= u[r] * wq;
    }
    __syncthreads();
    if (i + 1 >= k) break;
    // ---- right reflector from row i (columns i+1..k-1) ----
    if (warp == 0) {
      double s = 0.0;
      for (int q = i + 2 + lane; q < k; q += 32) s += S[q * ld + i] * S[q * ld + i];
      s = warp_sum(s);
      const double alpha = S[(i + 1) * ld + i];
      double tau = 0.0, scal = 0.0, beta = alpha;
      if (s > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + s), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      for (int q = i + 2 + lane; q < k; q += 32) vv[q] = S[q * ld + i] * scal;
      if (lane == 0) { vv[i + 1] = 1.0; sh[1] = tau; e[i] = beta; }
    }
    __syncthreads();
    const double tv = sh[1];
    // w[r] = tv · Σ_{q > i} S[r, q] vv[q]  (r > i), four lanes per row, fixed order
    for (int r0 = i + 1; r0 < k; r0 += NG) {
      const int r = r0 + grp;
      double s = 0.0;
      if (r < k)
        for (int q = i + 1 + sub; q < k; q += 4) s += S[q * ld + r] * vv[q];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (r < k && sub == 0) w[r] = s * tv;
    }
    __syncthreads();
    for (int q = i + 1 + warp; q < k; q += NW) {
      const double vq = vv[q];
      double* Sq = S + q * ld;
      for (int r = i + 1 + lane; r < k; r += 32) Sq[r] -= w[r] * vq;
    }
    __syncthreads();
  }
  if (tid == 0) e[k - 1] = 0.0;
}
}  // namespace hb
