// Adaptive cross approximation on the device: hodlr::BlockSpec / aca_sweep / compress / apply
// (/root/reference/proj/include/hodlr/aca.hpp:16-213), the reference's own rank(ε) factorisation.
//
// One sweep is inherently sequential in its pivots, so a block is owned by a group of G CTAs
// (G = 1 for small blocks, which then run many per launch: gridDim.y = blocks) that keep the
// same control state redundantly and meet at two group barriers per pivot:
//   phase A  residual row  row(j) = K(next_row, j) − Σ_k u_k(next_row) v_k(j)    (aca.hpp:85-86)
//            [+ the cross-term partials of the previous pivot's stopping test]
//            column argmax over unused columns (first maximum)                      (aca.hpp:87-96)
//   -- barrier B1 --  stopping test of the previous pivot (aca.hpp:120-130), pivot column
//   phase B  v = row / pivot, u = K(:, piv) − Σ_k v_k(piv) u_k                      (aca.hpp:108-111)
//            partial ||u||², ||v||², u_kᵀu, v_kᵀv (k < r); row argmax over unused rows (aca.hpp:136-147)
//   -- barrier B2 --  next row
// Entries are recomputed on the fly (BlockSpec::entry, aca.hpp:30-33) with the k2 entry rule, so
// the u / v updates are bit-identical to the CPU restatement whenever the entries are (always for
// 1/r; log / exp are libdevice, <= 2 ulp).  Reductions (norms, dots) use a fixed per-CTA order:
// deterministic, but not Eigen's order, so ||u||·||v|| vs ε||A_r||_F can differ in the last bits.
// Layout: u_k / v_k are the columns of U (rows x cap) and V (cols x cap), column-major, so every
// residual update streams one coalesced column per k.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "context.h"
#include "entries.cuh"


namespace hb {

namespace {

constexpr int kAcaThreads = 512;
constexpr int kAcaWarps = kAcaThreads / 32;
constexpr int kAcaChunk = 1024;      // coefficients staged in shared memory per pass
constexpr int64_t kAcaMaxSlice = 4096;  // rows / columns one CTA owns (shared memory)

struct AcaState {
  int64_t rank, next_row, rows_left;
  double fro2;
  int32_t met, done, grow;
  uint32_t bad;
};

struct AcaBlockDev {
  const double* x;
  const double* y;
  int64_t nt, ns;
  int64_t rb, rows, cb, cols;
  int64_t lim, cap;
  double* U;  // rows x cap
  double* V;  // cols x cap
  double* piv;
  int64_t* sig;  // block-local row pivots
  int64_t* tau;  // block-local column pivots
  unsigned char* used_row;
  unsigned char* used_col;
  double* rowbuf;  // cols
  double* part;    // partial area, see PartLayout
  AcaState* st;
  unsigned int* bar;  // {count, .., gen at +32}
};

struct AcaParams {
  AcaBlockDev* blocks;
  DevKernel K;
  int d;
  double eps;
};

// Partial area of one block: argA[2][G] (double-buffered by barrier parity), argC[G], nrm[G] (nu²,
// nv²), crossp[G], then pu[G][cap], pv[G][cap].  (value, index) pairs are stored as 2 doubles.
struct PartLayout {
  double* argA;
  double* argC;
  double* nrm;
  double* crossp;
  double* pu;
  double* pv;
  __host__ __device__ PartLayout(double* base, int G, int64_t cap) {
    argA = base;
    argC = argA + 4 * G;
    nrm = argC + 2 * G;
    crossp = nrm + 2 * G;
    pu = crossp + G;
    pv = pu + (int64_t)G * cap;
  }
  __host__ __device__ static int64_t elems(int G, int64_t cap) { return 9ll * G + 2ll * G * cap; }
};

// Barrier over the G CTAs of one group (blockIdx.x), same protocol as GridSync.
struct GroupSync {
  unsigned int* count;
  unsigned int* gen;
  unsigned int g = 0;
  int G;
  __device__ __forceinline__ GroupSync(unsigned int* bar, int G_) : count(bar), gen(bar + 32), G(G_) {
    if (G > 1 && threadIdx.x == 0) g = ld_acquire_gpu(gen);
  }
  __device__ __forceinline__ void sync() {
    __syncthreads();
    if (G == 1) return;
    if (threadIdx.x == 0) {
      if (atom_add_acq_rel_gpu(count, 1u) == (unsigned)G - 1) {
        *count = 0;
        st_release_gpu(gen, g + 1);
      } else {
        unsigned int spins = 0;
        while (ld_acquire_gpu(gen) == g) {
          if (++spins == (1u << 28)) {
            printf("[hb aca barrier] block %d of %d stuck\n", blockIdx.x, G);
            __trap();
          }
        }
      }
      ++g;
    }
    __syncthreads();
  }
};

// (value, index) maximum with ties to the smaller index: the first maximum of a left-to-right
// scan with strict '>' (aca.hpp:91-95, 142-146).  NaN never wins (comparisons are false).
__device__ __forceinline__ void amax_merge(double& v, int64_t& i, double v2, int64_t i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

__device__ void block_amax(double& v, int64_t& i, double* sv, int64_t* si) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t i2 = __shfl_xor_sync(0xffffffffu, i, o);
    amax_merge(v, i, v2, i2);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    sv[w] = v;
    si[w] = i;
  }
  __syncthreads();
  v = sv[0];
  i = si[0];
  for (int q = 1; q < kAcaWarps; ++q) amax_merge(v, i, sv[q], si[q]);
}

// Σ_k over a deterministic order; result in every thread.
__device__ double block_sum_d(double v, double* s) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) s[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int q = 0; q < kAcaWarps; ++q) t += s[q];
  return t;
}

// dot partials: out[k] = Σ_{t < n} M[t + k*ld] * vec[t] for k < r (warp per k, lanes over t)
__device__ void dots_warp(const double* __restrict__ M, int64_t ld, const double* vec, int64_t n,
                          int64_t r, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t k = w; k < r; k += kAcaWarps) {
    const double* col = M + k * ld;
    double a = 0.0;
    for (int64_t t = lane; t < n; t += 32) a = fma(col[t], vec[t], a);
    a = warp_sum(a);
    if (lane == 0) out[k] = a;
  }
}

// a − Σ_k coef[k]·col[k*ld] for k < kn, subtracting in k order with every product and difference
// rounded separately (aca.hpp:86 / :111 `row -= us[k](i) * vs[k]`); the loads of a batch of 24
// (8 for one-CTA batched blocks, where the wider batch spills and slowed 512 x 256² by 1.9x) are issued together so the chain waits on one L2 latency per batch, not per term (the sweep
// is bound by these chains: ncu of a 4000 x 4000 sweep showed 45 % long-scoreboard stalls).
template <bool WIDE>
__device__ __forceinline__ double residual_chain(double a, const double* coef, const double* col,
                                                 int64_t ld, int64_t kn) {
  int64_t k = 0;
  if (WIDE)
  for (; k + 24 <= kn; k += 24) {
    double v[24];
#pragma unroll
    for (int q = 0; q < 24; ++q) v[q] = __ldcg(col + (k + q) * ld);
#pragma unroll
    for (int q = 0; q < 24; ++q) a = __dsub_rn(a, __dmul_rn(coef[k + q], v[q]));
  }
  for (; k + 8 <= kn; k += 8) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __ldcg(col + (k + q) * ld);
#pragma unroll
    for (int q = 0; q < 8; ++q) a = __dsub_rn(a, __dmul_rn(coef[k + q], v[q]));
  }
  for (; k < kn; ++k) a = __dsub_rn(a, __dmul_rn(coef[k], __ldcg(col + k * ld)));
  return a;
}

template <bool WIDE>
__global__ void __launch_bounds__(kAcaThreads) aca_sweep_kernel(AcaParams p) {
  extern __shared__ double smem[];
  __shared__ double s_red[kAcaWarps];
  __shared__ int64_t s_ired[kAcaWarps];
  __shared__ int64_t s_scan;
  const AcaBlockDev B = p.blocks[blockIdx.y];
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
  const int64_t m = B.rows, n = B.cols;
  const int64_t cs = ceil_div(n, G), rs = ceil_div(m, G);
  const int64_t c0 = min((int64_t)c * cs, n), nc = min(c0 + cs, n) - c0;
  const int64_t r0 = min((int64_t)c * rs, m), nrw = min(r0 + rs, m) - r0;
  double* sv = smem;           // row / v over my columns
  double* su = sv + cs;        // u over my rows
  double* coef = su + rs;      // staged coefficients
  PartLayout P(B.part, G, B.cap);
  const double* X = B.x;
  const double* Y = B.y;
  const int64_t xrow0 = B.rb, ycol0 = B.cb;

  GroupSync gs(B.bar, G);
  int64_t r = B.st->rank, nrow = B.st->next_row, rows_left = B.st->rows_left;
  double fro2 = B.st->fro2;
  int met = 0, done = 0;
  unsigned int bad = 0;
  bool pending = false;
  int it = 0;
  double pend_nu2 = 0.0, pend_nv2 = 0.0;

  while (true) {
    // ---- cross-term partial of the pending stopping test: k < r - 1 (the dots of pivot r-1)
    if (pending) {
      double nu2 = 0.0, nv2 = 0.0;
      for (int q = 0; q < G; ++q) {
        nu2 += __ldcg(P.nrm + 2 * q);
        nv2 += __ldcg(P.nrm + 2 * q + 1);
      }
      pend_nu2 = nu2;
      pend_nv2 = nv2;
      const int64_t kk = r - 1, per = ceil_div(kk, G);
      const int64_t k0 = min((int64_t)c * per, kk), k1 = min(k0 + per, kk);
      double acc = 0.0;
      for (int64_t k = k0 + tid; k < k1; k += kAcaThreads) {
        double su_k = 0.0, sv_k = 0.0;
        for (int q = 0; q < G; ++q) {
          su_k += __ldcg(P.pu + (int64_t)q * B.cap + k);
          sv_k += __ldcg(P.pv + (int64_t)q * B.cap + k);
        }
        acc += su_k * sv_k;
      }
      acc = block_sum_d(acc, s_red);
      if (tid == 0) P.crossp[c] = acc;
    }
    const bool spec = (r < B.lim) && (r < B.cap);
    if (spec) {
      // ---- phase A: residual row nrow over my columns
      for (int64_t t = tid; t < nc; t += kAcaThreads)
        sv[t] = entry_soa(p.K, X, B.nt, xrow0 + nrow, Y, B.ns, ycol0 + c0 + t, p.d, &bad);
      for (int64_t k0 = 0; k0 < r; k0 += kAcaChunk) {
        const int64_t kn = (r - k0 < kAcaChunk) ? r - k0 : (int64_t)kAcaChunk;
        __syncthreads();
        for (int64_t t = tid; t < kn; t += kAcaThreads) coef[t] = __ldcg(B.U + nrow + (k0 + t) * m);
        __syncthreads();
        for (int64_t t = tid; t < nc; t += kAcaThreads)
          sv[t] = residual_chain<WIDE>(sv[t], coef, B.V + c0 + t + k0 * n, n, kn);
      }
      double bv = -1.0;
      int64_t bi = INT64_MAX;
      for (int64_t t = tid; t < nc; t += kAcaThreads) {
        B.rowbuf[c0 + t] = sv[t];
        if (!__ldcg(B.used_col + c0 + t)) amax_merge(bv, bi, fabs(sv[t]), c0 + t);
      }
      block_amax(bv, bi, s_red, s_ired);
      if (tid == 0) {
        P.argA[4 * c + 2 * (it & 1)] = bv;
        P.argA[4 * c + 2 * (it & 1) + 1] = (double)bi;
      }
    }
    gs.sync();  // B1
    if (pending) {
      double cross = 0.0;
      for (int q = 0; q < G; ++q) cross += __ldcg(P.crossp + q);
      const double nu = sqrt(pend_nu2), nv = sqrt(pend_nv2);
      fro2 += 2.0 * cross + nu * nu * nv * nv;  // aca.hpp:123
      pending = false;
      if (nu * nv <= p.eps * sqrt(fmax(fro2, 0.0))) {  // aca.hpp:127-130
        met = 1;
        done = 1;
        break;
      }
    }
    if (!spec) break;
    double pvv = -1.0;
    int64_t pc = INT64_MAX;
    for (int q = 0; q < G; ++q)
      amax_merge(pvv, pc, __ldcg(P.argA + 4 * q + 2 * (it & 1)),
                 (int64_t)__ldcg(P.argA + 4 * q + 2 * (it & 1) + 1));
    ++it;
    if (!(pvv > 0.0)) {  // zero residual row (aca.hpp:97-107)
      if (tid == 0) B.used_row[nrow] = 1;
      if (--rows_left == 0) {
        met = 1;
        done = 1;
        break;
      }
      // next unused row (first index), treating nrow as used
      if (tid == 0) s_scan = INT64_MAX;
      __syncthreads();
      for (int64_t i = tid; i < m; i += kAcaThreads)
        if (i != nrow && !__ldcg(B.used_row + i)) {
          atomicMin((unsigned long long*)&s_scan, (unsigned long long)i);
          break;
        }
      __syncthreads();
      nrow = s_scan;
      __syncthreads();
      continue;
    }
    // ---- phase B
    const double pivot = __ldcg(B.rowbuf + pc);
    double nv2 = 0.0;
    for (int64_t t = tid; t < nc; t += kAcaThreads) {
      const double v = __ddiv_rn(sv[t], pivot);  // aca.hpp:109
      sv[t] = v;
      B.V[c0 + t + r * n] = v;
      nv2 += v * v;
    }
    __syncthreads();
    dots_warp(B.V + c0, n, sv, nc, r, P.pv + (int64_t)c * B.cap);
    for (int64_t t = tid; t < nrw; t += kAcaThreads)
      su[t] = entry_soa(p.K, X, B.nt, xrow0 + r0 + t, Y, B.ns, ycol0 + pc, p.d, &bad);
    for (int64_t k0 = 0; k0 < r; k0 += kAcaChunk) {
      const int64_t kn = (r - k0 < kAcaChunk) ? r - k0 : (int64_t)kAcaChunk;
      __syncthreads();
      for (int64_t t = tid; t < kn; t += kAcaThreads) coef[t] = __ldcg(B.V + pc + (k0 + t) * n);
      __syncthreads();
      for (int64_t t = tid; t < nrw; t += kAcaThreads)
        su[t] = residual_chain<WIDE>(su[t], coef, B.U + r0 + t + k0 * m, m, kn);
    }
    __syncthreads();
    double nu2 = 0.0, bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t t = tid; t < nrw; t += kAcaThreads) {
      const double u = su[t];
      B.U[r0 + t + r * m] = u;
      nu2 += u * u;
      const int64_t i = r0 + t;
      if (i != nrow && !__ldcg(B.used_row + i)) amax_merge(bv, bi, fabs(u), i);
    }
    dots_warp(B.U + r0, m, su, nrw, r, P.pu + (int64_t)c * B.cap);
    nu2 = block_sum_d(nu2, s_red);
    nv2 = block_sum_d(nv2, s_red);
    block_amax(bv, bi, s_red, s_ired);
    if (tid == 0) {
      P.nrm[2 * c] = nu2;
      P.nrm[2 * c + 1] = nv2;
      P.argC[2 * c] = bv;
      P.argC[2 * c + 1] = (double)bi;
      B.used_row[nrow] = 1;
      B.used_col[pc] = 1;
      if (c == 0) {
        B.sig[r] = nrow;
        B.tau[r] = pc;
        B.piv[r] = pivot;
      }
    }
    gs.sync();  // B2
    ++r;
    pending = true;
    if (--rows_left == 0) {
      // every row pivoted or zero (aca.hpp:131-134); the pending test would also give met
      met = 1;
      done = 1;
      break;
    }
    double nb = -1.0;
    int64_t ni = INT64_MAX;
    for (int q = 0; q < G; ++q)
      amax_merge(nb, ni, __ldcg(P.argC + 2 * q), (int64_t)__ldcg(P.argC + 2 * q + 1));
    nrow = ni;
  }
  if (bad) atomicOr(&B.st->bad, bad);
  if (c == 0 && tid == 0) {
    AcaState* S = B.st;
    S->rank = r;
    S->next_row = nrow;
    S->rows_left = rows_left;
    S->fro2 = fro2;
    if (!done && r >= B.lim) done = 1;  // loop condition (aca.hpp:83)
    S->met = met;
    S->done = done;
    S->grow = (!done && r >= B.cap) ? 1 : 0;
  }
}

// L(a,k) = u_k(σ_a) / pivot_k, U(k,b) = pivot_k v_k(τ_b)  (aca.hpp:157-160)
// L(a,k) = u_k(σ_a) / pivot_k, U(k,b) = pivot_k v_k(τ_b)  (aca.hpp:157-160), every block of a
// batch in one launch (blockIdx.y = block)
struct LuJob {
  const double* Ua;
  const double* Va;
  const int64_t* sig;
  const int64_t* tau;
  const double* piv;
  int64_t m, n, r;
  double* L;
  double* U;
};
__global__ void aca_build_lu_kernel(const LuJob* __restrict__ jobs) {
  const LuJob J = jobs[blockIdx.y];
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < J.r * J.r;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = idx % J.r, k = idx / J.r;  // L column k, row a ; U row k, column a
    J.L[a + k * J.r] = __ddiv_rn(J.Ua[J.sig[a] + k * J.m], J.piv[k]);
    J.U[k + a * J.r] = __dmul_rn(J.piv[k], J.Va[J.tau[a] + k * J.n]);
  }
}

// t_k = K(σ_k, J) · q  (aca.hpp:207); one CTA per k, fixed-order reduction
__global__ void aca_apply_rows_kernel(DevKernel K, int d, const double* x, int64_t nt,
                                      const double* y, int64_t ns, int64_t cb, int64_t cols,
                                      const int64_t* sig_global, const double* q, double* t,
                                      unsigned int* flags) {
  __shared__ double s[32];
  const int64_t k = blockIdx.x;
  unsigned int bad = 0;
  const int64_t i = sig_global[k];
  double a = 0.0;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x)
    a += entry_soa(K, x, nt, i, y, ns, cb + j, d, &bad) * q[j];
  a = block_sum(a, s);
  if (threadIdx.x == 0) t[k] = a;
  if (bad) atomicOr(flags, bad);
}

// L⁻¹ then U⁻¹ in place on t (aca.hpp:208-209), column-oriented substitution, one CTA
__global__ void aca_apply_solve_kernel(const double* __restrict__ L, const double* __restrict__ U,
                                       int64_t r, double* t) {
  for (int64_t k = 0; k < r; ++k) {
    __syncthreads();
    const double tk = t[k];
    for (int64_t i = k + 1 + threadIdx.x; i < r; i += blockDim.x)
      t[i] = __dsub_rn(t[i], __dmul_rn(L[i + k * r], tk));
  }
  for (int64_t k = r - 1; k >= 0; --k) {
    __syncthreads();
    const double tk = __ddiv_rn(t[k], U[k + k * r]);
    __syncthreads();
    if (threadIdx.x == 0) t[k] = tk;
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x)
      t[i] = __dsub_rn(t[i], __dmul_rn(U[i + k * r], tk));
  }
}

// b(i) = Σ_k t_k K(i, τ_k), k in order (aca.hpp:210-211)
__global__ void aca_apply_cols_kernel(DevKernel K, int d, const double* x, int64_t nt,
                                      const double* y, int64_t ns, int64_t rb, int64_t rows,
                                      const int64_t* tau_global, const double* t, int64_t r,
                                      double* b, unsigned int* flags) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  unsigned int bad = 0;
  double acc = 0.0;
  for (int64_t k = 0; k < r; ++k)
    acc = __dadd_rn(acc, __dmul_rn(t[k], entry_soa(K, x, nt, rb + i, y, ns, tau_global[k], d, &bad)));
  b[i] = acc;
  if (bad) atomicOr(flags, bad);
}

DevKernel dev_kernel(const hb_kernel& k) {
  DevKernel K;
  K.id = k.id;
  K.has_diag = k.has_diag != 0;
  K.diag = k.diag;
  K.singular = kernel_singular_at_origin(k.id) ? 1 : 0;
  return K;
}

// Device buffers of one block's sweep.
struct SweepBufs {
  int64_t cap = 0;
  int G = 1;
  double *U = nullptr, *V = nullptr, *piv = nullptr, *rowbuf = nullptr, *part = nullptr;
  int64_t *sig = nullptr, *tau = nullptr;
  unsigned char *used_row = nullptr, *used_col = nullptr;
  AcaState* st = nullptr;
  unsigned int* bar = nullptr;
  bool own_uvp = false;  // U, V, part individually allocated (after growth); the rest lives in
                         // the per-call arena
};

template <typename T>
T* dalloc(size_t n, cudaStream_t s) {
  void* p = nullptr;
  HB_CUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), s));
  return static_cast<T*>(p);
}
void dfree(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

void free_bufs(SweepBufs& b, cudaStream_t s) {
  if (b.own_uvp)
    for (void* p : {(void*)b.U, (void*)b.V, (void*)b.part}) dfree(p, s);
  b = SweepBufs{};
}

// One stream-ordered allocation per run_sweeps call, carved by buffer kind so the per-block
// states / pivots / flags of a whole batch move with one copy or memset each.
struct Arena {
  char* base = nullptr;
  size_t used = 0;
  template <typename T>
  T* take(size_t n) {
    T* p = reinterpret_cast<T*>(base + used);
    used += round_up((int64_t)(std::max<size_t>(n, 1) * sizeof(T)), 256);
    return p;
  }
};

}  // namespace

struct AcaBlockReq {
  hb_block blk;
  double eps;
  int64_t max_rank;
  // results
  int64_t rank = 0;
  int met = 0;
  uint32_t bad = 0;
  SweepBufs bufs;
  int64_t lim = 0;
  std::vector<double> piv_h;  // pivots (host), filled when the sweep finished
  std::vector<int64_t> sig_h, tau_h;  // block-local pivot ids (host)
};

// Run the sweeps of `reqs` (all with the same G) to completion, growing U / V on demand.  The
// buffers of all blocks come from one arena (kept alive in `arenas` until the caller is done).
static void run_sweeps(hb_context* c, const DevKernel& K, const double* x, int64_t nt, const double* y,
                       int64_t ns, int d, std::vector<AcaBlockReq*>& reqs, int G,
                       std::vector<void*>& arenas) {
  cudaStream_t st = c->stream;
  const size_t kCapBudget = (size_t)1 << 31;  // initial U+V bytes per block before growth
  const size_t nb = reqs.size();
  static const int64_t init_cap = [] {  // test hook: exercise the growth path
    const char* e = getenv("HB_ACA_INIT_CAP");
    return e ? std::max<int64_t>(1, atoll(e)) : (int64_t)0;
  }();
  int64_t sum_lim = 0, sum_m = 0, sum_n = 0, sum_mcap = 0, sum_ncap = 0, sum_part = 0;
  for (AcaBlockReq* q : reqs) {
    const int64_t m = q->blk.rows, n = q->blk.cols;
    q->lim = std::min({m, n, q->max_rank});
    SweepBufs& b = q->bufs;
    b = SweepBufs{};
    b.G = G;
    b.cap = std::min<int64_t>(q->lim, std::max<int64_t>(64, (int64_t)(kCapBudget / (8 * (m + n)))));
    if (init_cap) b.cap = std::min<int64_t>(q->lim, init_cap);
    sum_lim += round_up(q->lim, 32);
    sum_m += round_up(m, 256);
    sum_n += round_up(n, 256);
    sum_mcap += round_up(m * b.cap, 32);
    sum_ncap += round_up(n * b.cap, 32);
    sum_part += round_up(PartLayout::elems(G, b.cap), 32);
  }
  // layout by kind: [states][bars][used_row][used_col] (zeroed / uploaded together), then
  // [piv][sig][tau], [rowbuf], [part], [U], [V]
  const size_t bytes = (nb * sizeof(AcaState) + 256) + (nb * 64 * sizeof(unsigned int) + 256) +
                       (size_t)(sum_m + sum_n) + 512 + (size_t)sum_lim * 24 + 768 +
                       (size_t)(sum_n + sum_part + sum_mcap + sum_ncap) * 8 + 1024 + nb * 4 * 256;
  void* raw = nullptr;
  HB_CUDA(cudaMallocAsync(&raw, bytes, st));
  arenas.push_back(raw);
  Arena ar{static_cast<char*>(raw), 0};
  AcaState* states = ar.take<AcaState>(nb);
  unsigned int* bars = ar.take<unsigned int>(nb * 64);
  unsigned char* urow = ar.take<unsigned char>((size_t)sum_m);
  unsigned char* ucol = ar.take<unsigned char>((size_t)sum_n);
  const size_t zero_bytes = (size_t)(reinterpret_cast<char*>(ucol) - reinterpret_cast<char*>(bars)) + (size_t)sum_n;
  std::vector<AcaState> s0(nb);
  int64_t om = 0, on = 0;
  for (size_t i = 0; i < nb; ++i) {
    AcaBlockReq* q = reqs[i];
    SweepBufs& b = q->bufs;
    b.st = states + i;
    b.bar = bars + 64 * i;
    b.used_row = urow + om;
    b.used_col = ucol + on;
    om += round_up(q->blk.rows, 256);
    on += round_up(q->blk.cols, 256);
    s0[i].rank = 0;
    s0[i].next_row = 0;
    s0[i].rows_left = q->blk.rows;
    s0[i].fro2 = 0.0;
  }
  for (AcaBlockReq* q : reqs) q->bufs.piv = ar.take<double>((size_t)q->lim);
  for (AcaBlockReq* q : reqs) q->bufs.sig = ar.take<int64_t>((size_t)q->lim);
  for (AcaBlockReq* q : reqs) q->bufs.tau = ar.take<int64_t>((size_t)q->lim);
  for (AcaBlockReq* q : reqs) q->bufs.rowbuf = ar.take<double>((size_t)q->blk.cols);
  for (AcaBlockReq* q : reqs) q->bufs.part = ar.take<double>((size_t)PartLayout::elems(G, q->bufs.cap));
  for (AcaBlockReq* q : reqs) q->bufs.U = ar.take<double>((size_t)(q->blk.rows * q->bufs.cap));
  for (AcaBlockReq* q : reqs) q->bufs.V = ar.take<double>((size_t)(q->blk.cols * q->bufs.cap));
  HB_REQUIRE(ar.used <= bytes, HB_ECUDA, "aca: arena layout overflow");
  HB_CUDA(cudaMemsetAsync(bars, 0, zero_bytes, st));
  // pageable source: the call returns once the data is staged, so s0 may go out of scope
  HB_CUDA(cudaMemcpyAsync(states, s0.data(), nb * sizeof(AcaState), cudaMemcpyHostToDevice, st));
  std::vector<AcaBlockReq*> live = reqs;
  while (!live.empty()) {
    std::vector<AcaBlockDev> hb(live.size());
    int64_t cs_max = 0, rs_max = 0;
    for (size_t i = 0; i < live.size(); ++i) {
      AcaBlockReq* q = live[i];
      SweepBufs& b = q->bufs;
      AcaBlockDev& D = hb[i];
      D.x = x;
      D.y = y;
      D.nt = nt;
      D.ns = ns;
      D.rb = q->blk.row_begin;
      D.rows = q->blk.rows;
      D.cb = q->blk.col_begin;
      D.cols = q->blk.cols;
      D.lim = q->lim;
      D.cap = b.cap;
      D.U = b.U;
      D.V = b.V;
      D.piv = b.piv;
      D.sig = b.sig;
      D.tau = b.tau;
      D.used_row = b.used_row;
      D.used_col = b.used_col;
      D.rowbuf = b.rowbuf;
      D.part = b.part;
      D.st = b.st;
      D.bar = b.bar;
      cs_max = std::max(cs_max, ceil_div(D.cols, G));
      rs_max = std::max(rs_max, ceil_div(D.rows, G));
    }
    AcaBlockDev* dblocks = dalloc<AcaBlockDev>(hb.size(), st);
    HB_CUDA(cudaMemcpyAsync(dblocks, hb.data(), hb.size() * sizeof(AcaBlockDev), cudaMemcpyHostToDevice, st));
    AcaParams prm{dblocks, K, d, 0.0};
    const size_t smem = (size_t)(cs_max + rs_max + kAcaChunk) * sizeof(double);
    ensure_dyn_smem((const void*)aca_sweep_kernel<true>, smem);
    ensure_dyn_smem((const void*)aca_sweep_kernel<false>, smem);
    // blocks of one launch share eps only when it is equal; launch per distinct eps
    std::vector<double> epss;
    for (AcaBlockReq* q : live)
      if (std::find(epss.begin(), epss.end(), q->eps) == epss.end()) epss.push_back(q->eps);
    if (epss.size() == 1) {
      prm.eps = epss[0];
      if (G > 1) {
        void* args[] = {&prm};
        HB_CUDA(cudaLaunchCooperativeKernel((const void*)aca_sweep_kernel<true>, dim3(G, (unsigned)live.size()),
                                            dim3(kAcaThreads), args, smem, st));
        launch_counter().fetch_add(1);
      } else {
        for (size_t b0 = 0; b0 < live.size(); b0 += 65535) {
          AcaParams pp = prm;
          pp.blocks = dblocks + b0;
          const unsigned nb = (unsigned)std::min<size_t>(65535, live.size() - b0);
          aca_sweep_kernel<false><<<dim3(1, nb), kAcaThreads, smem, st>>>(pp);
          HB_LAUNCH_CHECK();
        }
      }
    } else {
      for (size_t i = 0; i < live.size(); ++i) {
        AcaParams pp = prm;
        pp.blocks = dblocks + i;
        pp.eps = live[i]->eps;
        if (G > 1) {
          void* args[] = {&pp};
          HB_CUDA(cudaLaunchCooperativeKernel((const void*)aca_sweep_kernel<true>, dim3(G, 1), dim3(kAcaThreads),
                                              args, smem, st));
          launch_counter().fetch_add(1);
        } else {
          aca_sweep_kernel<false><<<dim3(1, 1), kAcaThreads, smem, st>>>(pp);
          HB_LAUNCH_CHECK();
        }
      }
    }
    if (sync_debug_enabled()) debug_sync_after_launch(__FILE__, __LINE__);
    std::vector<AcaState> hs(live.size());
    if (live.size() == nb) {  // first round: all states contiguous, one copy
      HB_CUDA(cudaMemcpyAsync(hs.data(), states, nb * sizeof(AcaState), cudaMemcpyDeviceToHost, st));
    } else {
      for (size_t i = 0; i < live.size(); ++i)
        HB_CUDA(cudaMemcpyAsync(&hs[i], live[i]->bufs.st, sizeof(AcaState), cudaMemcpyDeviceToHost, st));
    }
    HB_CUDA(cudaStreamSynchronize(st));
    dfree(dblocks, st);
    std::vector<AcaBlockReq*> next;
    for (size_t i = 0; i < live.size(); ++i) {
      AcaBlockReq* q = live[i];
      const AcaState& s = hs[i];
      q->rank = s.rank;
      q->met = (s.met || s.rank == std::min(q->blk.rows, q->blk.cols)) ? 1 : 0;  // aca.hpp:152
      q->bad |= s.bad;
      if (s.grow && !s.bad) {
        // grow U / V (ld unchanged, so the first cap columns copy as one block)
        SweepBufs& b = q->bufs;
        const int64_t m = q->blk.rows, n = q->blk.cols;
        const int64_t ncap = std::min<int64_t>(q->lim, 2 * b.cap);
        double* U2 = dalloc<double>((size_t)(m * ncap), st);
        double* V2 = dalloc<double>((size_t)(n * ncap), st);
        HB_CUDA(cudaMemcpyAsync(U2, b.U, sizeof(double) * m * b.cap, cudaMemcpyDeviceToDevice, st));
        HB_CUDA(cudaMemcpyAsync(V2, b.V, sizeof(double) * n * b.cap, cudaMemcpyDeviceToDevice, st));
        if (b.own_uvp) {
          dfree(b.U, st);
          dfree(b.V, st);
          dfree(b.part, st);
        }
        b.U = U2;
        b.V = V2;
        b.cap = ncap;
        b.part = dalloc<double>((size_t)PartLayout::elems(b.G, b.cap), st);
        b.own_uvp = true;
        next.push_back(q);
      }
    }
    live.swap(next);
  }
  // pivots and pivot ids of the whole batch: the [piv][sig][tau] pieces are contiguous in the
  // arena, so one copy brings them all to the host
  const char* lo = reinterpret_cast<const char*>(reqs.front()->bufs.piv);
  const char* hi = reinterpret_cast<const char*>(reqs.back()->bufs.tau + std::max<int64_t>(reqs.back()->lim, 1));
  std::vector<char> h((size_t)(hi - lo));
  HB_CUDA(cudaMemcpyAsync(h.data(), lo, h.size(), cudaMemcpyDeviceToHost, st));
  HB_CUDA(cudaStreamSynchronize(st));
  for (AcaBlockReq* q : reqs) {
    const size_t r = (size_t)q->rank;
    const double* pv = reinterpret_cast<const double*>(h.data() + (reinterpret_cast<const char*>(q->bufs.piv) - lo));
    const int64_t* sg = reinterpret_cast<const int64_t*>(h.data() + (reinterpret_cast<const char*>(q->bufs.sig) - lo));
    const int64_t* tu = reinterpret_cast<const int64_t*>(h.data() + (reinterpret_cast<const char*>(q->bufs.tau) - lo));
    q->piv_h.assign(pv, pv + r);
    q->sig_h.assign(sg, sg + r);
    q->tau_h.assign(tu, tu + r);
  }
}

static bool degenerate_piv(const std::vector<double>& piv, int64_t r, int64_t* keep) {
  // aca.hpp:177-181 (|diag U| = |pivot_k| since v_k(τ_k) = 1) and the truncation of :186-190
  if (r == 0) {
    *keep = 0;
    return false;
  }
  double mn = std::fabs(piv[0]), mx = mn;
  for (int64_t k = 1; k < r; ++k) {
    mn = std::min(mn, std::fabs(piv[(size_t)k]));
    mx = std::max(mx, std::fabs(piv[(size_t)k]));
  }
  const double cut = 1e-14 * mx;
  int64_t q = 0;
  while (q < r && std::fabs(piv[(size_t)q]) >= cut) ++q;
  *keep = q;
  return mn < cut;
}

static int choose_group(hb_context* c, const hb_block& b) {
  const int64_t big = std::max(b.rows, b.cols);
  // one residual chain per thread: 256-wide slices keep half of the 512 threads busy while
  // the group (and its barriers) stays small; past 37.9k rows every SM takes a slice
  int G = (int)std::min<int64_t>(c->coop_sms, std::max<int64_t>(1, ceil_div(big, 256)));
  if (big <= 512) G = 1;
  G = std::max<int>(G, (int)ceil_div(big, kAcaMaxSlice));
  return G;
}

// compress (aca.hpp:171-198) for nb blocks; G = 1 blocks run batched, larger ones alone.
void aca_compress(hb_context* c, const hb_kernel& kern, const double* x, int64_t nt, const double* y,
                  int64_t ns, int d, const hb_block* blks, int64_t nb, double eps, int64_t max_rank,
                  hb_aca_factor** out) {
  const DevKernel K = dev_kernel(kern);
  cudaStream_t st = c->stream;
  std::vector<AcaBlockReq> reqs((size_t)nb);
  for (int64_t i = 0; i < nb; ++i) {
    reqs[(size_t)i].blk = blks[i];
    reqs[(size_t)i].eps = eps;
    reqs[(size_t)i].max_rank = max_rank;
  }
  std::vector<void*> arenas;
  auto release = [&]() {
    for (auto& r : reqs) free_bufs(r.bufs, st);
    for (void* p : arenas) dfree(p, st);
    arenas.clear();
  };
  auto run_all = [&](std::vector<AcaBlockReq*>& v) {
    std::vector<AcaBlockReq*> small;
    for (AcaBlockReq* q : v) {
      const int G = choose_group(c, q->blk);
      if (G == 1) {
        small.push_back(q);
      } else {
        std::vector<AcaBlockReq*> one{q};
        run_sweeps(c, K, x, nt, y, ns, d, one, G, arenas);
      }
    }
    if (!small.empty()) run_sweeps(c, K, x, nt, y, ns, d, small, 1, arenas);
  };
  try {
    std::vector<AcaBlockReq*> all;
    for (auto& q : reqs) all.push_back(&q);
    run_all(all);
    // degenerate pivots: one more sweep at eps/10 (aca.hpp:184)
    std::vector<AcaBlockReq*> redo;
    for (auto& q : reqs) {
      if (q.bad) throw Error(HB_ESINGULAR, "kernel eval: r == 0 on a singular kernel with no diagonal value");
      int64_t keep = 0;
      if (degenerate_piv(q.piv_h, q.rank, &keep)) {
        free_bufs(q.bufs, st);
        q.eps = eps / 10.0;
        redo.push_back(&q);
      }
    }
    if (!redo.empty()) run_all(redo);
    // factors: L / U of every block from one allocation, built by one launch
    std::vector<int64_t> rk((size_t)nb);
    int64_t tot = 0;
    for (int64_t i = 0; i < nb; ++i) {
      AcaBlockReq& q = reqs[(size_t)i];
      int64_t r = q.rank, keep = r;
      if (degenerate_piv(q.piv_h, r, &keep)) r = keep;  // aca.hpp:185-196
      rk[(size_t)i] = r;
      tot += 2 * r * r;
    }
    std::shared_ptr<double> store;
    if (tot > 0) {
      double* p = nullptr;
      HB_CUDA(cudaMalloc(&p, sizeof(double) * (size_t)tot));
      const int dev = c->device;
      store = std::shared_ptr<double>(p, [dev](double* q) {
        cudaSetDevice(dev);
        cudaFree(q);
      });
    }
    std::vector<LuJob> jobs;
    int64_t off = 0, rmax = 0;
    for (int64_t i = 0; i < nb; ++i) {
      AcaBlockReq& q = reqs[(size_t)i];
      const int64_t r = rk[(size_t)i];
      auto* f = new hb_aca_factor();
      out[i] = f;
      f->device = c->device;
      f->rank = (int32_t)r;
      f->met = q.met;
      f->sigma.assign(q.sig_h.begin(), q.sig_h.begin() + r);
      f->tau.assign(q.tau_h.begin(), q.tau_h.begin() + r);
      for (int64_t k = 0; k < r; ++k) {
        f->sigma[(size_t)k] += q.blk.row_begin;
        f->tau[(size_t)k] += q.blk.col_begin;
      }
      if (r > 0) {
        f->store = store;
        f->L = store.get() + off;
        f->U = f->L + r * r;
        off += 2 * r * r;
        jobs.push_back(LuJob{q.bufs.U, q.bufs.V, q.bufs.sig, q.bufs.tau, q.bufs.piv, q.blk.rows, q.blk.cols, r,
                             f->L, f->U});
        rmax = std::max(rmax, r);
      }
    }
    if (!jobs.empty()) {
      LuJob* dj = dalloc<LuJob>(jobs.size(), st);
      HB_CUDA(cudaMemcpyAsync(dj, jobs.data(), jobs.size() * sizeof(LuJob), cudaMemcpyHostToDevice, st));
      for (size_t j0 = 0; j0 < jobs.size(); j0 += 65535) {
        const unsigned ny = (unsigned)std::min<size_t>(65535, jobs.size() - j0);
        const unsigned nx = (unsigned)std::min<int64_t>(1024, ceil_div(rmax * rmax, 256));
        aca_build_lu_kernel<<<dim3(nx, ny), 256, 0, st>>>(dj + j0);
        HB_LAUNCH_CHECK();
      }
      dfree(dj, st);
    }
    release();
    HB_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    for (int64_t i = 0; i < nb; ++i) {
      delete out[i];
      out[i] = nullptr;
    }
    release();
    throw;
  }
}

// apply (aca.hpp:202-213): b = K(I, τ) U⁻¹ L⁻¹ K(σ, J) q, device vectors q (cols), b (rows)
void aca_apply(hb_context* c, const hb_aca_factor* f, const hb_kernel& kern, const double* x, int64_t nt,
               const double* y, int64_t ns, int d, const hb_block& blk, const double* q, double* b) {
  cudaStream_t st = c->stream;
  const DevKernel K = dev_kernel(kern);
  const int64_t r = f->rank;
  if (r == 0) {
    HB_CUDA(cudaMemsetAsync(b, 0, sizeof(double) * blk.rows, st));
    HB_CUDA(cudaStreamSynchronize(st));
    return;
  }
  int64_t* dsig = dalloc<int64_t>((size_t)r, st);
  int64_t* dtau = dalloc<int64_t>((size_t)r, st);
  double* t = dalloc<double>((size_t)r, st);
  unsigned int* flags = dalloc<unsigned int>(1, st);
  HB_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned int), st));
  HB_CUDA(cudaMemcpyAsync(dsig, f->sigma.data(), sizeof(int64_t) * r, cudaMemcpyHostToDevice, st));
  HB_CUDA(cudaMemcpyAsync(dtau, f->tau.data(), sizeof(int64_t) * r, cudaMemcpyHostToDevice, st));
  aca_apply_rows_kernel<<<(unsigned)r, 256, 0, st>>>(K, d, x, nt, y, ns, blk.col_begin, blk.cols, dsig, q, t, flags);
  HB_LAUNCH_CHECK();
  aca_apply_solve_kernel<<<1, 1024, 0, st>>>(f->L, f->U, r, t);
  HB_LAUNCH_CHECK();
  aca_apply_cols_kernel<<<(unsigned)ceil_div(blk.rows, 256), 256, 0, st>>>(K, d, x, nt, y, ns, blk.row_begin,
                                                                           blk.rows, dtau, t, r, b, flags);
  HB_LAUNCH_CHECK();
  unsigned int hf = 0;
  HB_CUDA(cudaMemcpyAsync(&hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, st));
  HB_CUDA(cudaStreamSynchronize(st));
  for (void* p : {(void*)dsig, (void*)dtau, (void*)t, (void*)flags}) dfree(p, st);
  if (hf & 1u) throw Error(HB_ESINGULAR, "kernel eval: r == 0 on a singular kernel with no diagonal value");
}

}  // namespace hb
