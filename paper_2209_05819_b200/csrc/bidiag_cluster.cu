// One-stage Golub–Kahan bidiagonalisation of a mid-size k x k triangle (kSmallBidiag < k <=
// cluster capacity) held in the distributed shared memory of ONE thread-block cluster (sm_100a).
//
// Why: the two-stage path (GEMM band reduction + bulge chasing) is latency-bound below k ~ 10^3 —
// ~2·k/64 panel factorisations in stage 1 plus a chase whose critical path is ~4k dependent tasks.
// Here the whole triangle lives in the cluster's shared memory (column-cyclic over G CTAs: CTA g
// owns columns g, g+G, ...), every exchange is a DSMEM store/load, and each of the k steps costs
// two hardware cluster barriers.
//
// Step i (left reflector u_i from column i, right reflector v_i from row i; LAPACK dgebrd order):
//   every CTA holds u_i (computed redundantly, bit-identically, from the published column);
//   1. publish row i of own columns q > i, and (owner) column i+1, into every CTA   | barrier #1
//   2. v_i from the full row i (redundant); zp = M[:, own] · v_own (partial)          | barrier #2
//   3. z = Σ_g zp_g (remote loads, fixed order); column i+1 after R_i -> u_{i+1};
//   4. own columns q > i+1: apply R_i then L_{i+1} in one pass.
// The reflector algebra is that of bidiag_small_kernel (svd.cu) and of dgebrd; d, e feed the same
// Sturm-count certification as the two-stage path.
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"
#include "qr.h"

namespace cg = cooperative_groups;

namespace hb {

namespace {
constexpr int kBdThreads = 256;
constexpr int kBdWarps = kBdThreads / 32;

// Householder reflector of x[lo..k-1] (x[lo] = alpha): returns tau; scal = 1/(alpha - beta).
__device__ __forceinline__ void reflector(double alpha, double s, double* tau, double* scal,
                                          double* beta) {
  *tau = 0.0; *scal = 0.0; *beta = alpha;
  if (s > 0.0) {
    *beta = -copysign(sqrt(alpha * alpha + s), alpha);
    *tau = (*beta - alpha) / *beta;
    *scal = 1.0 / (alpha - *beta);
  }
}
}  // namespace

size_t bidiag_cluster_smem(int k, int G) {
  const size_t ncl = (size_t)(k + G - 1) / G;
  return (ncl * (size_t)(k + 1) + 8 * (size_t)k) * sizeof(double);
}

__global__ void __launch_bounds__(kBdThreads) bidiag_cluster_kernel(const double* __restrict__ Mk,
                                                                    int64_t ldm, int k,
                                                                    double* __restrict__ d,
                                                                    double* __restrict__ e) {
  cg::cluster_group cl = cg::this_cluster();
  const int G = (int)cl.num_blocks(), g = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ld = k + 1;
  const int ncl = (k - g + G - 1) / G;       // owned columns: g + jl·G, jl < ncl
  const int ncl_max = (k + G - 1) / G;
  extern __shared__ double sm[];
  double* M = sm;                            // [ncl_max][ld]
  double* row = M + (size_t)ncl_max * ld;    // [2][k]  published row i (all columns)
  double* col = row + 2 * k;                 // [2][k]  published column i+1 (before R_i)
  double* zp = col + 2 * k;                  // [k]     own partial of z = M v
  double* z = zp + k;                        // [k]
  double* u = z + k;                         // [k]
  double* v = u + k;                         // [k]
  __shared__ double red[32];
  __shared__ double sh[4];

  for (int jl = warp; jl < ncl; jl += kBdWarps) {
    const int c = g + jl * G;
    for (int r = lane; r < k; r += 32) M[jl * ld + r] = r <= c ? Mk[r + (int64_t)c * ldm] : 0.0;
  }
  cl.sync();  // every CTA of the cluster is running before any DSMEM access
  // column 0 (owned by CTA 0) to every CTA's col[0]
  if (g == 0)
    for (int idx = tid; idx < k * G; idx += kBdThreads) {
      const int r = idx % k, h = idx / k;
      cl.map_shared_rank(col, h)[r] = M[r];
    }
  cl.sync();
  // u_0
  {
    double s = 0.0;
    for (int r = 1 + tid; r < k; r += kBdThreads) s += col[r] * col[r];
    s = block_sum(s, red);
    if (tid == 0) {
      double tau, scal, beta;
      reflector(col[0], s, &tau, &scal, &beta);
      sh[0] = tau; sh[1] = scal;
      if (g == 0) d[0] = beta;
    }
    __syncthreads();
    const double scal = sh[1];
    for (int r = tid; r < k; r += kBdThreads) u[r] = r == 0 ? 1.0 : col[r] * scal;
    __syncthreads();
  }
  // L_0 on own columns q >= 1
  {
    const double tu = sh[0];
    for (int jl = warp; jl < ncl; jl += kBdWarps) {
      const int q = g + jl * G;
      if (q < 1) continue;
      double* Mq = M + jl * ld;
      double s = 0.0;
      for (int r = lane; r < k; r += 32) s = fma(u[r], Mq[r], s);
      const double w = warp_sum(s) * tu;
      for (int r = lane; r < k; r += 32) Mq[r] = fma(-u[r], w, Mq[r]);
    }
  }
  __syncthreads();

  for (int i = 0; i + 1 < k; ++i) {
    const int p = (i + 1) & 1;
    double* rowp = row + p * k;
    double* colp = col + p * k;
    // ---- 1. publish row i (own columns q > i) and column i+1 (its owner) ----
    {
      const int jl0 = (i + 1 - g + G - 1) / G > 0 ? (i + 1 - g + G - 1) / G : 0;  // first own q > i
      const int nq = ncl - jl0;
      for (int idx = tid; idx < nq * G; idx += kBdThreads) {
        const int jl = jl0 + idx % nq, h = idx / nq;
        cl.map_shared_rank(rowp, h)[g + jl * G] = M[jl * ld + i];
      }
      if ((i + 1) % G == g) {
        const int jl = (i + 1) / G;
        const int nr = k - (i + 1);
        for (int idx = tid; idx < nr * G; idx += kBdThreads) {
          const int r = i + 1 + idx % nr, h = idx / nr;
          cl.map_shared_rank(colp, h)[r] = M[jl * ld + r];
        }
      }
    }
    cl.sync();
    // ---- 2. v_i from row i (columns i+1..k-1), partial z ----
    {
      double s = 0.0;
      for (int q = i + 2 + tid; q < k; q += kBdThreads) s += rowp[q] * rowp[q];
      s = block_sum(s, red);
      if (tid == 0) {
        double tau, scal, beta;
        reflector(rowp[i + 1], s, &tau, &scal, &beta);
        sh[2] = tau; sh[3] = scal;
        if (g == 0) e[i] = beta;
      }
      __syncthreads();
      const double scal = sh[3];
      for (int q = i + 1 + tid; q < k; q += kBdThreads) v[q] = q == i + 1 ? 1.0 : rowp[q] * scal;
      __syncthreads();
      const int jl0 = (i + 1 - g + G - 1) / G > 0 ? (i + 1 - g + G - 1) / G : 0;
      for (int r = i + 1 + tid; r < k; r += kBdThreads) {
        double acc = 0.0;
        for (int jl = jl0; jl < ncl; ++jl) acc = fma(M[jl * ld + r], v[g + jl * G], acc);
        zp[r] = acc;
      }
    }
    cl.sync();
    // ---- 3. z = Σ_g zp_g; column i+1 after R_i -> u_{i+1} ----
    const double tv = sh[2];
    {
      double s = 0.0;
      for (int r = i + 1 + tid; r < k; r += kBdThreads) {
        double acc = 0.0;
#pragma unroll 8
        for (int h = 0; h < G; ++h) acc += cl.map_shared_rank(zp, h)[r];
        z[r] = acc;
        const double cr = colp[r] - tv * acc;  // v_{i+1} = 1
        u[r] = cr;
        if (r > i + 1) s += cr * cr;
      }
      s = block_sum(s, red);  // (its leading barrier also publishes u[] / z[])
      if (tid == 0) {
        double tau, scal, beta;
        reflector(u[i + 1], s, &tau, &scal, &beta);
        sh[0] = tau; sh[1] = scal;
        if (g == 0) d[i + 1] = beta;
      }
      __syncthreads();
      const double scal = sh[1];
      for (int r = i + 1 + tid; r < k; r += kBdThreads) u[r] = r == i + 1 ? 1.0 : u[r] * scal;
      __syncthreads();
    }
    // ---- 4. own columns q > i+1: R_i then L_{i+1} ----
    {
      const double tu = sh[0];
      for (int jl = warp; jl < ncl; jl += kBdWarps) {
        const int q = g + jl * G;
        if (q <= i + 1) continue;
        double* Mq = M + jl * ld;
        const double cv = tv * v[q];
        double s = 0.0;
        for (int r = i + 1 + lane; r < k; r += 32) {
          const double x = fma(-z[r], cv, Mq[r]);
          Mq[r] = x;
          s = fma(u[r], x, s);
        }
        const double w = warp_sum(s) * tu;
        for (int r = i + 1 + lane; r < k; r += 32) Mq[r] = fma(-u[r], w, Mq[r]);
      }
    }
    __syncthreads();
  }
  if (g == 0 && tid == 0) e[k - 1] = 0.0;
  cl.sync();  // no CTA may exit while others still read its shared memory
}

// Largest cluster this kernel can launch with (16 needs the non-portable opt-in), or 0.
int bidiag_cluster_size(int k) {
  static int cap = -1;
  if (cap < 0) {
    cap = 0;
    for (int G : {16, 8}) {
      if (G == 16 &&
          cudaFuncSetAttribute((const void*)bidiag_cluster_kernel,
                               cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      const size_t smem = bidiag_cluster_smem(600, G);
      ensure_dyn_smem((const void*)bidiag_cluster_kernel, smem);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(kBdThreads);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = G; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, (const void*)bidiag_cluster_kernel, &cfg) == cudaSuccess && n > 0) {
        cap = G;
        break;
      }
      cudaGetLastError();
    }
  }
  if (cap == 0) return 0;
  static const int force = [] {
    const char* s = getenv("HB_BD_CLUSTER");
    return s ? atoi(s) : 0;
  }();
  if (force < 0) return 0;  // A/B: two-stage path only
  if ((force == 8 || force == 16) && force <= cap && bidiag_cluster_smem(k, force) <= kBidiagClusterSmem)
    return force;
  // prefer the largest cluster (measured: 16 CTAs slightly ahead of 8 at k = 368)
  for (int G = cap; G >= 8; G /= 2)
    if (bidiag_cluster_smem(k, G) <= kBidiagClusterSmem) return G;
  return 0;
}

void launch_bidiag_cluster(const double* Mk, int64_t ldm, int k, double* d, double* e, int G,
                           cudaStream_t st) {
  const size_t smem = bidiag_cluster_smem(k, G);
  ensure_dyn_smem((const void*)bidiag_cluster_kernel, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kBdThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  HB_CUDA(cudaLaunchKernelEx(&cfg, bidiag_cluster_kernel, Mk, ldm, k, d, e));
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  if (sync_debug_enabled()) debug_sync_after_launch("bidiag_cluster", G);
}

}  // namespace hb
