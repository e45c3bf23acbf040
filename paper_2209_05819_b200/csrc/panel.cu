// Householder panel QR with the panel resident in shared memory (sm_100a).
//
// The mp x b panel is split into row chunks, one per CTA (grid-cooperative, co-resident); each
// CTA copies its chunk into shared memory once, runs all b column steps on it, and writes R, V
// back at the end.  Per column one cross-CTA reduction touches global memory (one grid barrier,
// below); everything else is shared-memory work.  The host (rank.cu: panel_and_T) splits panels whose chunk would not fit
// (tall panels) into column sub-panels and joins them with DMMA GEMM updates.
#include "common.cuh"
#include "kernels.h"
#include "qr.h"

namespace hb {

// One grid barrier per column.  For column c every CTA publishes, over its own rows i > c, the
// partial products g_q = Σ x_i·P[i,q] for q >= c (g_c is the squared norm below the diagonal),
// and the CTA owning row c publishes that row.  After the barrier every CTA reduces the partials
// itself (fixed order: deterministic, identical in all CTAs), forms the reflector
//   β = −sign(α)·sqrt(α² + g_c),  τ = (β − α)/β,  v = (x − β e_c)/(α − β)  (v_c = 1),
// and w_q = τ·vᵀP[:,q] = τ·(P[c,q] + g_q/(α − β)) without a second reduction, updates its rows,
// and accumulates the partials of column c+1 in the same pass.
__global__ void __launch_bounds__(kPanelThreads) panel_qr_smem_kernel(PanelParams p) {
  GridSync gbar(p.bar);
  constexpr int NW = kPanelThreads / 32;
  extern __shared__ double psm[];
  __shared__ double red[NW][128];
  const int G = gridDim.x, g = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = p.b;
  const int64_t chunk = p.chunk;
  const int64_t r0 = g * chunk, r1 = min(p.mp, r0 + chunk);
  const int rows = (int)max((int64_t)0, r1 - r0);
  const int ldS = (int)chunk + 1;        // odd stride: column-wise and row-wise smem access both spread
  double* S = psm;                       // [b][ldS]
  double* ws = psm + (size_t)b * ldS;    // [b]  w_q
  double* P = p.P;
  const int64_t ld = p.ld;
  const int nref = (int)min((int64_t)b, p.mp);
  double* part = p.wslot;                // [2][G][b]
  double* rowc = p.scal;                 // [2][b]

  for (int q = warp; q < b; q += NW)
    for (int i = lane; i < rows; i += 32) S[q * ldS + i] = P[r0 + i + (int64_t)q * ld];
  __syncthreads();
  // partials of column 0
  if (nref > 0) {
    const int i0 = r0 == 0 ? 1 : 0;
    for (int q = warp; q < b; q += NW) {
      const double* Sq = S + q * ldS;
      double s = 0.0;
      for (int i = i0 + lane; i < rows; i += 32) s = fma(S[i], Sq[i], s);
      s = warp_sum(s);
      if (lane == 0) part[(size_t)g * b + q] = s;
    }
    if (r0 == 0 && rows > 0)
      for (int q = tid; q < b; q += kPanelThreads) rowc[q] = S[q * ldS];
  }
  gbar.sync();

  for (int c = 0; c < nref; ++c) {
    const int par = c & 1;
    const double* pp = part + (size_t)par * G * b;
    const double* rc = rowc + par * b;
    // ---- reduce the partials of column c: lanes over q, warps over CTAs, fixed order ----
    {
      double s[4] = {0.0, 0.0, 0.0, 0.0};
      for (int h = warp; h < G; h += NW) {
        const double* row = pp + (size_t)h * b;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int q = c + lane + 32 * j;
          if (q < b) s[j] += __ldcg(row + q);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) red[warp][lane + 32 * j] = s[j];
    }
    __syncthreads();
    // every thread forms the reflector itself from the reduced g_c (same arithmetic, same order:
    // identical in all threads and CTAs) — no extra barrier for a broadcast
    double gc = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) gc += red[w][0];
    const double alpha = __ldcg(rc + c);
    double tau = 0.0, scal = 0.0, beta = alpha;
    if (gc > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + gc), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (g == 0 && tid == 0) p.tau[c] = tau;
    for (int q = c + 1 + tid; q < b; q += kPanelThreads) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) t += red[w][q - c];
      ws[q] = tau * (__ldcg(rc + q) + scal * t);
    }
    const int ic = (int)max((int64_t)0, (int64_t)c - r0);        // first local row >= c
    const int i1 = (int)max((int64_t)0, (int64_t)(c + 1) - r0);  // first local row > c
    const int in = (int)max((int64_t)0, (int64_t)(c + 2) - r0);  // first local row > c+1
    double* Sc = S + c * ldS;
    // scale v (column c) and, in the same pass and thread→row mapping, update column c+1 (its
    // entries feed the partials of the other columns); w_{c+1} is formed by every thread
    if (c + 1 < b) {
      double t1 = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) t1 += red[w][1];
      const double wq = tau * (__ldcg(rc + c + 1) + scal * t1);  // == ws[c+1]
      double* Sq = S + (c + 1) * ldS;
      for (int i = i1 + tid; i < rows; i += kPanelThreads) {
        const double v = Sc[i] * scal;
        Sc[i] = v;
        Sq[i] = fma(-v, wq, Sq[i]);
      }
      if (ic < i1 && ic < rows && tid == 0) {  // row c: R diagonal (v_c = 1 implicit)
        Sc[ic] = beta;
        Sq[ic] -= wq;
      }
    } else {
      for (int i = i1 + tid; i < rows; i += kPanelThreads) Sc[i] *= scal;
      if (ic < i1 && ic < rows && tid == 0) Sc[ic] = beta;
    }
    __syncthreads();
    if (c + 1 >= b) break;
    const bool more = c + 1 < nref;
    double* pn = part + (size_t)(par ^ 1) * G * b;
    double* rn = rowc + (par ^ 1) * b;
    const double* Sn = S + (c + 1) * ldS;
    const bool owner = r0 <= c + 1 && c + 1 < r1;
    for (int q = c + 1 + warp; q < b; q += NW) {
      double* Sq = S + q * ldS;
      double acc = 0.0;
      if (q > c + 1) {
        const double wq = ws[q];
        if (lane == 0)  // rows c and c+1 (at most two, owned by this CTA or not)
          for (int i = ic; i < min(in, rows); ++i) Sq[i] -= (i < i1 ? 1.0 : Sc[i]) * wq;
        for (int i = in + lane; i < rows; i += 32) {
          const double x = fma(-Sc[i], wq, Sq[i]);
          Sq[i] = x;
          acc = fma(Sn[i], x, acc);
        }
      } else {
        for (int i = in + lane; i < rows; i += 32) acc = fma(Sn[i], Sq[i], acc);
      }
      if (more) {
        __syncwarp();
        acc = warp_sum(acc);
        if (lane == 0) {
          pn[(size_t)g * b + q] = acc;
          if (owner) rn[q] = Sq[c + 1 - r0];
        }
      }
    }
    if (!more) break;
    gbar.sync();
  }
  // the last column(s) beyond nref (wide panels) were updated in place above
  for (int q = warp; q < b; q += NW) {
    const double* Sq = S + q * ldS;
    double* vq = p.V + (int64_t)q * p.ldv;
    double* pq = P + (int64_t)q * ld;
    for (int i = lane; i < rows; i += 32) {
      const int64_t r = r0 + i;
      pq[r] = Sq[i];
      vq[r] = q >= nref ? 0.0 : (r > q ? Sq[i] : (r == q ? 1.0 : 0.0));
    }
  }
  if (g == 0)
    for (int q = nref + tid; q < b; q += kPanelThreads) p.tau[q] = 0.0;
}

}  // namespace hb

// ---------------------------------------------------------------------------------------------
// Cluster variant for panels that fit the distributed shared memory of one thread-block cluster
// (G <= 16 CTAs, rows split in contiguous chunks as above).  Same algebra and the same one
// exchange per column, but the exchange is DSMEM: each CTA stores its partials g_q (and the row
// owner its row c+1) straight into every CTA's shared memory and the column ends on a hardware
// cluster barrier (barrier.cluster arrive.release / wait.acquire) instead of a grid barrier and
// an L2 round trip.  Every CTA then reduces the G partials of each q locally in a fixed order
// (identical in all CTAs).
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace hb {

size_t panel_cluster_smem(int64_t chunk, int b, int G) {
  return ((size_t)b * (chunk + 1) + (size_t)b + 2 * (size_t)G * b + 2 * (size_t)b) * sizeof(double);
}

__global__ void __launch_bounds__(kPanelThreads) panel_qr_cluster_kernel(PanelParams p) {
  cg::cluster_group cl = cg::this_cluster();
  constexpr int NW = kPanelThreads / 32;
  extern __shared__ double psm[];
  const int G = (int)cl.num_blocks(), g = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = p.b;
  const int64_t chunk = p.chunk;
  const int64_t r0 = g * chunk, r1 = min(p.mp, r0 + chunk);
  const int rows = (int)max((int64_t)0, r1 - r0);
  const int ldS = (int)chunk + 1;
  double* S = psm;                        // [b][ldS]
  double* ws = S + (size_t)b * ldS;       // [b]       w_q
  double* part = ws + b;                  // [2][G][b] partials of every CTA (DSMEM-written)
  double* rowc = part + 2 * (size_t)G * b;  // [2][b]  published row c
  double* P = p.P;
  const int64_t ld = p.ld;
  const int nref = (int)min((int64_t)b, p.mp);

  for (int q = warp; q < b; q += NW)
    for (int i = lane; i < rows; i += 32) S[q * ldS + i] = P[r0 + i + (int64_t)q * ld];
  __syncthreads();
  cl.sync();  // every CTA is running before any DSMEM store
  if (nref > 0) {
    const int i0 = r0 == 0 ? 1 : 0;
    for (int q = warp; q < b; q += NW) {
      const double* Sq = S + q * ldS;
      double s = 0.0;
      for (int i = i0 + lane; i < rows; i += 32) s = fma(S[i], Sq[i], s);
      s = warp_sum(s);
      if (lane < G) cl.map_shared_rank(part, lane)[(size_t)g * b + q] = s;
    }
    if (r0 == 0 && rows > 0)
      for (int idx = tid; idx < b * G; idx += kPanelThreads)
        cl.map_shared_rank(rowc, idx / b)[idx % b] = S[(idx % b) * ldS];
  }
  cl.sync();

  for (int c = 0; c < nref; ++c) {
    const int par = c & 1;
    const double* pp = part + (size_t)par * G * b;
    const double* rc = rowc + par * b;
    // reduced partials, fixed order over CTAs (identical everywhere)
    double gc = 0.0;
    for (int h = 0; h < G; ++h) gc += pp[(size_t)h * b + c];
    const double alpha = rc[c];
    double tau = 0.0, scal = 0.0, beta = alpha;
    if (gc > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + gc), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (g == 0 && tid == 0) p.tau[c] = tau;
    for (int q = c + 1 + tid; q < b; q += kPanelThreads) {
      double t = 0.0;
      for (int h = 0; h < G; ++h) t += pp[(size_t)h * b + q];
      ws[q] = tau * (rc[q] + scal * t);
    }
    const int ic = (int)max((int64_t)0, (int64_t)c - r0);
    const int i1 = (int)max((int64_t)0, (int64_t)(c + 1) - r0);
    const int in = (int)max((int64_t)0, (int64_t)(c + 2) - r0);
    double* Sc = S + c * ldS;
    if (c + 1 < b) {
      double t1 = 0.0;
      for (int h = 0; h < G; ++h) t1 += pp[(size_t)h * b + c + 1];
      const double wq = tau * (rc[c + 1] + scal * t1);  // == ws[c+1]
      double* Sq = S + (c + 1) * ldS;
      for (int i = i1 + tid; i < rows; i += kPanelThreads) {
        const double v = Sc[i] * scal;
        Sc[i] = v;
        Sq[i] = fma(-v, wq, Sq[i]);
      }
      if (ic < i1 && ic < rows && tid == 0) {
        Sc[ic] = beta;
        Sq[ic] -= wq;
      }
    } else {
      for (int i = i1 + tid; i < rows; i += kPanelThreads) Sc[i] *= scal;
      if (ic < i1 && ic < rows && tid == 0) Sc[ic] = beta;
    }
    __syncthreads();
    if (c + 1 >= b) break;
    const bool more = c + 1 < nref;
    double* pn = part + (size_t)(par ^ 1) * G * b;
    double* rn = rowc + (par ^ 1) * b;
    const double* Sn = S + (c + 1) * ldS;
    const bool owner = r0 <= c + 1 && c + 1 < r1;
    for (int q = c + 1 + warp; q < b; q += NW) {
      double* Sq = S + q * ldS;
      double acc = 0.0;
      if (q > c + 1) {
        const double wq = ws[q];
        if (lane == 0)
          for (int i = ic; i < min(in, rows); ++i) Sq[i] -= (i < i1 ? 1.0 : Sc[i]) * wq;
        __syncwarp();
        for (int i = in + lane; i < rows; i += 32) {
          const double x = fma(-Sc[i], wq, Sq[i]);
          Sq[i] = x;
          acc = fma(Sn[i], x, acc);
        }
      } else {
        for (int i = in + lane; i < rows; i += 32) acc = fma(Sn[i], Sq[i], acc);
      }
      if (more) {
        acc = warp_sum(acc);
        __syncwarp();
        if (lane < G) {
          cl.map_shared_rank(pn, lane)[(size_t)g * b + q] = acc;
          if (owner) cl.map_shared_rank(rn, lane)[q] = Sq[c + 1 - r0];
        }
      }
    }
    if (!more) break;
    cl.sync();
  }
  for (int q = warp; q < b; q += NW) {
    const double* Sq = S + q * ldS;
    double* vq = p.V + (int64_t)q * p.ldv;
    double* pq = P + (int64_t)q * ld;
    for (int i = lane; i < rows; i += 32) {
      const int64_t r = r0 + i;
      pq[r] = Sq[i];
      vq[r] = q >= nref ? 0.0 : (r > q ? Sq[i] : (r == q ? 1.0 : 0.0));
    }
  }
  if (g == 0)
    for (int q = nref + tid; q < b; q += kPanelThreads) p.tau[q] = 0.0;
  cl.sync();  // no CTA exits while others may still store into its shared memory
}

}  // namespace hb

namespace hb {

int cluster_cap(const void* kern, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<const void*, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(kern);
  if (it != cache.end()) return it->second;
  int cap = 0;
  for (int G : {16, 8}) {
    if (G == 16 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    ensure_dyn_smem(kern, smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) {
      cap = G;
      break;
    }
    cudaGetLastError();
  }
  cache[kern] = cap;
  return cap;
}

// Largest cluster size the panel kernel can launch with at the full shared-memory budget.
int panel_cluster_max() {
  return cluster_cap((const void*)panel_qr_cluster_kernel, kPanelThreads, kPanelClusterSmem);
}

void launch_panel_cluster(const PanelParams& pp, int G, cudaStream_t st) {
  const size_t smem = panel_cluster_smem(pp.chunk, pp.b, G);
  ensure_dyn_smem((const void*)panel_qr_cluster_kernel, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kPanelThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  HB_CUDA(cudaLaunchKernelEx(&cfg, panel_qr_cluster_kernel, pp));
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  if (sync_debug_enabled()) debug_sync_after_launch("panel_cluster", G);
}

}  // namespace hb
