// Householder panel QR with the panel resident in shared memory (sm_100a).
//
// The mp x b panel is split into row chunks, one per CTA (grid-cooperative, co-resident); each
// CTA copies its chunk into shared memory once, runs all b column steps on it, and writes R, V
// back at the end.  Per column only two cross-CTA reductions touch global memory (the column
// norm, and w = vᵀP for the trailing panel columns), each one grid barrier; everything else is
// shared-memory work.  The host (rank.cu: panel_and_T) splits panels whose chunk would not fit
// (tall panels) into column sub-panels and joins them with DMMA GEMM updates.
#include "common.cuh"
#include "kernels.h"
#include "qr.h"

namespace hb {

__global__ void __launch_bounds__(256) panel_qr_smem_kernel(PanelParams p) {
  extern __shared__ double psm[];
  const int G = gridDim.x, g = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = p.b;
  const int64_t chunk = p.chunk;
  const int64_t r0 = g * chunk, r1 = min(p.mp, r0 + chunk);
  const int rows = (int)max((int64_t)0, r1 - r0);
  const int ldS = (int)chunk + 1;  // odd stride: column-wise and row-wise smem access both spread
  double* S = psm;                 // [b][ldS]
  double* ws = psm + (size_t)b * ldS;  // [b]
  __shared__ double sh[4];
  __shared__ double red[32];
  double* P = p.P;
  const int64_t ld = p.ld;
  const int nref = (int)min((int64_t)b, p.mp);

  // load the chunk (coalesced along rows)
  for (int q = warp; q < b; q += 8)
    for (int i = lane; i < rows; i += 32) S[q * ldS + i] = P[r0 + i + (int64_t)q * ld];
  __syncthreads();
  // column 0: partial norm over rows > 0, owner publishes alpha
  if (warp == 0) {
    double s = 0.0;
    for (int i = lane; i < rows; i += 32)
      if (r0 + i > 0) s += S[i] * S[i];
    s = warp_sum(s);
    if (lane == 0) {
      p.nslot[g] = s;
      if (r0 == 0 && rows > 0) p.scal[0] = S[0];
    }
  }
  grid_sync(p.bar);

  for (int c = 0; c < nref; ++c) {
    const int par = c & 1;
    // ---- reflector of column c ----
    {
      const double s = block_sum_strided(p.nslot, G, 1, red);
      if (tid == 0) {
        const double alpha = p.scal[par];
        double tau = 0.0, scal = 0.0, beta = alpha;
        if (s > 0.0) {
          beta = -copysign(sqrt(alpha * alpha + s), alpha);
          tau = (beta - alpha) / beta;
          scal = 1.0 / (alpha - beta);
        }
        sh[0] = tau; sh[1] = scal; sh[2] = beta;
        if (g == 0) p.tau[c] = tau;
      }
    }
    __syncthreads();
    const double tau = sh[0], scal = sh[1];
    const int ic = (int)max((int64_t)0, (int64_t)c - r0);  // first local row >= c
    double* Sc = S + c * ldS;
    for (int i = ic + tid; i < rows; i += 256) {
      if (r0 + i > c) Sc[i] *= scal;
    }
    __syncthreads();
    // v_i = Sc[i] for rows > c, 1 at row c
    // ---- w_q = sum_i v_i P[i, q] (q > c), partial over own rows ----
    for (int q = c + 1 + warp; q < b; q += 8) {
      const double* Sq = S + q * ldS;
      double s = 0.0;
      for (int i = ic + lane; i < rows; i += 32) {
        const double vi = (r0 + i == c) ? 1.0 : Sc[i];
        s += vi * Sq[i];
      }
      s = warp_sum(s);
      if (lane == 0) p.wslot[(size_t)g * b + q] = s;
    }
    grid_sync(p.bar);
    for (int q = c + 1 + warp; q < b; q += 8) {
      const double s = warp_sum_strided(p.wslot + q, G, b);
      if (lane == 0) ws[q] = s * tau;
    }
    __syncthreads();
    // ---- update own rows; partial norm of column c+1 (rows > c+1); owner publishes alpha ----
    double nrm = 0.0;
    for (int q = c + 1 + warp; q < b; q += 8) {
      double* Sq = S + q * ldS;
      const double wq = ws[q];
      for (int i = ic + lane; i < rows; i += 32) {
        const double vi = (r0 + i == c) ? 1.0 : Sc[i];
        const double x = Sq[i] - vi * wq;
        Sq[i] = x;
        if (q == c + 1 && r0 + i > c + 1) nrm += x * x;
      }
    }
    if (warp == 0) {  // q == c + 1 is handled by warp 0
      nrm = warp_sum(nrm);
      if (lane == 0) p.nslot[g] = nrm;
    }
    if (r0 <= c && c < r1 && tid == 0) Sc[c - r0] = sh[2];  // R diagonal
    __syncthreads();
    if (c + 1 < nref && r0 <= c + 1 && c + 1 < r1 && tid == 0)
      p.scal[par ^ 1] = S[(c + 1) * ldS + (c + 1 - r0)];
    grid_sync(p.bar);
  }
  // write back R / V and the explicit V (unit diagonal, zeros above, zero columns >= nref)
  for (int q = warp; q < b; q += 8) {
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
    for (int q = nref + tid; q < b; q += 256) p.tau[q] = 0.0;
}

}  // namespace hb
