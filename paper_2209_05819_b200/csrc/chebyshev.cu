// Chebyshev interpolation bound check on the device (chebyshev.hpp:125-193).
//
// interpolation_decay(spec, targets, cube, p_list): for every degree p, the max entry error
// max |K(X, S) - U V| of the tensor Chebyshev interpolant of the kernel along the source cube,
// over the reference's sample grid S (m^d interior points, m = 20 reduced until m^d <= 6.25e6):
//   U (T x M)   = F(x_i, node_k)  -- k2 (launch_assemble) against the Chebyshev nodes,
//   V (M x |S|) = per-axis Lagrange weight products at each sample (cheb_weights_kernel),
//   K (T x |S|) = F(x_i, s_j)     -- k2 against the samples,
//   K <- K - U V                  -- FP64 DMMA GEMM,  err_p = max |K|  (order-free max).
// Samples are processed in slabs so V and K stay within a few GB at any (d, p).
// Nodes, samples and weights follow the reference's arithmetic step for step (separately
// rounded operations, no contraction), so V matches chebyshev.hpp bit for bit; U and K are k2
// entries (<= 1e-13 relative); the GEMM sums in its own order, so err is compared within a
// rounding tolerance (tests/test_gpu_chebyshev.py).
#include <cmath>
#include <vector>

#include "context.h"

namespace hb {

namespace {

// reference sample grid (chebyshev.hpp:160-169): axis d-1 fastest,
// s(a) = lower(a) + side * (idx(a) + 1) / (m + 1)
__global__ void sample_grid_kernel(int d, int m, const double* __restrict__ lower, double side,
                                   int64_t j0, int64_t cnt, double* __restrict__ out) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  int64_t flat = j0 + j;
  for (int a = d - 1; a >= 0; --a) {
    const int64_t idx = flat % m;
    flat /= m;
    const double num = __dmul_rn(side, (double)idx + 1.0);
    out[(int64_t)a * cnt + j] = __dadd_rn(lower[a], __ddiv_rn(num, (double)m + 1.0));
  }
}

// V(:, j) for sample j: per-axis Lagrange weights (chebyshev.hpp:26-45) at the sample's reference
// coordinate (y - lower) / (0.5 side) - 1 (chebyshev.hpp:95), then the tensor products in the
// reference's order (axis 0 slowest, left-to-right multiplication, chebyshev.hpp:93-101).
// One CTA per sample; the d x (p+1) axis weights live in shared memory.
__global__ void cheb_weights_kernel(int d, int p, const double* __restrict__ ref_nodes,
                                    const double* __restrict__ lower, double side,
                                    const double* __restrict__ samples, int64_t cnt,
                                    double* __restrict__ V, int64_t M) {
  extern __shared__ double w[];  // [d][p+1]
  const int64_t j = blockIdx.x;
  const int np1 = p + 1;
  for (int t = threadIdx.x; t < d * np1; t += blockDim.x) {
    const int a = t / np1, jj = t % np1;
    const double y = __dsub_rn(__ddiv_rn(__dsub_rn(samples[(int64_t)a * cnt + j], lower[a]), 0.5 * side), 1.0);
    bool exact = false;
    int hit = -1;
    for (int k = 0; k < np1; ++k)
      if (y == ref_nodes[k]) { exact = true; hit = k; break; }
    double prod;
    if (exact) {
      prod = jj == hit ? 1.0 : 0.0;
    } else {
      prod = 1.0;
      for (int k = 0; k < np1; ++k) {
        if (k == jj) continue;
        prod = __dmul_rn(prod, __ddiv_rn(__dsub_rn(y, ref_nodes[k]), __dsub_rn(ref_nodes[jj], ref_nodes[k])));
      }
    }
    w[t] = prod;
  }
  __syncthreads();
  double* col = V + j * M;
  for (int64_t k = threadIdx.x; k < M; k += blockDim.x) {
    // multi-index of node k, axis 0 slowest
    int64_t rem = k, div = M / np1;
    double v = 1.0;
    for (int a = 0; a < d; ++a) {
      const int ia = (int)(rem / div);
      rem -= (int64_t)ia * div;
      div /= np1;
      v = __dmul_rn(v, w[a * np1 + ia]);
    }
    col[k] = v;
  }
}

__global__ void absmax_kernel(const double* __restrict__ C, int64_t m, int64_t n, int64_t ld,
                              double* __restrict__ parts) {
  __shared__ double red[32];
  double mx = 0.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < m * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const double v = fabs(C[idx % m + (idx / m) * ld]);
    mx = (v > mx || v != v) ? v : mx;  // NaN propagates
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (t > mx || t != t) ? t : mx;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = (red[w] > r || red[w] != red[w]) ? red[w] : r;
    parts[blockIdx.x] = r;
  }
}

}  // namespace

// chebyshev_nodes (chebyshev.hpp:16-23): cos(pi k / p), k = 0..p; p = 0 -> {0}.
std::vector<double> cheb_nodes_host(int p) {
  if (p < 0) throw Error(HB_EINVAL, "chebyshev_nodes: p must be >= 0");
  if (p == 0) return {0.0};
  std::vector<double> y((size_t)p + 1);
  for (int k = 0; k <= p; ++k) y[(size_t)k] = std::cos(M_PI * k / p);
  return y;
}

void interpolation_decay(hb_context* c, const hb_kernel& kern, const double* tgt_soa, int64_t T,
                         const hb_cube& cube, const int32_t* p_list, int np, double* err_out) {
  const int d = cube.d;
  cudaStream_t st = c->stream;
  // the reference's sample density (chebyshev.hpp:156-158)
  int m = 20;
  while (std::pow(double(m), d) > 6.25e6 && m > 2) --m;
  int64_t count = 1;
  for (int a = 0; a < d; ++a) count *= m;
  const int64_t ldt = round_up(T, 8);
  double* X = ws<double>(c, B_X, (size_t)d * T);
  double* lo = ws<double>(c, B_PN, 16);
  HB_CUDA(cudaMemcpyAsync(X, tgt_soa, sizeof(double) * d * T, cudaMemcpyHostToDevice, st));
  HB_CUDA(cudaMemcpyAsync(lo, cube.lower, sizeof(double) * d, cudaMemcpyHostToDevice, st));
  unsigned int* flags = ws<unsigned int>(c, B_FLAGS, 4);
  HB_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned int), st));
  double* parts = ws<double>(c, B_FRO, 592);
  std::vector<double> host_parts(592);
  for (int ip = 0; ip < np; ++ip) {
    const int p = p_list[ip];
    const std::vector<double> ref = cheb_nodes_host(p);
    const int np1 = p + 1;
    int64_t M = 1;
    for (int a = 0; a < d; ++a) M *= np1;
    // Chebyshev grid of the cube (chebyshev.hpp:66-86): node(flat, a) = c(a) + h * ref(idx(a)),
    // c = lower + 0.5 side (cube.center()), h = 0.5 side; axis d-1 fastest
    std::vector<double> nodes((size_t)(d * M));
    {
      std::vector<int> idx(d, 0);
      const double h = 0.5 * cube.side;
      for (int64_t flat = 0; flat < M; ++flat) {
        for (int a = 0; a < d; ++a) {
          const double ca = cube.lower[a] + 0.5 * cube.side;
          nodes[(size_t)(a * M + flat)] = ca + h * ref[(size_t)idx[a]];
        }
        for (int a = d - 1; a >= 0; --a) {
          if (++idx[a] <= p) break;
          idx[a] = 0;
        }
      }
    }
    double* Nd = ws<double>(c, B_Y, (size_t)d * M);
    double* R = ws<double>(c, B_RDIAG2, (size_t)np1);
    HB_CUDA(cudaMemcpyAsync(Nd, nodes.data(), sizeof(double) * d * M, cudaMemcpyHostToDevice, st));
    HB_CUDA(cudaMemcpyAsync(R, ref.data(), sizeof(double) * np1, cudaMemcpyHostToDevice, st));
    double* U = ws<double>(c, B_CERT_M, (size_t)ldt * M);
    launch_assemble(kern, X, T, Nd, M, d, U, ldt, flags, st);
    // sample slabs: V (M x s) and K (T x s) within ~6 GB
    const int64_t per = 8 * (M + ldt + d);
    const int64_t slab = std::max<int64_t>(1, std::min<int64_t>(count, (int64_t(6) << 30) / per));
    double err = 0.0;
    for (int64_t j0 = 0; j0 < count; j0 += slab) {
      const int64_t cnt = std::min(slab, count - j0);
      double* S = ws<double>(c, B_OMEGA, (size_t)d * cnt);
      double* V = ws<double>(c, B_CERT_B, (size_t)M * cnt);
      double* K = ws<double>(c, B_A, (size_t)ldt * cnt);
      sample_grid_kernel<<<(unsigned)ceil_div(cnt, 256), 256, 0, st>>>(d, m, lo, cube.side, j0, cnt, S);
      HB_LAUNCH_CHECK();
      const size_t wsm = sizeof(double) * d * np1;
      ensure_dyn_smem((const void*)cheb_weights_kernel, wsm);
      cheb_weights_kernel<<<(unsigned)cnt, 256, wsm, st>>>(d, p, R, lo, cube.side, S, cnt, V, M);
      HB_LAUNCH_CHECK();
      launch_assemble(kern, X, T, S, cnt, d, K, ldt, flags, st);
      GemmArgs g{};
      g.M = T; g.N = cnt; g.K = M; g.alpha = -1.0; g.A = U; g.lda = ldt; g.transA = false;
      g.B = V; g.ldb = M; g.beta = 1.0; g.C = K; g.ldc = ldt;
      double* sk = ws<double>(c, B_SPLITK, 24ll << 20);
      launch_dgemm(g, sk, 24ll << 20, c->num_sms, st);
      absmax_kernel<<<592, 256, 0, st>>>(K, T, cnt, ldt, parts);
      HB_LAUNCH_CHECK();
      HB_CUDA(cudaMemcpyAsync(host_parts.data(), parts, sizeof(double) * 592, cudaMemcpyDeviceToHost, st));
      HB_CUDA(cudaStreamSynchronize(st));
      for (double v : host_parts) err = (v > err || v != v) ? v : err;
    }
    err_out[ip] = err;
  }
  unsigned int f = 0;
  HB_CUDA(cudaMemcpy(&f, flags, sizeof(f), cudaMemcpyDeviceToHost));
  if (f & 1u) throw Error(HB_ESINGULAR, "kernel eval: r == 0 on a singular kernel with no diagonal value");
  if (f & 2u) throw Error(HB_EDOMAIN, "non-finite kernel entries");
}

}  // namespace hb
