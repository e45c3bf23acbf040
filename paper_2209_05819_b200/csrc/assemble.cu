// k1 (seeded / grid point generator) and k2 (FP64 kernel-block assembly) for sm_100a.
//
// k2 restates hodlr::assemble_dense (kernel.hpp:168-181) with the entry rule of eval_radial
// (kernel.hpp:149-157) and KernelSpec::operator() (kernel.hpp:93-109):
//   K(i, j) = F(||x_i - y_j||_2),  column-major T x N (types.hpp:11 Matrix = MatrixXd),
//   r computed as a left-to-right sum of squared differences (the order Eigen uses for the
//   strided rows of a column-major PointSet, kernel.hpp:179), every multiply/add rounded
//   separately (__dmul_rn/__dadd_rn: no FMA contraction), IEEE sqrt, so r is bit-identical to
//   the CPU oracle; F uses CUDA libdevice log/exp/sin/cos (<= 2 ulp).
// Layout: a CTA owns a 128-row x 64-column tile; target/source coordinates of the tile are
// staged in shared memory (SoA); each thread produces 2 consecutive rows of 16 columns and
// writes them with 16-byte vector stores, so a warp stores 512 contiguous bytes per column.
#include "common.cuh"
#include "kernels.h"
#include "entries.cuh"

namespace hb {

__global__ void points_kernel(hb_cube cube, int64_t n, int d, int mode, int64_t m_axis,
                              uint64_t seed, int role, double* __restrict__ out) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n * d) return;
  const int k = (int)(idx / n);
  const int64_t i = idx - (int64_t)k * n;
  double t;
  if (mode == HB_POINTS_UNIFORM) {
    const uint64_t stream = splitmix64(seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(role + 1)));
    const uint64_t bits = splitmix64(stream + (uint64_t)i * 8u + (uint64_t)k);
    t = __dmul_rn((double)(bits >> 12) + 0.5, 0x1p-52);
  } else {
    int64_t rest = i;
    for (int q = 0; q < k; ++q) rest /= m_axis;
    const int64_t g = rest % m_axis;
    t = (mode == HB_POINTS_GRID_INTERIOR) ? __ddiv_rn((double)(g + 1), (double)(m_axis + 1))
                                          : __ddiv_rn((double)g, (double)(m_axis - 1));
  }
  out[idx] = __dadd_rn(cube.lower[k], __dmul_rn(cube.side, t));
}

constexpr int kTileRows = 128, kTileCols = 64;

// D > 0: compile-time dimension; D == 0: runtime d (5..8).
template <int KID, int D, bool VEC>
__global__ void __launch_bounds__(256) assemble_kernel(const double* __restrict__ x, int64_t T,
                                                       const double* __restrict__ y, int64_t N,
                                                       int d_rt, double* __restrict__ K,
                                                       int64_t ldk, int has_diag, double diag,
                                                       int singular, unsigned int* flags) {
  const int d = D > 0 ? D : d_rt;
  __shared__ double xs[8][kTileRows];
  __shared__ double ys[8][kTileCols];
  const int64_t r0 = (int64_t)blockIdx.x * kTileRows;
  const int64_t c0 = (int64_t)blockIdx.y * kTileCols;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  for (int q = tid; q < d * kTileRows; q += 256) {
    const int k = q / kTileRows, i = q % kTileRows;
    xs[k][i] = (r0 + i < T) ? x[(int64_t)k * T + r0 + i] : 0.0;
  }
  for (int q = tid; q < d * kTileCols; q += 256) {
    const int k = q / kTileCols, j = q % kTileCols;
    ys[k][j] = (c0 + j < N) ? y[(int64_t)k * N + c0 + j] : 0.0;
  }
  __syncthreads();
  const int li = 2 * threadIdx.x;  // local row pair
  const int64_t i0 = r0 + li;
  unsigned int bad = 0;
  for (int jj = threadIdx.y; jj < kTileCols; jj += blockDim.y) {
    const int64_t j = c0 + jj;
    if (j >= N) break;
    double v[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < (D > 0 ? D : 8); ++k) {
        if (D == 0 && k >= d) break;
        const double df = __dsub_rn(xs[k][li + h], ys[k][jj]);
        const double sq = __dmul_rn(df, df);
        s = (k == 0) ? sq : __dadd_rn(s, sq);
      }
      const double r = __dsqrt_rn(s);
      double f;
      if (r == 0.0) {
        if (has_diag) {
          f = diag;
        } else if (singular) {
          bad |= 1u;
          f = 0.0;
        } else {
          f = radial<KID>(0.0);
        }
      } else {
        f = radial<KID>(r);
      }
      if (!isfinite(f)) bad |= 2u;
      v[h] = f;
    }
    double* col = K + j * ldk;
    if (VEC && i0 + 1 < T) {
      *reinterpret_cast<double2*>(col + i0) = make_double2(v[0], v[1]);
    } else {
      if (i0 < T) col[i0] = v[0];
      if (i0 + 1 < T) col[i0 + 1] = v[1];
    }
  }
  if (bad) atomicOr(flags, bad);
}

__global__ void negate_block_kernel(double* __restrict__ A, int64_t m, int64_t n, int64_t ld) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= m * n) return;
  const int64_t i = idx % m, j = idx / m;
  A[i + j * ld] = -A[i + j * ld];
}

void launch_negate(double* A, int64_t m, int64_t n, int64_t ld, cudaStream_t st) {
  negate_block_kernel<<<(unsigned)ceil_div(m * n, 256), 256, 0, st>>>(A, m, n, ld);
  HB_LAUNCH_CHECK();
}

void launch_points(const hb_cube& cube, int64_t n, int mode, int64_t m_axis, uint64_t seed,
                   int role, double* out, cudaStream_t st) {
  const int64_t total = n * cube.d;
  const int threads = 256;
  points_kernel<<<(unsigned)ceil_div(total, threads), threads, 0, st>>>(cube, n, cube.d, mode,
                                                                         m_axis, seed, role, out);
  HB_LAUNCH_CHECK();
}

template <int KID, int D>
static void launch_assemble_kd(const double* x, int64_t T, const double* y, int64_t N, int d,
                               double* K, int64_t ldk, int has_diag, double diag, int singular,
                               unsigned int* flags, cudaStream_t st) {
  dim3 block(64, 4);
  dim3 grid((unsigned)ceil_div(T, kTileRows), (unsigned)ceil_div(N, kTileCols));
  HB_REQUIRE(grid.y <= 65535u, HB_ECAP, "assemble: N too large for the grid");
  const bool vec = (ldk % 2 == 0) && ((reinterpret_cast<uintptr_t>(K) & 15) == 0);
  if (vec)
    assemble_kernel<KID, D, true><<<grid, block, 0, st>>>(x, T, y, N, d, K, ldk, has_diag, diag,
                                                          singular, flags);
  else
    assemble_kernel<KID, D, false><<<grid, block, 0, st>>>(x, T, y, N, d, K, ldk, has_diag, diag,
                                                           singular, flags);
  HB_LAUNCH_CHECK();
}

template <int KID>
static void launch_assemble_k(const double* x, int64_t T, const double* y, int64_t N, int d,
                              double* K, int64_t ldk, int has_diag, double diag, int singular,
                              unsigned int* flags, cudaStream_t st) {
  switch (d) {
    case 1: launch_assemble_kd<KID, 1>(x, T, y, N, d, K, ldk, has_diag, diag, singular, flags, st); break;
    case 2: launch_assemble_kd<KID, 2>(x, T, y, N, d, K, ldk, has_diag, diag, singular, flags, st); break;
    case 3: launch_assemble_kd<KID, 3>(x, T, y, N, d, K, ldk, has_diag, diag, singular, flags, st); break;
    case 4: launch_assemble_kd<KID, 4>(x, T, y, N, d, K, ldk, has_diag, diag, singular, flags, st); break;
    default: launch_assemble_kd<KID, 0>(x, T, y, N, d, K, ldk, has_diag, diag, singular, flags, st); break;
  }
}

bool kernel_singular_at_origin(int id) {  // kernel.hpp:76-89
  return id == HB_K_INVERSE_R || id == HB_K_LOG_R || id == HB_K_HELMHOLTZ3D_RE ||
         id == HB_K_HANKEL_H12_IM;
}

void launch_assemble(const hb_kernel& kern, const double* x, int64_t T, const double* y,
                     int64_t N, int d, double* K, int64_t ldk, unsigned int* flags,
                     cudaStream_t st) {
  const int singular = kernel_singular_at_origin(kern.id);
  const int hd = kern.has_diag != 0;
  const double dg = kern.diag;
  switch (kern.id) {
#define HB_CASE(ID) \
  case ID: launch_assemble_k<ID>(x, T, y, N, d, K, ldk, hd, dg, singular, flags, st); break;
    HB_CASE(HB_K_INVERSE_R)
    HB_CASE(HB_K_LOG_R)
    HB_CASE(HB_K_HELMHOLTZ3D_RE)
    HB_CASE(HB_K_HELMHOLTZ3D_IM)
    HB_CASE(HB_K_HANKEL_H12_RE)
    HB_CASE(HB_K_HANKEL_H12_IM)
    HB_CASE(HB_K_R)
    HB_CASE(HB_K_SIN_R)
    HB_CASE(HB_K_INV_SQRT_1_PLUS_R)
    HB_CASE(HB_K_EXP_NEG_R)
    HB_CASE(HB_K_EXP_NEG_R2)
#undef HB_CASE
    default:
      throw Error(HB_EUNSUPPORTED, "assemble: kernel id " + std::to_string(kern.id) +
                                       " is not available on the device path");
  }
}

}  // namespace hb
