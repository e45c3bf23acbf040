// FP64 GEMM on the sm_100a double-precision tensor path (mma.sync m8n8k4 f64 -> SASS DMMA).
//
// tcgen05 has no f64 kind, so FP64 tensor work on B200 goes through the legacy warp-level
// mma.sync; the probe in tools/fp64_peak.cu measured DMMA = DFMA = 36.9 TF/s on this pool.
// Used for every dense contraction of the rank-reveal: the sketch Y = Ω·A, the compact-WY
// trailing update W = Vᵀ·A2, W ← Tᵀ·W, A2 −= V·W, the sketch downdate Y2 −= Z·R12, and the same
// shapes inside the certification QR.
//
// Tiling: 256 threads (8 warps), CTA tile BM x BN x 16, 3-stage cp.async pipeline, padded
// shared-memory layouts chosen so every fragment load is bank-conflict free:
//   A (N-mode, M x K col-major): As[k][m] with row stride BM+4   (m contiguous)
//   A (T-mode, K x M col-major): As[m][k] with row stride 16+4   (k contiguous)
//   B (K x N col-major):         Bs[n][k] with row stride 16+4   (k contiguous)
// m8n8k4 fragments: a = A[m=lane/4][k=lane%4], b = B[k=lane%4][n=lane/4],
//                   c = C[m=lane/4][n=2*(lane%4)+{0,1}].
// Optional epilogue: per-CTA sum of squares of the updated C below a row offset (the exact
// Frobenius norm of the trailing matrix A22, used by the QR stopping rule), written in a fixed
// order so the result is deterministic.  Split-K (for skinny outputs with a long reduction)
// writes per-slice partials that a second kernel sums in a fixed order.
#include <cstring>
#include <string>

#include "common.cuh"
#include "kernels.h"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace hb {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(unsigned dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(unsigned dst, const void* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct GemmParams {
  int64_t M, N, K;
  double alpha, beta;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  double* partial;  // split-K slices (M x N each, ld = M) or nullptr
  int64_t kchunk;
  double* fro;      // per-CTA Frobenius partials or nullptr
  int64_t fro_row0;
};

template <bool TA, int WARPS_M, int WARPS_N, int WM, int WN, int BK_ = 16, int ST_ = 3>
struct Cfg {
  static constexpr int NT = WARPS_M * WARPS_N * 32;  // threads per CTA
  static constexpr int BM = WARPS_M * WM * 8;
  static constexpr int BN = WARPS_N * WN * 8;
  static constexpr int BK = BK_;
  static constexpr int STAGES = ST_;
  static constexpr int AS = TA ? (BK + 4) : (BM + 4);  // A row stride
  static constexpr int A_ELEMS = TA ? BM * (BK + 4) : BK * (BM + 4);
  static constexpr int B_ELEMS = BN * (BK + 4);
  static constexpr int SMEM = STAGES * (A_ELEMS + B_ELEMS) * 8;
};

template <bool TA, int WARPS_M, int WARPS_N, int WM, int WN, bool VEC, int BK_, int ST_>
__global__ void __launch_bounds__(Cfg<TA, WARPS_M, WARPS_N, WM, WN, BK_, ST_>::NT,
                                  (WM * WN <= 16 && WARPS_M * WARPS_N == 4) ? 3
                                      : (Cfg<TA, WARPS_M, WARPS_N, WM, WN, BK_, ST_>::NT == 128 ? 2 : 1))
    dgemm_kernel(GemmParams p) {
  using C_ = Cfg<TA, WARPS_M, WARPS_N, WM, WN, BK_, ST_>;
  constexpr int BM = C_::BM, BN = C_::BN, BK = C_::BK, STAGES = C_::STAGES, NT = C_::NT;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * C_::A_ELEMS;
  __shared__ double red[32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * p.kchunk;
  const int64_t kend = min(p.K, kbeg + p.kchunk);
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;
  if (p.beta != 0.0 && !p.partial) {
    // warm L2 with this CTA's C tile while the main loop runs (128-byte lines)
    for (int v = tid; v < BN * (BM / 16); v += NT) {
      const int64_t m = m0 + (v % (BM / 16)) * 16, n = n0 + v / (BM / 16);
      if (m < p.M && n < p.N)
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p.C + m + n * p.ldc));
    }
  }

  // ---- tile loader: per-thread source pointers / shared offsets / bound masks are set up
  // once; each k-tile only advances the pointers (the K tail is checked per tile).
  constexpr int VPC = BM / 2;   // N-mode A: 16-byte vectors per k-column of the tile
  constexpr int VPR = BK / 2;   // T-mode A and B: vectors per m/n-row of the tile
  constexpr int A_PT = (TA ? BM * VPR : BK * VPC) / NT;
  constexpr int B_PT = (BN * VPR) / NT;
  static_assert((TA ? BM * VPR : BK * VPC) % NT == 0 && (BN * VPR) % NT == 0, "loader split");
  static_assert(TA ? (NT % VPR == 0) : (NT % VPC == 0), "loader stride");
  // N-mode A: mm fixed, kk_i = kk0 + i*(NT/VPC);  T-mode A / B: kk fixed, row_i = r0 + i*(NT/VPR)
  const int a_kk0 = TA ? (tid % VPR) * 2 : tid / VPC;
  const int a_r0 = TA ? tid / VPR : (tid % VPC) * 2;
  const int b_kk0 = (tid % VPR) * 2, b_r0 = tid / VPR;
  uint32_t a_rowok = 0, b_rowok = 0;  // T-mode: bit i = row i inside M / N
  int a_mbytes = 0;                   // N-mode: bytes valid along m (16 / 8 / 0)
  if (TA) {
#pragma unroll
    for (int i = 0; i < A_PT; ++i)
      if (m0 + a_r0 + i * (NT / VPR) < p.M) a_rowok |= 1u << i;
  } else {
    const int64_t gm = m0 + a_r0;
    a_mbytes = gm + 1 < p.M ? 16 : (gm < p.M ? 8 : 0);
  }
#pragma unroll
  for (int i = 0; i < B_PT; ++i)
    if (n0 + b_r0 + i * (NT / VPR) < p.N) b_rowok |= 1u << i;
  const double* a_ptr = TA ? p.A + (kbeg + a_kk0) + (m0 + a_r0) * p.lda
                           : p.A + (m0 + a_r0) + (kbeg + a_kk0) * p.lda;
  const double* b_ptr = p.B + (kbeg + b_kk0) + (n0 + b_r0) * p.ldb;
  const int64_t a_istride = TA ? (int64_t)(NT / VPR) * p.lda : (int64_t)(NT / VPC) * p.lda;
  const int64_t a_kstride = TA ? (int64_t)BK : (int64_t)BK * p.lda;
  const int64_t b_istride = (int64_t)(NT / VPR) * p.ldb;
  const uint32_t a_dst0 = smem_u32(As) + 8u * (TA ? (a_r0 * (BK + 4) + a_kk0) : (a_kk0 * (BM + 4) + a_r0));
  const uint32_t b_dst0 = smem_u32(Bs) + 8u * (b_r0 * (BK + 4) + b_kk0);
  constexpr uint32_t A_IDST = 8u * (TA ? (NT / VPR) * (BK + 4) : (NT / VPC) * (BM + 4));
  constexpr uint32_t B_IDST = 8u * (NT / VPR) * (BK + 4);

  auto load_tile = [&](int kt, int stage) {
    const int64_t k0 = kbeg + (int64_t)kt * BK;  // tile start
    const bool full_k = k0 + BK <= kend;
    const uint32_t a_st = a_dst0 + 8u * stage * C_::A_ELEMS;
    const uint32_t b_st = b_dst0 + 8u * stage * C_::B_ELEMS;
    const double* ap = a_ptr + kt * a_kstride;
    const double* bp = b_ptr + (int64_t)kt * BK;
    // T-mode / B: the k-extent of this thread's vector (uniform over i)
    const int64_t gk = k0 + (TA ? a_kk0 : 0);
    const int kb_a = full_k ? 16 : (gk + 1 < kend ? 16 : (gk < kend ? 8 : 0));
    const int64_t gkb = k0 + b_kk0;
    const int kb_b = full_k ? 16 : (gkb + 1 < kend ? 16 : (gkb < kend ? 8 : 0));
#pragma unroll
    for (int i = 0; i < A_PT; ++i) {
      const double* src = ap + i * a_istride;
      int bytes;
      if (TA) {
        bytes = ((a_rowok >> i) & 1u) ? kb_a : 0;
      } else {
        const bool kin = full_k || (k0 + a_kk0 + i * (NT / VPC) < kend);
        bytes = kin ? a_mbytes : 0;
      }
      const uint32_t dst = a_st + i * A_IDST;
      if (VEC) {
        cp_async16(dst, bytes ? src : p.A, bytes);
      } else {
        cp_async8(dst, bytes >= 8 ? src : p.A, bytes >= 8 ? 8 : 0);
        cp_async8(dst + 8, bytes >= 16 ? src + 1 : p.A, bytes >= 16 ? 8 : 0);
      }
    }
#pragma unroll
    for (int i = 0; i < B_PT; ++i) {
      const double* src = bp + i * b_istride;
      const int bytes = ((b_rowok >> i) & 1u) ? kb_b : 0;
      const uint32_t dst = b_st + i * B_IDST;
      if (VEC) {
        cp_async16(dst, bytes ? src : p.B, bytes);
      } else {
        cp_async8(dst, bytes >= 8 ? src : p.B, bytes >= 8 ? 8 : 0);
        cp_async8(dst + 8, bytes >= 16 ? src + 1 : p.B, bytes >= 16 ? 8 : 0);
      }
    }
  };

  double acc[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < WN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_tile(s, s);
    cp_commit();
  }
  const int ar = lane >> 2, ac = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      const int pf = kt + STAGES - 1;
      if (pf < nk) load_tile(pf, pf % STAGES);
      cp_commit();
    }
    const double* as = As + (kt % STAGES) * C_::A_ELEMS;
    const double* bs = Bs + (kt % STAGES) * C_::B_ELEMS;
    // one k-step (4 deep) of the warp tile
    auto kstep = [&](int kk) {
      double a[WM], b[WN];
#pragma unroll
      for (int i = 0; i < WM; ++i) {
        const int m = (wm * WM + i) * 8 + ar;
        a[i] = TA ? as[m * (BK + 4) + kk + ac] : as[(kk + ac) * (BM + 4) + m];
      }
#pragma unroll
      for (int j = 0; j < WN; ++j) {
        const int n = (wn * WN + j) * 8 + ar;
        b[j] = bs[n * (BK + 4) + kk + ac];
      }
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int j = 0; j < WN; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    };
    const int64_t krem = kend - kbeg - (int64_t)kt * BK;
    if (krem >= BK) {
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) kstep(kk);
    } else {
      // K tail: the last k-tile runs only its valid k-steps (the rest of the tile is zero-filled;
      // at K = b = 120, BK = 32 that saves 2 of the update's 32 k-steps), in a rolled loop so the
      // unrolled body above stays as it was
      const int kk_end = (int)((krem + 3) & ~(int64_t)3);
#pragma unroll 1
      for (int kk = 0; kk < kk_end; kk += 4) kstep(kk);
    }
  }
  cp_wait<0>();

  if (p.partial) {
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      const int64_t m = m0 + (wm * WM + i) * 8 + ar;
      if (m >= p.M) continue;
#pragma unroll
      for (int j = 0; j < WN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t n = n0 + (wn * WN + j) * 8 + 2 * ac + h;
          if (n < p.N) p.partial[(int64_t)blockIdx.z * p.M * p.N + m + n * p.M] = p.alpha * acc[i][j][h];
        }
    }
    return;
  }
  // Epilogue: stage the accumulator tile through shared memory (the operand buffers are free
  // now), half a tile of columns at a time, then read-modify-write C with 16-byte accesses and
  // all loads of a thread in flight together.  LDC = BM + 2 keeps the fragment stores
  // bank-conflict free.
  constexpr int LDC = BM + 2;
  constexpr int HALF = BN / 2;
  static_assert(HALF * LDC <= STAGES * (C_::A_ELEMS + C_::B_ELEMS), "epilogue tile too large");
  double* Cs = smem;
  double fro = 0.0;
  const bool cvec = ((p.ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(p.C) & 15) == 0);
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < WM; ++i)
#pragma unroll
      for (int j = 0; j < WN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int nl = (wn * WN + j) * 8 + 2 * ac + h - half * HALF;
          if (nl >= 0 && nl < HALF) Cs[nl * LDC + (wm * WM + i) * 8 + ar] = acc[i][j][h];
        }
    __syncthreads();
    constexpr int VPC = BM / 2;                 // 2-double vectors per column
    constexpr int PER = VPC * HALF / NT;        // vectors per thread
    double2 cv[PER];
    if (p.beta != 0.0) {
#pragma unroll
      for (int t = 0; t < PER; ++t) {
        const int v = tid + t * NT;
        const int ml = (v % VPC) * 2, nl = v / VPC;
        const int64_t m = m0 + ml, n = n0 + half * HALF + nl;
        cv[t] = make_double2(0.0, 0.0);
        if (n < p.N) {
          const double* c = p.C + m + n * p.ldc;
          if (cvec && m + 1 < p.M) cv[t] = *reinterpret_cast<const double2*>(c);
          else {
            if (m < p.M) cv[t].x = c[0];
            if (m + 1 < p.M) cv[t].y = c[1];
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int v = tid + t * NT;
      const int ml = (v % VPC) * 2, nl = v / VPC;
      const int64_t m = m0 + ml, n = n0 + half * HALF + nl;
      if (n >= p.N || m >= p.M) continue;
      double2 o;
      o.x = p.alpha * Cs[nl * LDC + ml];
      o.y = p.alpha * Cs[nl * LDC + ml + 1];
      if (p.beta != 0.0) {
        o.x += p.beta * cv[t].x;
        o.y += p.beta * cv[t].y;
      }
      double* c = p.C + m + n * p.ldc;
      if (cvec && m + 1 < p.M) {
        *reinterpret_cast<double2*>(c) = o;
      } else {
        c[0] = o.x;
        if (m + 1 < p.M) c[1] = o.y;
      }
      if (m >= p.fro_row0) fro += o.x * o.x;
      if (m + 1 >= p.fro_row0 && m + 1 < p.M) fro += o.y * o.y;
    }
  }
  if (p.fro) {
    const double s = block_sum(fro, red);
    if (tid == 0) p.fro[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}

// Split-K finish: C = sum_z P[z] + beta*C (fixed order), optional Frobenius partials.
__global__ void splitk_reduce(GemmParams p, int slices) {
  __shared__ double red[32];
  const int64_t total = p.M * p.N;
  double fro = 0.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = idx % p.M, n = idx / p.M;
    double s = 0.0;
    for (int z = 0; z < slices; ++z) s += p.partial[(int64_t)z * total + idx];
    double* c = p.C + m + n * p.ldc;
    const double out = p.beta == 0.0 ? s : s + p.beta * *c;
    *c = out;
    if (m >= p.fro_row0) fro += out * out;
  }
  if (p.fro) {
    const double s = block_sum(fro, red);
    if (threadIdx.x == 0) p.fro[blockIdx.x] = s;
  }
}

template <bool TA, int WARPS_M, int WARPS_N, int WM, int WN, int BK_ = 16, int ST_ = 3>
static void run_cfg(const GemmParams& p, int slices, bool vec, cudaStream_t st) {
  using C_ = Cfg<TA, WARPS_M, WARPS_N, WM, WN, BK_, ST_>;
  dim3 grid((unsigned)ceil_div(p.M, C_::BM), (unsigned)ceil_div(p.N, C_::BN), (unsigned)slices);
  HB_REQUIRE(grid.y <= 65535u && grid.z <= 65535u, HB_ECAP, "dgemm: grid too large");
  if (vec) {
    auto k = dgemm_kernel<TA, WARPS_M, WARPS_N, WM, WN, true, BK_, ST_>;
    ensure_dyn_smem((const void*)k, C_::SMEM);
    k<<<grid, C_::NT, C_::SMEM, st>>>(p);
  } else {
    auto k = dgemm_kernel<TA, WARPS_M, WARPS_N, WM, WN, false, BK_, ST_>;
    ensure_dyn_smem((const void*)k, C_::SMEM);
    k<<<grid, C_::NT, C_::SMEM, st>>>(p);
  }
  HB_LAUNCH_CHECK();
}

static constexpr int kReduceBlocks = 592;  // 4 x 148 SMs

// Kernel variant for a shape (HB_GEMM_VAR overrides, for A/B experiments):
//   4 (default): 64x64 tiles, 4 warps (32x32 warp tiles), BK 32, 2 stages, 3 CTAs/SM — fastest on
//      every rank-reveal shape measured (tools/gemm_bench.py: 8192^3 34.6 TF/s, rank-120 update
//      26.1, Vᵀ·A2 31.4, Ω·A 33.9 of the 36.9 TF/s DMMA peak);
//   2: 128x64 tiles, 2 CTAs/SM;  100: 64x128 tiles, 8 warps (small M)
static int gemm_variant(int64_t M, int64_t N, int64_t K) {
  static const int env = [] {
    const char* e = getenv("HB_GEMM_VAR");
    return e ? atoi(e) : -1;
  }();
  (void)N; (void)K;
  if (env >= 0) return (M <= 64 && env != 4 && env != 100) ? 100 : env;
  return 4;
}
static int64_t tiles_of(int64_t M, int64_t N, int64_t K) {
  const int v = gemm_variant(M, N, K);
  const int bm = v == 100 ? 64 : (v == 4 ? 64 : (v == 3 ? 64 : 128));
  const int bn = v == 100 ? 128 : (v == 4 ? 64 : (v == 3 ? 128 : 64));
  return ceil_div(M, bm) * ceil_div(N, bn);
}

// Split-K count from a wave model: a 64x64 tile costs ~kTileKNs per k at 3 CTAs/SM, a grid of
// `tiles * s` CTAs runs in ceil(tiles * s / (3 * SMs)) waves of K/s each, and the split adds one
// pass over (s + 1) M x N partials.  Skinny-M, long-K shapes (Ω·A, Vᵀ·A2 with M <= 128) have only
// ~1.1 waves of tiles and gain ~1.6x from it.
static int choose_slices(int64_t M, int64_t N, int64_t K, int num_sms, int64_t ws_elems) {
  const int64_t tiles = tiles_of(M, N, K);
  const int64_t slots = 3ll * num_sms;
  if (K < 1024 || tiles >= 8 * slots) return 1;
  constexpr double kTileKNs = 98.6;         // 2*64*64 flop / (36.9 TF/s / 148 / 3)
  constexpr double kBytesPerNs = 5000.0;    // ~HBM rate for the partial pass
  constexpr double kReduceLaunchNs = 5000.0;
  double best_t = (double)ceil_div(tiles, slots) * K * kTileKNs;
  int best = 1;
  for (int s = 2; s <= 32; ++s) {
    if (K / s < 256 || (int64_t)s * M * N > ws_elems) break;
    const int64_t kc = round_up(ceil_div(K, s), 16);
    const int64_t se = ceil_div(K, kc);
    const double t = (double)ceil_div(tiles * se, slots) * kc * kTileKNs +
                     (double)(se + 1) * M * N * 8.0 / kBytesPerNs + kReduceLaunchNs;
    if (t < 0.97 * best_t) { best_t = t; best = s; }
  }
  return best;
}

// TMA-fed persistent-strip kernel for the NN shapes (dgemm_tma.cu)
bool tma_gemm_eligible(const GemmArgs& g);
int64_t tma_gemm_fro_count(int64_t M, int64_t N, int num_sms);
void launch_dgemm_tma(const GemmArgs& g, int num_sms, cudaStream_t st);

// Frobenius partial slots a GEMM of this shape may write (either kernel); unused ones are zeroed.
int64_t gemm_fro_count(int64_t M, int64_t N, int64_t K, int num_sms) {
  const int64_t a = std::max<int64_t>(tiles_of(M, N, K), (int64_t)kReduceBlocks);
  return std::max<int64_t>(a, tma_gemm_fro_count(M, N, num_sms));
}

// HB_GEMM_CHECK=1 (diagnostics): every TMA-routed GEMM is re-run by the cp.async kernel on a copy
// of C and the two results (and Frobenius sums) are compared on the host.
__global__ void gemm_check_diff(const double* C, int64_t ldc, const double* D, int64_t M, int64_t N,
                                double* out) {
  double mx = 0.0, ref = 0.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < M * N;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = idx % M, n = idx / M;
    const double a = C[m + n * ldc], b = D[idx];
    mx = fmax(mx, fabs(a - b));
    ref = fmax(ref, fabs(b));
  }
  atomicMax(reinterpret_cast<unsigned long long*>(out), __double_as_longlong(mx));
  atomicMax(reinterpret_cast<unsigned long long*>(out + 1), __double_as_longlong(ref));
}

static void launch_dgemm_cpasync(const GemmArgs& g, double* ws, int64_t ws_elems, int num_sms, cudaStream_t st);
int tma_gemm_strip(int64_t M, int64_t N, int num_sms);

// Diagnostics of a flagged update: the first bad elements with the three 40-deep chunk products
// of their own column and of the same column of the neighbouring tiles (c -+ 64), to tell a stale
// or missing ring chunk from a wrong C value.  out: [0] = count, then 12 doubles per element.
__global__ void gemm_check_diag(const double* C, int64_t ldc, const double* D, int64_t M, int64_t N,
                                const double* A, int64_t lda, const double* B, int64_t ldb, int64_t K,
                                double tol, double* out, int max_out, unsigned long long* hist) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < M * N;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = idx % M, n = idx / M;
    const double a = C[m + n * ldc], b = D[idx];
    if (!(fabs(a - b) <= tol)) {
      atomicAdd(&hist[m % 128], 1ull);          // row inside the m-block
      atomicAdd(&hist[128 + n % 64], 1ull);     // column inside the tile
      const int slot = (int)atomicAdd(reinterpret_cast<unsigned long long*>(out), 1ull);
      if (slot < max_out) {
        double* o = out + 1 + slot * 12;
        o[0] = (double)m; o[1] = (double)n; o[2] = a - b;
        for (int w = 0; w < 3; ++w) {
          const int64_t nn = n + (w - 1) * 64;
          for (int ch = 0; ch < 3; ++ch) {
            double s = 0.0;
            if (nn >= 0 && nn < N)
              for (int64_t k = ch * 40; k < min((int64_t)(ch + 1) * 40, K); ++k) s += A[m + k * lda] * B[k + nn * ldb];
            o[3 + w * 3 + ch] = s;
          }
        }
      }
    }
  }
}

static void checked_tma(const GemmArgs& g, double* ws, int64_t ws_elems, int num_sms, cudaStream_t st) {
  double *D = nullptr, *F = nullptr, *out = nullptr;
  const int64_t cnt = gemm_fro_count(g.M, g.N, g.K, num_sms);
  HB_CUDA(cudaMallocAsync(&D, sizeof(double) * g.M * g.N, st));
  HB_CUDA(cudaMallocAsync(&F, sizeof(double) * (cnt + 2), st));
  HB_CUDA(cudaMallocAsync(&out, sizeof(double) * 4, st));
  HB_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * 4, st));
  HB_CUDA(cudaMemcpy2DAsync(D, g.M * 8, g.C, g.ldc * 8, g.M * 8, g.N, cudaMemcpyDeviceToDevice, st));
  GemmArgs r = g;
  r.C = D;
  r.ldc = g.M;
  r.fro_partials = g.fro_partials ? F : nullptr;
  // control (HB_GEMM_CHECK=2): the primary run is the cp.async kernel too, so any flag then comes
  // from the check itself or from operands changing under it, not from the TMA kernel
  static const bool control = atoi(getenv("HB_GEMM_CHECK")) == 2;
  if (control) launch_dgemm_cpasync(g, ws, ws_elems, num_sms, st);
  else launch_dgemm_tma(g, num_sms, st);
  launch_dgemm_cpasync(r, ws, ws_elems, num_sms, st);
  gemm_check_diff<<<296, 256, 0, st>>>(g.C, g.ldc, D, g.M, g.N, out);
  std::vector<double> hp(cnt), hq(cnt);
  double h[2];
  HB_CUDA(cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, st));
  if (g.fro_partials) {
    const int64_t written = tma_gemm_fro_count(g.M, g.N, num_sms);
    HB_CUDA(cudaMemcpyAsync(hp.data(), g.fro_partials, sizeof(double) * written, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaMemcpyAsync(hq.data(), F, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    double a = 0, b = 0;
    for (int64_t i = 0; i < written; ++i) a += hp[(size_t)i];
    for (int64_t i = 0; i < cnt; ++i) b += hq[(size_t)i];
    if (!(std::fabs(a - b) <= 1e-12 * std::fabs(b)))
      fprintf(stderr, "[gemm check] FRO M=%lld N=%lld K=%lld: tma %.17g ref %.17g\n", (long long)g.M,
              (long long)g.N, (long long)g.K, a, b);
  }
  HB_CUDA(cudaStreamSynchronize(st));
  if (!(h[0] <= 1e-13 * h[1])) {
    fprintf(stderr, "[gemm check] C M=%lld N=%lld K=%lld lda=%lld ldb=%lld ldc=%lld A=%p B=%p C=%p: maxdiff %.3g ref %.3g\n",
            (long long)g.M, (long long)g.N, (long long)g.K, (long long)g.lda, (long long)g.ldb,
            (long long)g.ldc, (const void*)g.A, (const void*)g.B, (void*)g.C, h[0], h[1]);
    constexpr int kMax = 6;
    double* dg = nullptr;
    unsigned long long* hist = nullptr;
    HB_CUDA(cudaMallocAsync(&dg, sizeof(double) * (1 + 12 * kMax), st));
    HB_CUDA(cudaMallocAsync(&hist, sizeof(unsigned long long) * 192, st));
    HB_CUDA(cudaMemsetAsync(dg, 0, sizeof(double) * (1 + 12 * kMax), st));
    HB_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * 192, st));
    gemm_check_diag<<<296, 256, 0, st>>>(g.C, g.ldc, D, g.M, g.N, g.A, g.lda, g.B, g.ldb, g.K,
                                         1e-13 * h[1], dg, kMax, hist);
    double hd[1 + 12 * kMax];
    unsigned long long hh[192];
    HB_CUDA(cudaMemcpyAsync(hd, dg, sizeof(hd), cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaMemcpyAsync(hh, hist, sizeof(hh), cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    unsigned long long cnt_bad;
    memcpy(&cnt_bad, &hd[0], 8);
    const int strip = tma_gemm_strip(g.M, g.N, num_sms);
    std::string line = "[gemm diag] bad " + std::to_string(cnt_bad) + " strip " + std::to_string(strip) +
                       " mblocks " + std::to_string((g.M + 127) / 128) + " rows%128:";
    for (int i = 0; i < 128; ++i) if (hh[i]) line += " " + std::to_string(i) + "x" + std::to_string(hh[i]);
    line += " cols%64:";
    for (int i = 0; i < 64; ++i) if (hh[128 + i]) line += " " + std::to_string(i) + "x" + std::to_string(hh[128 + i]);
    fprintf(stderr, "%s\n", line.c_str());
    for (int e = 0; e < (int)std::min<unsigned long long>(cnt_bad, kMax); ++e) {
      const double* o = hd + 1 + e * 12;
      fprintf(stderr, "[gemm diag]  r=%lld (mb %lld, row %lld) c=%lld (tile %lld, in-strip %lld, col %lld): got-want %+.4e; "
              "chunk products own %+.4e %+.4e %+.4e | c-64 %+.4e %+.4e %+.4e | c+64 %+.4e %+.4e %+.4e\n",
              (long long)o[0], (long long)o[0] / 128, (long long)o[0] % 128, (long long)o[1],
              (long long)o[1] / 64, ((long long)o[1] / 64) % strip, (long long)o[1] % 64, o[2], o[6], o[7], o[8],
              o[3], o[4], o[5], o[9], o[10], o[11]);
    }
    HB_CUDA(cudaFreeAsync(dg, st));
    HB_CUDA(cudaFreeAsync(hist, st));
  }
  // the caller's C must hold the TMA result (already there); the check buffers go back
  HB_CUDA(cudaFreeAsync(D, st));
  HB_CUDA(cudaFreeAsync(F, st));
  HB_CUDA(cudaFreeAsync(out, st));
}

void launch_dgemm(const GemmArgs& g, double* ws, int64_t ws_elems, int num_sms, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return;
  static const bool check = getenv("HB_GEMM_CHECK") != nullptr;
  if (tma_gemm_eligible(g)) {
    if (check) {
      checked_tma(g, ws, ws_elems, num_sms, st);
      if (g.fro_partials && atoi(getenv("HB_GEMM_CHECK")) != 2) {
        const int64_t written = tma_gemm_fro_count(g.M, g.N, num_sms);
        const int64_t cnt = gemm_fro_count(g.M, g.N, g.K, num_sms);
        if (cnt > written)
          HB_CUDA(cudaMemsetAsync(g.fro_partials + written, 0, (cnt - written) * sizeof(double), st));
      }
      return;
    }
    launch_dgemm_tma(g, num_sms, st);
    if (g.fro_partials) {
      const int64_t written = tma_gemm_fro_count(g.M, g.N, num_sms);
      const int64_t cnt = gemm_fro_count(g.M, g.N, g.K, num_sms);
      if (cnt > written)
        HB_CUDA(cudaMemsetAsync(g.fro_partials + written, 0, (cnt - written) * sizeof(double), st));
    }
    return;
  }
  launch_dgemm_cpasync(g, ws, ws_elems, num_sms, st);
}

// The cp.async DMMA kernel (every shape; the product path for the trailing update too).
static void launch_dgemm_cpasync(const GemmArgs& g, double* ws, int64_t ws_elems, int num_sms, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return;
  GemmParams p{};
  p.M = g.M; p.N = g.N; p.K = g.K;
  p.alpha = g.alpha; p.beta = g.beta;
  p.A = g.A; p.lda = g.lda; p.B = g.B; p.ldb = g.ldb; p.C = g.C; p.ldc = g.ldc;
  p.fro = g.fro_partials; p.fro_row0 = g.fro_row0;
  if (g.K <= 0) {  // C = beta*C
    p.partial = nullptr;
    p.kchunk = 1;
  }
  const bool vec = (g.lda % 2 == 0) && (g.ldb % 2 == 0) &&
                   ((reinterpret_cast<uintptr_t>(g.A) | reinterpret_cast<uintptr_t>(g.B)) & 15) == 0;
  const int slices = g.K > 0 ? choose_slices(g.M, g.N, g.K, num_sms, ws ? ws_elems : 0) : 1;
  p.kchunk = slices > 1 ? round_up(ceil_div(g.K, slices), 16) : std::max<int64_t>(g.K, 1);
  const int s_eff = slices > 1 ? (int)ceil_div(g.K, p.kchunk) : 1;
  GemmParams q = p;
  if (s_eff > 1) {
    q.partial = ws;
    q.fro = nullptr;
  }
  const int var = gemm_variant(g.M, g.N, g.K);
  if (var == 100) {
    if (g.transA) run_cfg<true, 1, 8, 8, 2>(q, s_eff, vec, st);
    else run_cfg<false, 1, 8, 8, 2>(q, s_eff, vec, st);
  } else if (var == 4) {
    if (g.transA) run_cfg<true, 2, 2, 4, 4, 32, 2>(q, s_eff, vec, st);
    else run_cfg<false, 2, 2, 4, 4, 32, 2>(q, s_eff, vec, st);
  } else if (var == 3) {
    if (g.transA) run_cfg<true, 2, 2, 4, 8, 16, 3>(q, s_eff, vec, st);
    else run_cfg<false, 2, 2, 4, 8, 16, 3>(q, s_eff, vec, st);
  } else if (var == 0) {
    if (g.transA) run_cfg<true, 2, 2, 8, 4, 16, 3>(q, s_eff, vec, st);
    else run_cfg<false, 2, 2, 8, 4, 16, 3>(q, s_eff, vec, st);
  } else {
    // 128x64 tiles, 4 warps, BK 32, 2 stages, 2 CTAs per SM: one CTA's epilogue (C read-modify-
    // write) overlaps the other's DMMA main loop (measured fastest on the rank-reveal shapes)
    if (g.transA) run_cfg<true, 2, 2, 8, 4, 32, 2>(q, s_eff, vec, st);
    else run_cfg<false, 2, 2, 8, 4, 32, 2>(q, s_eff, vec, st);
  }
  if (s_eff > 1) {
    p.partial = ws;
    splitk_reduce<<<kReduceBlocks, 256, 0, st>>>(p, s_eff);
    HB_LAUNCH_CHECK();
    const int64_t cnt = gemm_fro_count(g.M, g.N, g.K, num_sms);
    if (g.fro_partials && cnt > kReduceBlocks)
      HB_CUDA(cudaMemsetAsync(g.fro_partials + kReduceBlocks, 0, (cnt - kReduceBlocks) * sizeof(double), st));
  } else if (g.fro_partials) {
    // pad the partial array to the fixed count with zeros so the consumer can always sum
    // gemm_fro_count(M, N) entries
    const int64_t written = tiles_of(g.M, g.N, g.K);
    const int64_t cnt = gemm_fro_count(g.M, g.N, g.K, num_sms);
    if (cnt > written)
      HB_CUDA(cudaMemsetAsync(g.fro_partials + written, 0, (cnt - written) * sizeof(double), st));
  }
}

}  // namespace hb
