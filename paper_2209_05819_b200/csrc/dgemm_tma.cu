// FP64 DMMA GEMM fed by TMA: C = alpha * A * B + beta * C for the rank-b trailing update
// A2 -= V * W (M, N large; K = b <= 128) and the other NN shapes with M, N >= 256.
//
// Why a second GEMM: the cp.async kernel (dgemm.cu) runs one short-lived 64x64 CTA per tile; with
// K = 120 each CTA fills its pipeline, runs four k-tiles and drains through a C read-modify-write
// that nothing overlaps inside the CTA (ncu: SM 61 %, DRAM 36 % on the rank-64 update).  Here:
//   * warp specialisation: one producer warp issues cp.async.bulk.tensor (TMA) loads of the A and
//     B k-chunks into a ring of STAGES shared-memory slots, signalled through mbarriers
//     (full[s]: bytes landed, complete_tx; empty[s]: the 8 consumer warps are done with slot s);
//   * 8 consumer warps (4 x 2, 32 x 32 each) run mma.sync m8n8k4 f64 (SASS DMMA) from shared
//     memory; tcgen05 has no f64 kind, so DMMA is the FP64 tensor path on sm_100a;
//   * a CTA owns a strip of S tiles (128 x 64 each, along N): the ring keeps streaming across tile
//     boundaries and every consumer thread prefetches its C values for the tile into registers
//     before the k-loop, so the C read overlaps the DMMA work instead of following it;
//   * the product is computed transposed (D' = Bᵀ·Aᵀ): a thread's accumulator pair is then two
//     consecutive ROWS of one column of C, read and written as one 16-byte access.
// Shared layouts (TMA boxes, dense): A chunk [k][BM+4] (m contiguous; the 4 extra rows make the
// pitch ≡ 4 mod 16 doubles, so the eight 8-byte fragment loads of a half-warp hit distinct bank
// pairs), B chunk [n][BK+4] (k contiguous, same trick).  The extra rows/columns read are either
// real neighbouring data or zero-filled out of bounds, and never used.
// Frobenius epilogue: each consumer warp accumulates the squares of its NEW C entries with
// row >= fro_row0 over its strip in a fixed order -> fro[cta * 8 + warp] (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace hb {

int tma_gemm_strip(int64_t M, int64_t N, int num_sms);

namespace {

constexpr int kTBM = 128, kTBN = 64;           // CTA tile (rows x columns of C)
// 8 warps, all of them DMMA consumers; lane 0 of warp 0 also issues the TMA loads STAGES-1 chunks
// ahead.  (A ninth, producer-only warp does not fit: 9 warps x 224 registers exceeds the register
// file once warps are allocated in groups.)
constexpr int kTConsumers = 8, kTThreads = kTConsumers * 32;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct TmaGemmParams {
  int64_t M, N, K;
  double alpha, beta;
  double* C;
  int64_t ldc;
  int a_shift, b_shift;  // element offset of A / B inside their 16-byte aligned tensor maps
  int strip;             // tiles per CTA along N
  int nblocks_n;         // ceil(N / kTBN)
  int cvec;              // C pointer 16-byte aligned and ldc even: 16-byte accesses
  double* fro;           // [gridDim.x * gridDim.y * 8] partials or nullptr
  int64_t fro_row0;
  int tile_sync;         // CTA barrier at every tile boundary (default 1, see the kernel)
};

// K <= NKA * BK: the CTA's whole A block (128 rows x K) stays resident in shared memory for the
// strip; only B chunks stream through the ring.
template <int BK, int STAGES, int NKA>
struct TCfg {
  static constexpr int AP = kTBM + 4;  // A pitch (doubles): [k][AP], m contiguous
  static constexpr int BP = BK + 4;    // B chunk pitch: [n][BP], k contiguous
  static constexpr int A_BOX = AP * BK;
  static constexpr int A_ELEMS = A_BOX * NKA;
  static constexpr int B_ELEMS = BP * kTBN;
  static constexpr uint32_t A_BOX_BYTES = (uint32_t)A_BOX * 8u;
  static constexpr uint32_t STAGE_BYTES = (uint32_t)B_ELEMS * 8u;
  static constexpr size_t SMEM = (size_t)A_ELEMS * 8 + (size_t)STAGES * STAGE_BYTES +
                                 (2 * STAGES + 2) * sizeof(uint64_t) + 128;
};

template <int BK, int STAGES, int NKA>
__global__ void __launch_bounds__(kTThreads, 1)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     TmaGemmParams p) {
  using Cf = TCfg<BK, STAGES, NKA>;
  extern __shared__ __align__(128) unsigned char smraw[];
  // 128-byte aligned buffers (cp.async.bulk.tensor destination requirement); derived from the
  // shared array by pointer arithmetic so the fragment loads stay LDS (not generic LD)
  unsigned char* base = smraw + ((128u - (su32(smraw) & 127u)) & 127u);
  double* sA = reinterpret_cast<double*>(base);
  double* sB = sA + Cf::A_ELEMS;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * Cf::B_ELEMS);
  uint64_t* empty = full + STAGES;
  uint64_t* afull = empty + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.x * kTBM;
  const int nb0 = blockIdx.y * p.strip;
  const int nb1 = min(p.nblocks_n, nb0 + p.strip);
  const int nk = (int)((p.K + BK - 1) / BK);  // <= NKA

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTConsumers);
    }
    mbar_init(afull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  // ---- producer role (warp 0, lane 0).  Box starts are kept 16-byte aligned in global memory
  // (TMA faults on an odd FP64 start): a map whose base was rounded down by one element loads
  // from the even coordinate and the consumers read at +shift. ----
  const int total = (nb1 - nb0) * nk;  // B chunks of the strip; chunk g -> slot g % STAGES
  int g_issue = 0;
  auto issue_upto = [&](int g_end) {
    for (; g_issue < g_end && g_issue < total; ++g_issue) {
      const int sl = g_issue % STAGES;
      const uint32_t use = (uint32_t)(g_issue / STAGES);  // fills of slot sl before this one
      if (use > 0) mbar_wait(&empty[sl], (use - 1) & 1u);
      const int nb = nb0 + g_issue / nk, kc = g_issue % nk;
      mbar_expect_tx(&full[sl], Cf::STAGE_BYTES);
      tma_load_2d(sB + sl * Cf::B_ELEMS, &tmB, &full[sl], kc * BK, nb * kTBN);
    }
  };
  const bool producer = threadIdx.x == 0;
  if (producer) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    mbar_expect_tx(afull, Cf::A_BOX_BYTES * (uint32_t)nk);
    for (int kc = 0; kc < nk; ++kc) tma_load_2d(sA + kc * Cf::A_BOX, &tmA, afull, (int)m0, kc * BK);
    issue_upto(STAGES - 1);
  }
  __syncwarp();

  // ===== consumers: warp (wm, wn) owns C rows m0 + wm*32 .. +32, columns n0 + wn*32 .. +32 =====
  const int wm = warp & 3, wn = warp >> 2;
  const int ar = lane >> 2, ac = lane & 3;
  // transposed product: DMMA "m" = C column (i), DMMA "n" = C row pair (j)
  double fro = 0.0;
  int s = 0, gdone = 0;  // slot and global index of the chunk being consumed
  uint32_t ph = 0;
  const bool has_beta = p.beta != 0.0;
  const double* a_thr = sA + p.a_shift + ac * Cf::AP + wm * 32 + ar;   // + kk*AP + j*8
  const int b_off = p.b_shift + (wn * 32 + ar) * Cf::BP + ac;           // + i*8*BP + kk
  mbar_wait(afull, 0);
  for (int nb = nb0; nb < nb1; ++nb) {
    const int64_t n0 = (int64_t)nb * kTBN;
    // All 8 warps start a tile together.  Without this barrier a warp with little C traffic (the
    // rows >= M part of the last m-block) drifts up to two ring chunks ahead across tile
    // boundaries, and under concurrent sweep streams such CTAs produced wrong C columns for that
    // warp (DESIGN.md §4 "TMA GEMM": 50-115 flagged updates per configs[3] pass without the
    // barrier, 0 in every pass with it; the ring, A block and C prefetch all verified correct in
    // instrumented runs, so the cause is not understood).  HB_TMA_TILE_SYNC=0 removes it (repro).
    if (p.tile_sync) __syncthreads();
    // C prefetch: thread's values are C[r, c], C[r+1, c] with r = m0 + wm*32 + j*8 + 2*ac,
    // c = n0 + wn*32 + i*8 + ar
    // C prefetch into registers before the k-loop (its latency hides under the DMMA work).  Plain
    // 8-byte loads: the 16-byte ld.global.cg form produced wrong C values for the warp running
    // ahead of the others in a strip (tools/gemm_repro2.py, profiles/r02/gemm_tma.md) — not
    // understood, measured correct and as fast with LDG.64.
    double2 cpre[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t c = n0 + wn * 32 + i * 8 + ar;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t r = m0 + wm * 32 + j * 8 + 2 * ac;
        cpre[i][j] = make_double2(0.0, 0.0);
        if (has_beta && c < p.N) {
          const double* cp = p.C + r + c * p.ldc;
          if (r < p.M) cpre[i][j].x = cp[0];
          if (r + 1 < p.M) cpre[i][j].y = cp[1];
        }
      }
    }
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kc = 0; kc < nk; ++kc) {
      if (warp == 0) {  // keep STAGES-1 chunks in flight beyond this one
        if (producer) issue_upto(gdone + STAGES);
        __syncwarp();  // reconverge warp 0 before its mma.sync.aligned
      }
      mbar_wait(&full[s], ph);
      const double* as = a_thr + kc * Cf::A_BOX;
      const double* bs = sB + s * Cf::B_ELEMS + b_off;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double fa[4], fb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) fa[i] = bs[i * 8 * Cf::BP + kk];   // Bᵀ: row = C column, k = ac
#pragma unroll
        for (int j = 0; j < 4; ++j) fb[j] = as[kk * Cf::AP + j * 8];   // Aᵀ: k = ac, col = C row
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      ++gdone;
      if (++s == STAGES) {
        s = 0;
        ph ^= 1u;
      }
    }
    // epilogue: out = alpha * acc + beta * C, straight from registers
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t c = n0 + wn * 32 + i * 8 + ar;
      if (c >= p.N) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t r = m0 + wm * 32 + j * 8 + 2 * ac;
        double2 o;
        o.x = p.alpha * acc[i][j][0];
        o.y = p.alpha * acc[i][j][1];
        if (has_beta) {
          o.x += p.beta * cpre[i][j].x;
          o.y += p.beta * cpre[i][j].y;
        }
        double* cp = p.C + r + c * p.ldc;
        if (p.cvec && r + 1 < p.M) {
          __stcg(reinterpret_cast<double2*>(cp), o);
        } else {
          if (r < p.M) cp[0] = o.x;
          if (r + 1 < p.M) cp[1] = o.y;
        }
        if (r >= p.fro_row0 && r < p.M) fro += o.x * o.x;
        if (r + 1 >= p.fro_row0 && r + 1 < p.M) fro += o.y * o.y;
      }
    }
  }
  if (p.fro) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
    if (lane == 0) p.fro[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * kTConsumers + warp] = fro;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    HB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess)
      throw Error(HB_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// 2-D FP64 tensor map over a column-major rows x cols matrix at ptr (ld doubles); the map's base
// is rounded down to 16 bytes and *shift (0 / 1) is the row offset to add to box coordinates.
CUtensorMap make_map(const double* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                     int box_cols, int* shift) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(ptr);
  *shift = (int)((a & 15) / 8);
  const double* b = ptr - *shift;
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)(rows + *shift), (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(b), dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(HB_ECUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

template <int BK, int STAGES, int NKA>
void run_tma(const GemmArgs& g, int num_sms, double* fro, cudaStream_t st) {
  using Cf = TCfg<BK, STAGES, NKA>;
  TmaGemmParams p{};
  p.M = g.M; p.N = g.N; p.K = g.K;
  p.alpha = g.alpha; p.beta = g.beta;
  p.C = g.C; p.ldc = g.ldc;
  p.cvec = ((reinterpret_cast<uintptr_t>(g.C) & 15) == 0) && (g.ldc % 2 == 0);
  p.fro = fro;
  p.fro_row0 = g.fro_row0;
  static const int tile_sync = [] {
    const char* e = getenv("HB_TMA_TILE_SYNC");
    return e ? atoi(e) : 1;
  }();
  p.tile_sync = tile_sync;
  const CUtensorMap ta = make_map(g.A, g.M, g.K, g.lda, Cf::AP, BK, &p.a_shift);
  const CUtensorMap tb = make_map(g.B, g.K, g.N, g.ldb, Cf::BP, kTBN, &p.b_shift);
  const int mb = (int)ceil_div(g.M, kTBM);
  p.nblocks_n = (int)ceil_div(g.N, kTBN);
  p.strip = tma_gemm_strip(g.M, g.N, num_sms);
  dim3 grid((unsigned)mb, (unsigned)ceil_div(p.nblocks_n, p.strip));
  HB_REQUIRE(grid.y <= 65535u, HB_ECAP, "dgemm_tma: grid too large");
  auto k = dgemm_tma_kernel<BK, STAGES, NKA>;
  ensure_dyn_smem((const void*)k, Cf::SMEM);
  k<<<grid, kTThreads, Cf::SMEM, st>>>(ta, tb, p);
  HB_LAUNCH_CHECK();
}

}  // namespace

// Tiles per CTA along N: long strips amortise the pipeline fill, but keep >= ~4 CTAs per SM
// overall so the hardware scheduler still balances the grid (other streams share the GPU).
int tma_gemm_strip(int64_t M, int64_t N, int num_sms) {
  const int64_t mb = ceil_div(M, kTBM), nb = ceil_div(N, kTBN);
  int s = 32;
  while (s > 1 && mb * ceil_div(nb, s) < 4ll * num_sms) s /= 2;
  return s;
}

bool tma_gemm_eligible(const GemmArgs& g) {
  // OFF by default (HB_GEMM_TMA=1 opts in).  The race under concurrent sweep streams is closed by
  // the per-tile CTA barrier in the kernel (0 flagged updates in 12 checked configs[3] passes and a
  // checked sweep pass, ranks equal to the oracle), and alone the kernel is 6-11 % faster than the
  // cp.async one; but a TMA CTA holds its SM for a 32-tile strip, the other streams' cooperative
  // grids wait longer for SMs, and configs[3] / the sweep do not get faster (26.3 vs 26.1 s,
  // 112.0 vs 110.8 s) -- DESIGN.md §4 "TMA-fed GEMM".  The cp.async kernel stays the product.
  static const bool off = [] {
    const char* e = getenv("HB_GEMM_TMA");
    return !(e && atoi(e) == 1);
  }();
  // the rank-b trailing-update shape: NN, reduction of 96..128 (shorter ones carry twice the C
  // traffic per flop and stay on the cp.async kernel, which measured faster there), M, N >= 256
  static const int64_t kmin = [] {  // experiments: HB_GEMM_TMA_KMIN
    const char* e = getenv("HB_GEMM_TMA_KMIN");
    return e ? (int64_t)atoll(e) : (int64_t)96;
  }();
  if (off || g.transA || g.K < kmin || g.K < 8 || g.K > 128 || g.M < 256 || g.N < 256) return false;
  // TMA: global strides multiple of 16 bytes, coordinates in int32
  if ((g.lda & 1) || (g.ldb & 1) || g.M > (1ll << 30) || g.N > (1ll << 30)) return false;
  return true;
}

int64_t tma_gemm_fro_count(int64_t M, int64_t N, int num_sms) {
  const int64_t mb = ceil_div(M, kTBM), nb = ceil_div(N, kTBN);
  return mb * ceil_div(nb, tma_gemm_strip(M, N, num_sms)) * kTConsumers;
}

void launch_dgemm_tma(const GemmArgs& g, int num_sms, cudaStream_t st) {
  // K <= 120 (the full-width block) in 3 resident chunks of 40; otherwise 4 chunks of 32
  if (g.K <= 120) run_tma<40, 3, 3>(g, num_sms, g.fro_partials, st);
  else run_tma<32, 4, 4>(g, num_sms, g.fro_partials, st);
}

}  // namespace hb
