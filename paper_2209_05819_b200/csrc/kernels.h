// Internal launch interface between the CUDA kernels and the host driver (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "hb.h"

namespace hb {

struct GridBarrier;

// ---- k1 / k2 -------------------------------------------------------------------------------
void launch_points(const hb_cube& cube, int64_t n, int mode, int64_t m_axis, uint64_t seed,
                   int role, double* out, cudaStream_t st);
bool kernel_singular_at_origin(int id);
void launch_negate(double* A, int64_t m, int64_t n, int64_t ld, cudaStream_t st);
void launch_assemble(const hb_kernel& kern, const double* x, int64_t T, const double* y,
                     int64_t N, int d, double* K, int64_t ldk, unsigned int* flags,
                     cudaStream_t st);

// ---- FP64 DMMA GEMM ------------------------------------------------------------------------
// C[M x N] = alpha * op(A) * B + beta * C, column-major; op(A) = A (M x K) or A^T (A is K x M).
// If fro_partials != nullptr, the sum of squares of the NEW C over rows >= fro_row0 is written
// per CTA to fro_partials[...] and their count to *fro_count (deterministic order).
struct GemmArgs {
  int64_t M, N, K;
  double alpha;
  const double* A;
  int64_t lda;
  bool transA;
  const double* B;
  int64_t ldb;
  double beta;
  double* C;
  int64_t ldc;
  double* fro_partials = nullptr;  // capacity >= gemm_fro_capacity(M, N)
  int64_t fro_row0 = 0;
};
void launch_dgemm(const GemmArgs& g, double* splitk_ws, int64_t splitk_ws_elems, int num_sms,
                  cudaStream_t st);
int64_t gemm_fro_count(int64_t M, int64_t N, int64_t K, int num_sms);  // partial slots for this shape

// ---- sketch ----------------------------------------------------------------------------------
void launch_gaussian(double* omega, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                     cudaStream_t st);

struct Workspace;  // defined in rank.cu

// ---- ACA (aca.cu) ---------------------------------------------------------------------------
void aca_compress(hb_context* c, const hb_kernel& kern, const double* x, int64_t nt, const double* y,
                  int64_t ns, int d, const hb_block* blks, int64_t nb, double eps, int64_t max_rank,
                  hb_aca_factor** out);
void aca_apply(hb_context* c, const hb_aca_factor* f, const hb_kernel& kern, const double* x, int64_t nt,
               const double* y, int64_t ns, int d, const hb_block& blk, const double* q, double* b);

}  // namespace hb
