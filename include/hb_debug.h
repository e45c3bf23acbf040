/*
 * hb_debug.h -- test hooks of libhb200.so (not part of the drop-in boundary; used by tests/ and
 * tools/ to check the FP64 DMMA GEMM on its own).
 */
#ifndef HB_DEBUG_H
#define HB_DEBUG_H
#include <stdint.h>
#include "hb.h"
#ifdef __cplusplus
extern "C" {
#endif
/* C = alpha*op(A)*B + beta*C on the context stream (device pointers, column-major);
 * op(A) = A (M x K) if transA == 0, else A^T with A stored K x M.  Synchronises. */
hb_status hb_debug_dgemm(hb_context* ctx, int32_t transA, int64_t M, int64_t N, int64_t K,
                         double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                         double beta, double* C, int64_t ldc);
/* Same, without synchronising, repeated reps times (timing hook). */
hb_status hb_debug_dgemm_async(hb_context* ctx, int32_t transA, int64_t M, int64_t N, int64_t K,
                               double alpha, const double* A, int64_t lda, const double* B,
                               int64_t ldb, double beta, double* C, int64_t ldc, int32_t reps);
/* Same GEMM with the Frobenius epilogue of the trailing update: *fro_out = sum of squares of the
 * new C over rows >= fro_row0 (deterministic partials + fixed-order sum), synchronised. */
hb_status hb_debug_dgemm_fro(hb_context* ctx, int32_t transA, int64_t M, int64_t N, int64_t K,
                             double alpha, const double* A, int64_t lda, const double* B,
                             int64_t ldb, double beta, double* C, int64_t ldc, int64_t fro_row0,
                             double* fro_out);
#ifdef __cplusplus
}
#endif
#endif
