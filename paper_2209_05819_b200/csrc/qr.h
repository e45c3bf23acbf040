// Parameter blocks of the cooperative QR / SVD kernels (internal).
#pragma once

#include "common.cuh"

namespace hb {

struct SketchParams {
  const double* Y;  // ℓ x n_tr sketch of the trailing columns (ld = ldy)
  double* Ys;       // scratch copy, same shape
  double* nrm;      // n_tr scratch column norms (-1 = chosen)
  int ell;
  int64_t ldy;
  int64_t n_tr;
  int b_req;        // pivots wanted (<= kBlockMax)
  int b_min;        // fewest pivots before the early stop may fire
  double stop_fro2; // early stop when the sketch estimate of ||A22||_F^2 <= this
  double* slots;    // [2][G][3]
  int* piv;         // [b_req] pivot column (relative to the trailing start)
  int* swaps;       // [b_req] LAPACK-style swap targets
  double* rdiag;    // [b_req] |R_cc| of the sketch
  double* out_est;  // [b_req + 1] sketch estimate of ||A22||_F^2 before step c
  int* out_b;       // pivots chosen
  double* cand;     // [2][G][ell] best candidate column per CTA (shared-memory variant)
  GridBarrier bar;
};

constexpr int kPanelThreads = 512;  // panel_qr_smem_kernel block size
constexpr size_t kPanelClusterSmem = 220 * 1024;  // per-CTA budget of the cluster panel kernel

struct PanelParams {
  double* P;  // panel (mp x b), column-major
  int64_t ld;
  int64_t mp;
  int b;
  int64_t chunk;   // rows per CTA
  double* tau;     // [b]
  double* V;       // explicit V (mp x b)
  int64_t ldv;
  double* nslot;   // [G]
  double* wslot;   // [G][b]
  double* scal;    // [2] published alpha (shared-memory panel kernel)
  GridBarrier bar;
};

size_t panel_cluster_smem(int64_t chunk, int b, int G);
// Largest cluster (16 with the non-portable opt-in, else 8, else 0) `kern` can launch with at
// `threads` threads and `smem` bytes of dynamic shared memory per CTA (cached per kernel).
int cluster_cap(const void* kern, int threads, size_t smem);
int panel_cluster_max();
void launch_panel_cluster(const PanelParams& pp, int G, cudaStream_t st);

struct PowerParams {
  const double* R;  // rows 0..b-1 of the factor
  int64_t ld;
  int b;
  int64_t n;
  int iters;
  int mask;       // 1: first b columns upper trapezoidal (R factor), 0: dense (sketch rows)
  double* slots;  // [2][G][b+1]
  double* out;
  double* yout;   // optional: Rᵀ x of the last iteration (right singular direction), length n
  GridBarrier bar;
};

__global__ void sketch_cpqr_kernel(SketchParams p);
// Shared-memory-resident variant (sketch columns of a CTA fit in ~200 KB): one barrier per pivot,
// the winner's column travels through a per-CTA candidate slot instead of the global sketch.
constexpr int kSketchThreads = 512;
__global__ void sketch_cpqr_smem_kernel(SketchParams p);
__global__ void permute_kernel(double* A, int64_t lda, int64_t m, double* Y, int64_t ldy, int ell,
                               int64_t* perm, int64_t j, const int* swaps, const int* bptr);
__global__ void panel_qr_kernel(PanelParams p);
__global__ void panel_qr_smem_kernel(PanelParams p);
__global__ void build_T_kernel(const double* S, int64_t lds, const double* tau, int b, double* T,
                               int64_t ldt);
__global__ void sketch_trsm_kernel(const double* Y1, int64_t ldy, int ell, const double* R,
                                   int64_t ldr, int b, double* Z, int64_t ldz);
__global__ void power_sigma1_kernel(PowerParams p);
__global__ void sum_kernel(const double* parts, int64_t n, double* out);
__global__ void sumsq_kernel(const double* A, int64_t m, int64_t n, int64_t ld, double* parts);
__global__ void gram_sigma1_kernel(const double* G, int b, int iters, double* out);
__global__ void transpose_upper_kernel(const double* A, int64_t lda, int64_t k, int64_t n, double* B,
                                       int64_t ldb);
__global__ void copy_upper_kernel(const double* B, int64_t ldb, int64_t k, double* C, int64_t ldc);

// Bisection on the upper bidiagonal (d, e): singular-value queries.
struct SigmaQuery {
  double tol;       // relative tolerance
  double delta;     // residual bound δ for rank_hi
  int counts_only;  // skip the σ_p / σ_{p+1} bisections
  int pad;
};
struct SigmaAnswer {
  double sigma1, sigma_p, sigma_p1;
  int rank_lo, rank_hi;
};
__global__ void transpose_kernel(const double* src, int64_t lds, int64_t rows, int64_t cols,
                                 double* dst, int64_t ldd);
__global__ void write_lower_from_R(const double* R, int64_t ldr, int b, int nc, double* M, int64_t ldm);
__global__ void band_extract_kernel(const double* M, int64_t ldm, int64_t k, int nb, double* Bd);
__global__ void band_bidiag_out(const double* Bd, int64_t k, int nb, double* d, double* e);
__global__ void bulge_chase_kernel(double* Bd, int64_t k, int nb, int* prog);
__global__ void bidiag_small_kernel(const double* Mk, int64_t ldm, int k, double* d, double* e);
constexpr int kSmallBidiagThreads = 512;
constexpr int kSmallBidiag = 144;  // k x k triangle up to this size: one-CTA shared-memory bidiag
// Mid-size k: one thread-block cluster holds the triangle in distributed shared memory
// (bidiag_cluster.cu).  bidiag_cluster_size(k) = cluster size to use (8 or 16), 0 = does not fit.
constexpr size_t kBidiagClusterSmem = 225 * 1024;
size_t bidiag_cluster_smem(int k, int G);
int bidiag_cluster_size(int k);
void launch_bidiag_cluster(const double* Mk, int64_t ldm, int k, double* d, double* e, int G,
                           cudaStream_t st);
__global__ void sigma_queries_kernel(const double* d, const double* e, int64_t k,
                                     const SigmaQuery* q, int nq, SigmaAnswer* out,
                                     double* tg_glob, int tg_smem);
__global__ void sigma_all_kernel(const double* d, const double* e, int64_t k, double sigma_max,
                                 double* out);

}  // namespace hb

namespace hb {
__global__ void iota_kernel(int64_t* p, int64_t n);
__global__ void colnorm_normalize_kernel(double* X, int64_t ld, int64_t rows, double* norms,
                                         double* best);
__global__ void max_kernel(const double* v, int n, double* out);
__global__ void nonfinite_kernel(const double* A, int64_t m, int64_t n, int64_t ld, unsigned int* flags);
}  // namespace hb
