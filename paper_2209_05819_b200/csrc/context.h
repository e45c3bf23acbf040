// hb_context: per-device, per-host-thread state (stream, workspace, barrier slot).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "qr.h"

struct hb_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  size_t total_mem = 0;  // bytes of device memory (queried once at creation)
  int coop_sms = 148;  // SM share for cooperative grids (< num_sms when streams run concurrently)
  int priority = 0;    // CUDA stream priority of `stream` (0 = default)
  int block_max = hb::kBlockMax;
  bool spectral = false;  // spectral (probabilistic) stopping test (off: measured +3% columns saved for 7% time)
  double eta = 0.05;  // first stop once ||A22||_F <= eta * tol * sigma1 (refined if a bracket stays open)
  unsigned int* bar = nullptr;  // {count, gen}
  double* pinned = nullptr;     // small host staging (pinned)
  std::string last_error;

  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  std::vector<Buf> bufs;
  cudaEvent_t ev[6] = {};

  // profiling (hb_context_set_profiling)
  bool profiling = false;
  std::vector<cudaEvent_t> evpool;
  size_t evused = 0;
  struct Mark { int phase; size_t e0, e1; double flops; };
  std::vector<Mark> marks;
  hb_stats stats{};

  // last certification (for hb_last_sigma)
  int64_t last_k = 0;
  double last_sigma1 = 0.0;
};

// ACAFactor (aca.hpp:50-62) behind the opaque hb_aca_factor handle; L / U stay on the device.
struct hb_aca_factor {
  int device = 0;
  int32_t rank = 0;
  int32_t met = 1;
  std::vector<int64_t> sigma, tau;  // global target / source ids
  double* L = nullptr;              // device, rank x rank column-major (unit lower)
  double* U = nullptr;              // device, rank x rank column-major (upper)
  std::shared_ptr<double> store;    // the batch's L / U allocation (shared by its factors)
};

namespace hb {

enum BufId {
  B_A, B_X, B_Y, B_OMEGA, B_YSK, B_YS, B_NRM, B_V, B_W, B_W2, B_S, B_T, B_Z, B_TAU, B_SLOTS,
  B_PIV, B_SWAPS, B_RDIAG, B_EST, B_BEFF, B_PERM, B_FRO, B_FROSUM, B_SPLITK, B_CERT_B, B_CERT_M,
  B_D, B_E, B_BW, B_BV, B_SCAL, B_FLAGS, B_QUERY, B_ANSWER, B_SIG1, B_CERT_B2, B_PROG, B_ST1_P, B_ST1_X, B_ST1_X2, B_ST1_VT, B_PSCAL, B_TSUB, B_PX, B_PY, B_PN, B_SKCAND, B_TG, B_RDIAG2, B_COUNT
};

template <typename T>
T* ws(hb_context* c, int id, size_t elems) {
  if ((int)c->bufs.size() <= id) c->bufs.resize(B_COUNT);
  auto& b = c->bufs[id];
  const size_t bytes = std::max<size_t>(elems, 1) * sizeof(T);
  if (b.cap < bytes) {
    if (b.p) {
      void* old = b.p;
      // forget the old buffer before anything can throw: a failed allocation below must not
      // leave a freed pointer behind with its (larger) capacity for the next call to reuse
      b.p = nullptr;
      b.cap = 0;
      HB_CUDA(cudaFreeAsync(old, c->stream));
    }
    const size_t nb = bytes + bytes / 8;  // headroom
    HB_CUDA(cudaMallocAsync(&b.p, nb, c->stream));
    b.cap = nb;
  }
  return static_cast<T*>(b.p);
}

// ---- profiling helpers (rank.cu) ----
size_t prof_event(hb_context* c);                 // record a pooled event on the stream
void prof_resolve(hb_context* c);                 // after a stream sync: fold marks into stats
constexpr int PH_GEMM = -1;                       // mark kind for single GEMM launches
struct Phase {
  hb_context* c;
  int ph;
  size_t e0 = 0;
  bool open = true;
  Phase(hb_context* c_, int ph_) : c(c_), ph(ph_) {
    if (c->profiling) e0 = prof_event(c);
  }
  void close() {
    if (open && c->profiling) {
      try {
        c->marks.push_back({ph, e0, prof_event(c), 0.0});
      } catch (...) {
      }
    }
    open = false;
  }
  ~Phase() { close(); }
};

// Internal entry points (rank.cu).
void rank_matrix_inplace(hb_context* c, double* A, int64_t m, int64_t n, int64_t lda,
                         const double* tols, int ntol, hb_rank_result* out, float* fact_ms,
                         float* cert_ms);
void context_init(hb_context* c, int device);
void context_set_priority(hb_context* c, int prio);
// free (stream-ordered, back to the device pool) every workspace buffer larger than keep_bytes
void context_trim(hb_context* c, size_t keep_bytes);
void context_free(hb_context* c);
// HODLRdD operator (hmatrix.cu)
void hmatrix_build(hb_hmatrix* h, const double* pts_soa, const hb_cube& dom, int64_t n_max, double eps,
                   int64_t max_rank, int64_t dense_cap);
void hmatrix_matvec(hb_hmatrix* h, const double* d_q, double* d_b);
void hmatrix_free(hb_hmatrix* h);
// Chebyshev bound check (chebyshev.cu, chebyshev.hpp:125-193)
std::vector<double> cheb_nodes_host(int p);
void interpolation_decay(hb_context* c, const hb_kernel& kern, const double* tgt_soa, int64_t T,
                         const hb_cube& cube, const int32_t* p_list, int np, double* err_out);

}  // namespace hb
