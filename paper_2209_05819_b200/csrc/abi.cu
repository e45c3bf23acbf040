// C ABI (include/hb.h): argument validation mirroring the reference's exceptions, k1/k2 entry
// points, hb_rank / hb_rank_matrix, the multi-device sweep driver (k4) and its LPT partition.
// No C++ exception crosses this file's extern "C" functions.
#include <algorithm>
#include <atomic>
#include <memory>
#include <cmath>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <numeric>
#include <thread>
#include <vector>

#include "context.h"
#include "bessel_dd.cuh"
#include "hmatrix.h"

namespace {

std::mutex g_err_mu;
std::string g_err;

void set_err(hb_context* c, const std::string& s) {
  if (c) c->last_error = s;
  std::lock_guard<std::mutex> lk(g_err_mu);
  g_err = s;
}

template <typename F>
hb_status guarded(hb_context* c, F&& f) {
  try {
    f();
    return HB_OK;
  } catch (const hb::Error& e) {
    set_err(c, e.what());
    return e.status;
  } catch (const std::bad_alloc& e) {
    set_err(c, "host allocation failed");
    return HB_ENOMEM;
  } catch (const std::exception& e) {
    set_err(c, e.what());
    return HB_ECUDA;
  } catch (...) {
    set_err(c, "unknown exception");
    return HB_ECUDA;
  }
}

using hb::Error;

void check_kernel(const hb_kernel* k) {
  if (!k) throw Error(HB_EINVAL, "kernel descriptor is NULL");
  if (k->id < 0 || k->id > HB_K_CUSTOM) throw Error(HB_EINVAL, "unknown kernel id");
  if (k->id == HB_K_CUSTOM)  // kernel.hpp:69-76: std::function cannot cross to the device
    throw Error(HB_EUNSUPPORTED, "Custom kernels (std::function) are not supported on the device");
}

// integer d-th root of n, or -1
int64_t int_root(int64_t n, int d) {
  int64_t r = (int64_t)std::llround(std::pow((double)n, 1.0 / d));
  for (int64_t c = std::max<int64_t>(1, r - 2); c <= r + 2; ++c) {
    int64_t p = 1;
    for (int k = 0; k < d; ++k) p *= c;
    if (p == n) return c;
  }
  return -1;
}

void check_cube(const hb_cube& c) {
  if (c.d < 1 || c.d > 8) throw Error(HB_EINVAL, "cube dimension must be in 1..8");
  if (!(c.side > 0.0)) throw Error(HB_EINVAL, "HyperCube: side must be positive");  // geometry.hpp:22
  for (int k = 0; k < c.d; ++k)
    if (!std::isfinite(c.lower[k])) throw Error(HB_EINVAL, "cube corner must be finite");
}

int64_t check_points(const hb_cube& c, int64_t n, int mode) {
  if (n < 1) throw Error(HB_EINVAL, "empty point set");  // kernel.hpp:171
  if (mode == HB_POINTS_UNIFORM) return 0;
  if (mode != HB_POINTS_GRID_INTERIOR && mode != HB_POINTS_GRID_CLOSED)
    throw Error(HB_EINVAL, "unknown point mode");
  const int64_t m = int_root(n, c.d);
  if (m < 1) throw Error(HB_EINVAL, "grid mode needs N = n^d (SPEC.md:540)");
  if (mode == HB_POINTS_GRID_CLOSED && m < 2) throw Error(HB_EINVAL, "closed grid needs n >= 2");
  return m;
}

// classify_pair (geometry.hpp:109-118) on per-axis grid offsets
hb_interaction classify_offsets(const int64_t* off, int d) {
  bool all_zero = true;
  int64_t mx = 0;
  int zeros = 0;
  for (int k = 0; k < d; ++k) {
    const int64_t o = off[k] < 0 ? -off[k] : off[k];
    all_zero &= o == 0;
    mx = std::max(mx, o);
    zeros += o == 0;
  }
  if (all_zero) return hb_interaction{HB_IC_SELF, -1};
  if (mx >= 2) return hb_interaction{HB_IC_FAR, -1};
  return hb_interaction{HB_IC_SURFACE, zeros};
}

// Two cubes of one uniform subdivision: equal sides, corner offsets integer multiples of the side
// (exactly representable here: the offsets are small integers times the side).  false if not.
bool cube_offsets(const hb_cube& a, const hb_cube& b, int64_t* off) {
  if (a.d != b.d || a.side != b.side) return false;
  for (int k = 0; k < a.d; ++k) {
    const double q = (b.lower[k] - a.lower[k]) / a.side;
    const double r = std::nearbyint(q);
    if (!(std::fabs(q - r) <= 1e-9 * std::max(1.0, std::fabs(q))) || std::fabs(r) > 1e15) return false;
    off[k] = (int64_t)r;
  }
  return true;
}

int32_t dprime_of(const hb_interaction& ic) {
  return ic.kind == HB_IC_SELF ? HB_DPRIME_SELF : (ic.kind == HB_IC_FAR ? HB_DPRIME_FAR : ic.surface_dim);
}

void check_pair(const hb_pair* p) {
  if (!p) throw Error(HB_EINVAL, "pair descriptor is NULL");
  check_cube(p->target);
  check_cube(p->source);
  if (p->target.d != p->source.d) throw Error(HB_EINVAL, "point dimensions differ");  // kernel.hpp:172
  check_points(p->target, p->n_target, p->point_mode);
  check_points(p->source, p->n_source, p->point_mode);
  if (p->d_prime < HB_DPRIME_SELF || p->d_prime >= p->target.d)
    throw Error(HB_EINVAL, "d_prime must be -2 (self), -1 (far) or a surface dimension 0..d-1");
  int64_t off[8];
  if (cube_offsets(p->target, p->source, off)) {  // boxes of one subdivision: d' is implied
    const int32_t implied = dprime_of(classify_offsets(off, p->target.d));
    if (implied != p->d_prime)
      throw Error(HB_EINVAL, "d_prime does not match the cube pair's interaction class (classify_pair)");
  }
}

void check_tols(const double* tols, int32_t ntol) {
  if (!tols || ntol < 1 || ntol > HB_MAX_TOLS) throw Error(HB_EINVAL, "need 1..4 tolerances");
  for (int t = 0; t < ntol; ++t)
    if (!(tols[t] > 0.0 && tols[t] < 1.0)) throw Error(HB_EINVAL, "tolerance must be in (0, 1)");
}

unsigned int read_flags(hb_context* c, unsigned int* dflags) {
  unsigned int f = 0;
  HB_CUDA(cudaMemcpyAsync(c->pinned, dflags, sizeof(f), cudaMemcpyDeviceToHost, c->stream));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  std::memcpy(&f, c->pinned, sizeof(f));
  return f;
}

void raise_flags(unsigned int f) {
  if (f & 1u)
    throw Error(HB_ESINGULAR,
                "kernel eval: r == 0 on a singular kernel with no diagonal value");  // kernel.hpp:152-153
  if (f & 2u) throw Error(HB_EDOMAIN, "non-finite kernel entries");
}

void gen_points(hb_context* c, const hb_pair* pair, double* dt, double* ds) {
  const int64_t mt = check_points(pair->target, pair->n_target, pair->point_mode);
  const int64_t ms = check_points(pair->source, pair->n_source, pair->point_mode);
  hb::launch_points(pair->target, pair->n_target, pair->point_mode, mt, pair->seed, 0, dt, c->stream);
  hb::launch_points(pair->source, pair->n_source, pair->point_mode, ms, pair->seed, 1, ds, c->stream);
}

void rank_pair(hb_context* c, const hb_kernel* kernel, const hb_pair* pair, const double* tols,
               int32_t ntol, hb_rank_result* out) {
  check_kernel(kernel);
  check_pair(pair);
  check_tols(tols, ntol);
  HB_CUDA(cudaSetDevice(c->device));
  {
    // a non-sticky error left by an earlier unchecked runtime call on this host thread must not
    // be reported as this problem's launch failure (sticky device faults still surface at sync)
    const cudaError_t stale = cudaGetLastError();
    if (stale != cudaSuccess && getenv("HB_DEBUG"))
      fprintf(stderr, "[hb] cleared stale CUDA error before problem: %s\n", cudaGetErrorString(stale));
  }
  const int d = pair->target.d;
  const int64_t m = pair->n_target, n = pair->n_source;
  const int64_t lda = hb::round_up(m, 8);
  // total device memory cached at context creation: the driver query was seen blocking every
  // sweep thread for tens of ms at once
  const size_t total_b = c->total_mem;
  if ((double)lda * n * 8.0 * 1.25 > (double)total_b)
    throw Error(HB_ENOMEM, "K does not fit in device memory");
  HB_CUDA(cudaEventRecord(c->ev[0], c->stream));
  hb::Phase ph(c, HB_PH_ASSEMBLY);
  double* X = hb::ws<double>(c, hb::B_X, (size_t)d * m);
  double* Yp = hb::ws<double>(c, hb::B_Y, (size_t)d * n);
  double* A = hb::ws<double>(c, hb::B_A, (size_t)lda * n);
  unsigned int* flags = hb::ws<unsigned int>(c, hb::B_FLAGS, 4);
  HB_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned int), c->stream));
  gen_points(c, pair, X, Yp);
  hb::launch_assemble(*kernel, X, m, Yp, n, d, A, lda, flags, c->stream);
  HB_CUDA(cudaEventRecord(c->ev[4], c->stream));
  ph.close();
  raise_flags(read_flags(c, flags));
  float fm = 0, cm = 0;
  hb::rank_matrix_inplace(c, A, m, n, lda, tols, ntol, out, &fm, &cm);
  float am = 0;
  HB_CUDA(cudaEventElapsedTime(&am, c->ev[0], c->ev[4]));
  for (int t = 0; t < ntol; ++t) {
    out[t].sec[0] = am * 1e-3;
    out[t].sec[3] = (am + fm + cm) * 1e-3;
  }
}

// ε-rank of K_re + i·K_im through the real embedding E = [[Re, −Im], [Im, Re]] (2m x 2n): its
// singular values are those of the complex block, each twice, so count(σ(E) > thr) = 2·rank.
void rank_pair_complex(hb_context* c, const hb_kernel* kre, const hb_kernel* kim, const hb_pair* pair,
                       const double* tols, int32_t ntol, hb_rank_result* out) {
  check_kernel(kre);
  check_kernel(kim);
  check_pair(pair);
  check_tols(tols, ntol);
  HB_CUDA(cudaSetDevice(c->device));
  cudaGetLastError();
  const int d = pair->target.d;
  const int64_t m = pair->n_target, n = pair->n_source;
  const int64_t m2 = 2 * m, n2 = 2 * n;
  const int64_t lda = hb::round_up(m2, 8);
  const size_t total_b = c->total_mem;
  if ((double)lda * n2 * 8.0 * 1.25 > (double)total_b)
    throw Error(HB_ENOMEM, "the real embedding does not fit in device memory");
  HB_CUDA(cudaEventRecord(c->ev[0], c->stream));
  hb::Phase ph(c, HB_PH_ASSEMBLY);
  double* X = hb::ws<double>(c, hb::B_X, (size_t)d * m);
  double* Yp = hb::ws<double>(c, hb::B_Y, (size_t)d * n);
  double* A = hb::ws<double>(c, hb::B_A, (size_t)lda * n2);
  unsigned int* flags = hb::ws<unsigned int>(c, hb::B_FLAGS, 4);
  HB_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned int), c->stream));
  gen_points(c, pair, X, Yp);
  hb::launch_assemble(*kre, X, m, Yp, n, d, A, lda, flags, c->stream);                  // Re
  hb::launch_assemble(*kre, X, m, Yp, n, d, A + m + n * lda, lda, flags, c->stream);    // Re
  hb::launch_assemble(*kim, X, m, Yp, n, d, A + m, lda, flags, c->stream);              // Im
  hb::launch_assemble(*kim, X, m, Yp, n, d, A + n * lda, lda, flags, c->stream);        // −Im
  hb::launch_negate(A + n * lda, m, n, lda, c->stream);
  HB_CUDA(cudaEventRecord(c->ev[4], c->stream));
  ph.close();
  raise_flags(read_flags(c, flags));
  float fm = 0, cm = 0;
  hb::rank_matrix_inplace(c, A, m2, n2, lda, tols, ntol, out, &fm, &cm);
  float am = 0;
  HB_CUDA(cudaEventElapsedTime(&am, c->ev[0], c->ev[4]));
  for (int t = 0; t < ntol; ++t) {
    hb_rank_result& r = out[t];
    const bool split = (r.rank_lo & 1) != 0;  // a σ pair of E straddles the threshold (near-tie)
    r.rank_lo = r.rank_lo / 2;
    r.rank_hi = (r.rank_hi + 1) / 2;
    r.rank = r.rank_lo;
    if (split || r.rank_lo != r.rank_hi) r.certificate = 0;
    r.sec[0] = am * 1e-3;
    r.sec[3] = (am + fm + cm) * 1e-3;
  }
}

// ---- cost model for the LPT partition --------------------------------
double predicted_rank(int d, int dprime, int64_t n) {
  // growth laws: far-field constant, vertex ~ log N, d'-surface ~ N^{d'/d};
  // magnitudes from the paper tables at their first N row (F1/F2/F8 average).
  static const double far_r[5] = {0, 7, 35, 100, 620};
  static const double vert_r[5] = {0, 20, 60, 135, 375};
  const double lg = std::log2(std::max<double>((double)n, 2.0) / 1000.0);
  if (dprime < 0) return far_r[std::min(d, 4)];
  if (dprime == 0) return vert_r[std::min(d, 4)] * (1.0 + 0.08 * std::max(0.0, lg));
  const double n0 = d == 2 ? 1600.0 : (d == 3 ? 1000.0 : 1296.0);
  double base = 200.0;
  if (d == 3) base = dprime == 1 ? 105.0 : 330.0;
  if (d >= 4) base = dprime == 1 ? 470.0 : (dprime == 2 ? 620.0 : 830.0);
  return std::min<double>((double)n, base * std::pow((double)n / n0, (double)dprime / d));
}

// Factorisation width k̂ (columns of the pivoted QR before certification).  For the three BASELINE
// kernels and d <= 4 it is interpolated geometrically in N between the widths measured at
// N = 1000, 8000 and 65536 (tol 1e-12; profiles/r02/solo_all_s3a.json); any other problem falls back
// to 1.4 p̂ + 32 from the paper's growth laws.  Scheduling only: a wrong k̂ costs balance, never a
// result.
double predicted_width(const hb_problem& p) {
  struct Row { int d, dp; double k[3][3]; };  // k[kernel: 1/r, log r, exp(-r)][N = 1000, 8000, 65536]
  static const Row tab[] = {
      {1, -1, {{16, 16, 16}, {8, 8, 8}, {8, 8, 8}}},
      {1, 0, {{32, 40, 48}, {24, 32, 40}, {8, 8, 8}}},
      {2, -1, {{64, 64, 64}, {24, 24, 32}, {56, 56, 56}}},
      {2, 0, {{112, 152, 192}, {48, 56, 64}, {96, 120, 144}}},
      {2, 1, {{232, 616, 1680}, {120, 272, 696}, {200, 480, 1200}}},
      {3, -1, {{176, 208, 216}, {256, 312, 328}, {232, 280, 288}}},
      {3, 0, {{216, 312, 432}, {320, 480, 600}, {280, 408, 560}}},
      {3, 1, {{296, 576, 1080}, {432, 888, 1680}, {360, 696, 1200}}},
      {3, 2, {{472, 1560, 5752}, {624, 2152, 7800}, {536, 1744, 6120}}},
      {4, -1, {{704, 1552, 2040}, {664, 1320, 1680}, {712, 1512, 1800}}},
      {4, 0, {{712, 1536, 2280}, {672, 1320, 1912}, {720, 1440, 2128}}},
      {4, 1, {{784, 2080, 3840}, {752, 1848, 3240}, {784, 1976, 3360}}},
      {4, 2, {{888, 3000, 8520}, {872, 2760, 6960}, {880, 2832, 6960}}},
      {4, 3, {{960, 4504, 19800}, {960, 4320, 18120}, {952, 4312, 17880}}},
  };
  const double n = (double)std::max(p.pair.n_target, p.pair.n_source);
  const int d = p.pair.target.d, dp = p.pair.d_prime < 0 ? -1 : p.pair.d_prime;
  const int kc = p.kernel.id == HB_K_INVERSE_R ? 0 : (p.kernel.id == HB_K_LOG_R ? 1 : (p.kernel.id == HB_K_EXP_NEG_R ? 2 : -1));
  if (kc >= 0)
    for (const Row& r : tab)
      if (r.d == d && r.dp == dp) {
        const int hi = n > 8000.0 ? 1 : 0;  // piecewise geometric: [1000, 8000], [8000, 65536]
        const double n0 = hi ? 8000.0 : 1000.0, n1 = hi ? 65536.0 : 8000.0;
        const double g = std::log(r.k[kc][hi + 1] / r.k[kc][hi]) / std::log(n1 / n0);
        return std::min(n, r.k[kc][hi] * std::pow(std::max(n, 64.0) / n0, g));
      }
  return std::min(n, 1.4 * predicted_rank(d, p.pair.d_prime, (int64_t)n) + 32.0);
}

// Predicted device seconds of one problem, as the LPT weight.  Coefficients: non-negative least
// squares of the solo device times of the 294 sweep problems (tools/solo_all.py,
// profiles/r02/solo_all_s3a.json; relative residual 21 % rms) on
//   g = 0.0355 s/TFLOP * (QR + certification flops) + 0.019 s per 1e9 entries   (device-filling)
//   l = 0.0204 s * blocks * N/1e6 + 0.0048 s * blocks + 0.0072 s * (k/1000)^2    (latency-bound)
// With 4 streams per GPU the latency-bound phases of one problem overlap other problems' GEMMs:
// measured share times of the 2/4/8-way splits follow sum(g) + sum(l)/2 within 0.87-1.07
// (profiles/r02/predict_scaling_s3a.json), so the weight is g + l/2.
double problem_cost(const hb_problem& p) {
  const double n = (double)std::max(p.pair.n_target, p.pair.n_source);
  const double k = predicted_width(p);
  const double qr = 4.0 * n * n * k - 4.0 * n * k * k + 4.0 / 3.0 * k * k * k;
  const double cert = 2.0 * k * k * (n - k / 3.0) + 8.0 / 3.0 * k * k * k;
  const double blocks = k / 120.0;
  const double g = 0.0355 * (qr + cert) * 1e-12 + 0.019 * n * n * 1e-9;
  const double l = 0.0204 * blocks * n * 1e-6 + 0.0048 * blocks + 0.0072 * (k * 1e-3) * (k * 1e-3);
  return g + 0.5 * l;
}

// live contexts (for process-wide stats) and the per-device cache used by hb_sweep
std::mutex g_reg_mu;
std::vector<hb_context*> g_live;
hb_stats g_retired{};
std::vector<std::pair<std::pair<int, int>, hb_context*>> g_cache;  // ((device, slot), ctx)

void add_stats(hb_stats& a, const hb_stats& b) {
  for (int i = 0; i < HB_NPHASE; ++i) a.phase_ms[i] += b.phase_ms[i];
  a.gemm_ms += b.gemm_ms;
  a.gemm_flops += b.gemm_flops;
  a.gemm_launches += b.gemm_launches;
  a.problems += b.problems;
}

}  // namespace

extern "C" {

const char* hb_version(void) { return "hb200 0.1 (sm_100a)"; }

const char* hb_status_string(hb_status s) {
  switch (s) {
    case HB_OK: return "ok";
    case HB_EINVAL: return "invalid argument";
    case HB_EDOMAIN: return "domain error";
    case HB_ECAP: return "size cap exceeded";
    case HB_ESINGULAR: return "singular kernel at r == 0";
    case HB_EUNSUPPORTED: return "unsupported";
    case HB_ENOMEM: return "out of memory";
    case HB_ECUDA: return "CUDA error";
    case HB_ENCCL: return "NCCL error";
  }
  return "unknown status";
}

const char* hb_last_error(const hb_context* ctx) {
  if (ctx) return ctx->last_error.c_str();
  std::lock_guard<std::mutex> lk(g_err_mu);
  static thread_local std::string copy;
  copy = g_err;
  return copy.c_str();
}

hb_status hb_context_create(int device, hb_context** out) {
  if (!out) return HB_EINVAL;
  *out = nullptr;
  hb_context* c = new (std::nothrow) hb_context();
  if (!c) return HB_ENOMEM;
  hb_status s = guarded(nullptr, [&] {
    int n = 0;
    HB_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw Error(HB_EINVAL, "no such CUDA device");
    hb::context_init(c, device);
  });
  if (s != HB_OK) {
    hb::context_free(c);
    delete c;
    return s;
  }
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    g_live.push_back(c);
  }
  *out = c;
  return HB_OK;
}

void hb_context_destroy(hb_context* ctx) {
  if (!ctx) return;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    add_stats(g_retired, ctx->stats);
    g_live.erase(std::remove(g_live.begin(), g_live.end(), ctx), g_live.end());
  }
  hb::context_free(ctx);
  delete ctx;
}

const char* hb_phase_name(int32_t ph) {
  static const char* names[HB_NPHASE] = {"assembly", "sketch", "pivot", "panel", "update",
                                         "downdate", "sigma1", "cert_qr", "bidiag", "bisect",
                                         "chase"};
  return (ph >= 0 && ph < HB_NPHASE) ? names[ph] : "?";
}

hb_status hb_context_set_profiling(hb_context* ctx, int32_t on) {
  if (!ctx) return HB_EINVAL;
  ctx->profiling = on != 0;
  return HB_OK;
}

hb_status hb_stats_get(const hb_context* ctx, hb_stats* out) {
  if (!out) return HB_EINVAL;
  hb_stats s{};
  if (ctx) {
    s = ctx->stats;
  } else {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    s = g_retired;
    for (auto* c : g_live) add_stats(s, c->stats);
  }
  s.launches = hb::launch_counter().load();
  *out = s;
  return HB_OK;
}

hb_status hb_stats_reset(hb_context* ctx) {
  if (ctx) {
    ctx->stats = hb_stats{};
  } else {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    g_retired = hb_stats{};
    for (auto* c : g_live) c->stats = hb_stats{};
  }
  return HB_OK;
}

void* hb_context_stream(hb_context* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

hb_status hb_context_set_tuning(hb_context* ctx, int32_t block_max, double eta) {
  if (!ctx) return HB_EINVAL;
  if (block_max < 8 || block_max > hb::kBlockMax || block_max % 8) return HB_EINVAL;
  if (!(eta > 0.0 && eta <= 0.1)) return HB_EINVAL;
  ctx->block_max = block_max;
  ctx->eta = eta;
  return HB_OK;
}

hb_status hb_context_set_stopping(hb_context* ctx, int32_t spectral) {
  if (!ctx || spectral < 0 || spectral > 1) return HB_EINVAL;
  ctx->spectral = spectral != 0;
  return HB_OK;
}

hb_status hb_generate_points(hb_context* ctx, const hb_pair* pair, double* d_tgt, double* d_src) {
  if (!ctx) return HB_EINVAL;
  return guarded(ctx, [&] {
    check_pair(pair);
    if (!d_tgt || !d_src) throw Error(HB_EINVAL, "NULL output buffer");
    HB_CUDA(cudaSetDevice(ctx->device));
    gen_points(ctx, pair, d_tgt, d_src);
  });
}

hb_status hb_assemble(hb_context* ctx, const hb_kernel* kernel, const double* d_tgt, int64_t T,
                      const double* d_src, int64_t N, int32_t d, double* d_K, int64_t ldk) {
  if (!ctx) return HB_EINVAL;
  return guarded(ctx, [&] {
    check_kernel(kernel);
    if (T <= 0 || N <= 0) throw Error(HB_EINVAL, "assemble_dense: empty point set");  // kernel.hpp:171
    if (d < 1 || d > 8) throw Error(HB_EINVAL, "assemble_dense: bad dimension");
    if (ldk < T) throw Error(HB_EINVAL, "assemble_dense: ldk < T");
    if (!d_tgt || !d_src || !d_K) throw Error(HB_EINVAL, "NULL buffer");
    HB_CUDA(cudaSetDevice(ctx->device));
    unsigned int* flags = hb::ws<unsigned int>(ctx, hb::B_FLAGS, 4);
    HB_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned int), ctx->stream));
    hb::launch_assemble(*kernel, d_tgt, T, d_src, N, d, d_K, ldk, flags, ctx->stream);
    raise_flags(read_flags(ctx, flags));
  });
}

hb_status hb_classify_pair(int32_t d, int32_t level_a, const int32_t* grid_a, int32_t level_b,
                           const int32_t* grid_b, hb_interaction* out) {
  return guarded(nullptr, [&] {
    if (!out || !grid_a || !grid_b) throw Error(HB_EINVAL, "classify_pair: NULL argument");
    if (level_a != level_b)  // geometry.hpp:110-111
      throw Error(HB_EINVAL, "classify_pair: boxes are at different levels");
    if (d < 1 || d > 64) throw Error(HB_EINVAL, "classify_pair: boxes have different dimensions");
    std::vector<int64_t> off((size_t)d);
    for (int k = 0; k < d; ++k) off[(size_t)k] = (int64_t)grid_a[k] - (int64_t)grid_b[k];
    *out = classify_offsets(off.data(), d);
  });
}

hb_status hb_classify_cubes(const hb_cube* a, const hb_cube* b, hb_interaction* out) {
  return guarded(nullptr, [&] {
    if (!a || !b || !out) throw Error(HB_EINVAL, "classify: NULL argument");
    check_cube(*a);
    check_cube(*b);
    int64_t off[8];
    if (!cube_offsets(*a, *b, off))
      throw Error(HB_EINVAL, "classify: cubes are not boxes of one uniform subdivision");
    *out = classify_offsets(off, a->d);
  });
}

int32_t hb_interaction_dprime(hb_interaction ic) { return dprime_of(ic); }

hb_status hb_fit_growth(const int64_t* N, const double* rank, int32_t n, hb_growth_fit* out) {
  return guarded(nullptr, [&] {
    if (!N || !rank || !out) throw Error(HB_EINVAL, "fit_growth: NULL argument");
    std::vector<double> x, y;
    for (int32_t i = 0; i < n; ++i) {
      if (N[i] <= 0 || !(rank[i] >= 0.0)) throw Error(HB_EINVAL, "fit_growth: N must be > 0, rank >= 0");
      x.push_back((double)N[i]);
      y.push_back(rank[i]);
    }
    std::vector<double> xs(x);
    std::sort(xs.begin(), xs.end());
    if (std::unique(xs.begin(), xs.end()) - xs.begin() < 4)
      throw Error(HB_EINVAL, "fit_growth: fewer than 4 distinct N values");
    const double m = (double)x.size();
    double ym = 0.0, ymin = INFINITY, ymax = 0.0;
    for (double v : y) { ym += v; ymin = std::min(ymin, v); ymax = std::max(ymax, v); }
    ym /= m;
    hb_growth_fit f{};
    f.n = (int32_t)x.size();
    f.max_min_ratio = ymin > 0.0 ? ymax / ymin : INFINITY;
    // constant
    f.constant = ym;
    for (double v : y) f.rss[0] += (v - ym) * (v - ym);
    // a + b ln N (ordinary least squares)
    auto linfit = [&](const std::vector<double>& u, double* a, double* b) {
      double um = 0.0;
      for (double v : u) um += v;
      um /= m;
      double sxy = 0.0, sxx = 0.0;
      for (size_t i = 0; i < u.size(); ++i) {
        sxy += (u[i] - um) * (y[i] - ym);
        sxx += (u[i] - um) * (u[i] - um);
      }
      *b = sxx > 0.0 ? sxy / sxx : 0.0;
      *a = ym - *b * um;
    };
    std::vector<double> lx(x.size());
    for (size_t i = 0; i < x.size(); ++i) lx[i] = std::log(x[i]);
    linfit(lx, &f.log_a, &f.log_b);
    for (size_t i = 0; i < x.size(); ++i) {
      const double r = y[i] - (f.log_a + f.log_b * lx[i]);
      f.rss[1] += r * r;
    }
    // a N^c: for fixed c the best a is closed-form; c by golden-section search on [0, 2]
    auto rss_pow = [&](double c, double* a_out) {
      double num = 0.0, den = 0.0;
      for (size_t i = 0; i < x.size(); ++i) {
        const double t = std::pow(x[i], c);
        num += t * y[i];
        den += t * t;
      }
      const double a = den > 0.0 ? num / den : 0.0;
      double r2 = 0.0;
      for (size_t i = 0; i < x.size(); ++i) {
        const double r = y[i] - a * std::pow(x[i], c);
        r2 += r * r;
      }
      if (a_out) *a_out = a;
      return r2;
    };
    double lo = 0.0, hi = 2.0;
    const double gr = 0.5 * (std::sqrt(5.0) - 1.0);
    double c1 = hi - gr * (hi - lo), c2 = lo + gr * (hi - lo);
    double f1 = rss_pow(c1, nullptr), f2 = rss_pow(c2, nullptr);
    for (int it = 0; it < 200 && hi - lo > 1e-12; ++it) {
      if (f1 <= f2) { hi = c2; c2 = c1; f2 = f1; c1 = hi - gr * (hi - lo); f1 = rss_pow(c1, nullptr); }
      else { lo = c1; c1 = c2; f1 = f2; c2 = lo + gr * (hi - lo); f2 = rss_pow(c2, nullptr); }
    }
    f.pow_c = 0.5 * (lo + hi);
    f.rss[2] = rss_pow(f.pow_c, &f.pow_a);
    // model choice: BIC with a floor on the residual scale (ties go to fewer parameters)
    const double s2 = (1e-3 * ym) * (1e-3 * ym) + 1e-300;
    const int params[3] = {1, 2, 2};
    double best = INFINITY;
    for (int k = 0; k < 3; ++k) {
      const double bic = m * std::log(f.rss[k] / m + s2) + params[k] * std::log(m);
      if (bic < best - 1e-9) { best = bic; f.best = k; }
    }
    *out = f;
  });
}

hb_status hb_hmatrix_build(hb_context* ctx, const hb_kernel* kernel, const double* pts, int64_t N, int32_t d,
                           const hb_cube* domain, int32_t policy, int64_t n_max, double epsilon,
                           int64_t max_rank, int64_t dense_entry_cap, hb_hmatrix** out,
                           hb_build_report* report) {
  if (!ctx || !out) return HB_EINVAL;
  *out = nullptr;
  hb_hmatrix* h = nullptr;
  const hb_status s = guarded(ctx, [&] {
    check_kernel(kernel);
    if (!(epsilon > 0)) throw Error(HB_EINVAL, "HMatrix: epsilon must be positive");  // hmatrix.hpp:56
    if (!pts || !domain) throw Error(HB_EINVAL, "HMatrix: NULL argument");
    if (N < 1) throw Error(HB_EINVAL, "build_tree: empty point set");  // cluster_tree.hpp:185
    if (n_max < 1) throw Error(HB_EINVAL, "build_tree: n_max must be >= 1");
    if (max_rank < 1) throw Error(HB_EINVAL, "aca::compress: max_rank must be >= 1");
    if (policy < HB_POLICY_WEAKDD || policy > HB_POLICY_WEAKALL) throw Error(HB_EINVAL, "unknown policy");
    check_cube(*domain);
    if (d != domain->d) throw Error(HB_EINVAL, "build_tree: point dimension does not match domain");
    for (int64_t i = 0; i < N; ++i)  // HyperCube::contains, closed bounds (geometry.hpp:39-44)
      for (int k = 0; k < d; ++k) {
        const double x = pts[(int64_t)k * N + i];
        if (x < domain->lower[k] || x > domain->lower[k] + domain->side)
          throw Error(HB_EDOMAIN, "build_tree: point outside the domain hyper-cube");
      }
    HB_CUDA(cudaSetDevice(ctx->device));
    h = new hb_hmatrix();
    h->ctx = ctx;
    h->device = ctx->device;
    h->kern = *kernel;
    h->d = d;
    h->N = N;
    h->policy = policy;
    hb::hmatrix_build(h, pts, *domain, n_max, epsilon, max_rank,
                      dense_entry_cap > 0 ? dense_entry_cap : 400000000ll);
    if (report) *report = h->report;
  });
  if (s != HB_OK) {
    if (h) {
      hb::hmatrix_free(h);
      delete h;
    }
    return s;
  }
  *out = h;
  return HB_OK;
}

hb_status hb_hmatrix_matvec_device(hb_hmatrix* h, const double* d_q, double* d_b) {
  if (!h || !d_q || !d_b) return HB_EINVAL;
  return guarded(h->ctx, [&] {
    HB_CUDA(cudaSetDevice(h->ctx->device));
    hb::hmatrix_matvec(h, d_q, d_b);
  });
}

hb_status hb_hmatrix_matvec(hb_hmatrix* h, const double* q, double* b, int32_t nvec) {
  if (!h || !q || !b || nvec < 1) return HB_EINVAL;
  return guarded(h->ctx, [&] {
    hb_context* c = h->ctx;
    HB_CUDA(cudaSetDevice(c->device));
    const int64_t n = h->N;
    double* dq = hb::ws<double>(c, hb::B_PX, (size_t)n);
    double* db = hb::ws<double>(c, hb::B_PY, (size_t)n);
    for (int32_t v = 0; v < nvec; ++v) {
      HB_CUDA(cudaMemcpyAsync(dq, q + (int64_t)v * n, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
      hb::hmatrix_matvec(h, dq, db);
      HB_CUDA(cudaMemcpyAsync(b + (int64_t)v * n, db, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    }
    unsigned int f = 0;
    HB_CUDA(cudaMemcpyAsync(&f, h->d_flags, sizeof(f), cudaMemcpyDeviceToHost, c->stream));
    HB_CUDA(cudaStreamSynchronize(c->stream));
    raise_flags(f);
  });
}

hb_status hb_hmatrix_tree_order(const hb_hmatrix* h, int64_t* orig) {
  if (!h || !orig) return HB_EINVAL;
  std::memcpy(orig, h->orig_of_tree.data(), sizeof(int64_t) * h->N);
  return HB_OK;
}

void hb_hmatrix_destroy(hb_hmatrix* h) {
  if (!h) return;
  hb::hmatrix_free(h);
  delete h;
}

hb_status hb_chebyshev_nodes(int32_t p, double* out) {
  return guarded(nullptr, [&] {
    if (!out) throw Error(HB_EINVAL, "chebyshev_nodes: NULL output");
    const std::vector<double> y = hb::cheb_nodes_host(p);
    std::memcpy(out, y.data(), sizeof(double) * y.size());
  });
}

hb_status hb_interpolation_decay(hb_context* ctx, const hb_kernel* kernel, const double* tgt, int64_t T,
                                 const hb_cube* cube, const int32_t* p_list, int32_t np, double* err_out) {
  if (!ctx) return HB_EINVAL;
  return guarded(ctx, [&] {
    check_kernel(kernel);
    if (!cube || !tgt || !p_list || !err_out || np < 1) throw Error(HB_EINVAL, "interpolation_decay: bad arguments");
    check_cube(*cube);
    if (T < 1) throw Error(HB_EINVAL, "interpolation_decay: no targets");  // chebyshev.hpp:132
    for (int i = 0; i < np; ++i)
      if (p_list[i] < 0) throw Error(HB_EINVAL, "chebyshev_nodes: p must be >= 0");
    const int d = cube->d;
    for (int64_t i = 0; i < T; ++i) {  // HyperCube::dist (geometry.hpp:46-53) > 0 (chebyshev.hpp:153-155)
      double s = 0.0;
      for (int k = 0; k < d; ++k) {
        const double x = tgt[(int64_t)k * T + i];
        const double gap = std::max({0.0, cube->lower[k] - x, x - (cube->lower[k] + cube->side)});
        s += gap * gap;
      }
      if (!(std::sqrt(s) > 0.0)) throw Error(HB_EINVAL, "interpolation_decay: targets touch the cube");
    }
    HB_CUDA(cudaSetDevice(ctx->device));
    hb::interpolation_decay(ctx, *kernel, tgt, T, *cube, p_list, np, err_out);
  });
}

hb_status hb_fit_decay_rate(const int32_t* p, const double* err, int32_t n, double* rho_out) {
  return guarded(nullptr, [&] {  // chebyshev.hpp:180-193
    if (!p || !err || !rho_out) throw Error(HB_EINVAL, "fit_decay_rate: NULL argument");
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    int64_t k = 0;
    for (int32_t i = 0; i < n; ++i) {
      if (!(err[i] > 0)) continue;
      const double x = p[i], y = std::log(err[i]);
      sx += x;
      sy += y;
      sxx += x * x;
      sxy += x * y;
      ++k;
    }
    if (k < 2) throw Error(HB_EINVAL, "fit_decay_rate: need at least two positive errors");
    const double slope = (k * sxy - sx * sy) / (k * sxx - sx * sx);
    *rho_out = std::exp(-slope);
  });
}

hb_status hb_v_d_constant(int32_t d, double rho, double* out) {
  return guarded(nullptr, [&] {  // chebyshev.hpp:139-147
    if (!out) throw Error(HB_EINVAL, "v_d_constant: NULL output");
    if (d < 1) throw Error(HB_EINVAL, "v_d_constant: d must be >= 1");
    if (!(rho > 1.0)) throw Error(HB_EDOMAIN, "v_d_constant: rho must be > 1");
    double sum = static_cast<double>(d);
    const double q = 1.0 - 1.0 / rho;
    for (int l = 2; l <= d; ++l)
      sum += std::pow(2.0, l - 1) * ((l - 1) + std::pow(2.0, l - 1) - 1.0) / std::pow(q, l - 1);
    *out = sum;
  });
}

hb_status hb_assemble_dense_host(hb_context* ctx, const hb_kernel* kernel, const double* tgt, int64_t T,
                                 const double* src, int64_t N, int32_t d, double* K, int64_t ldk,
                                 int64_t entry_cap) {
  if (!ctx) return HB_EINVAL;
  return guarded(ctx, [&] {
    check_kernel(kernel);
    if (T <= 0 || N <= 0) throw Error(HB_EINVAL, "assemble_dense: empty point set");  // kernel.hpp:171
    if (d < 1 || d > 8) throw Error(HB_EINVAL, "assemble_dense: point dimensions differ");
    if (!tgt || !src || !K) throw Error(HB_EINVAL, "NULL buffer");
    if (ldk < T) throw Error(HB_EINVAL, "assemble_dense: ldk < T");
    if (entry_cap > 0 && T > entry_cap / N)  // kernel.hpp:174-175
      throw Error(HB_ECAP, "assemble_dense: T*N exceeds the entry cap");
    HB_CUDA(cudaSetDevice(ctx->device));
    const int64_t ldd = hb::round_up(T, 8);
    double* dx = hb::ws<double>(ctx, hb::B_X, (size_t)d * T);
    double* dy = hb::ws<double>(ctx, hb::B_Y, (size_t)d * N);
    double* dk = hb::ws<double>(ctx, hb::B_A, (size_t)ldd * N);
    HB_CUDA(cudaMemcpyAsync(dx, tgt, sizeof(double) * d * T, cudaMemcpyHostToDevice, ctx->stream));
    HB_CUDA(cudaMemcpyAsync(dy, src, sizeof(double) * d * N, cudaMemcpyHostToDevice, ctx->stream));
    unsigned int* flags = hb::ws<unsigned int>(ctx, hb::B_FLAGS, 4);
    HB_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned int), ctx->stream));
    hb::launch_assemble(*kernel, dx, T, dy, N, d, dk, ldd, flags, ctx->stream);
    raise_flags(read_flags(ctx, flags));
    HB_CUDA(cudaMemcpy2DAsync(K, ldk * 8, dk, ldd * 8, T * 8, N, cudaMemcpyDeviceToHost, ctx->stream));
    HB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

hb_status hb_eval_radial_host(const hb_kernel* k, double r, double* out) {
  return guarded(nullptr, [&] {
    check_kernel(k);
    if (!out) throw Error(HB_EINVAL, "NULL output");
    if (r == 0.0) {  // kernel.hpp:150-155
      if (k->has_diag) { *out = k->diag; return; }
      if (hb::kernel_singular_at_origin(k->id))
        throw Error(HB_ESINGULAR, "kernel eval: r == 0 on a singular kernel with no diagonal value");
    }
    switch (k->id) {  // kernel.hpp:93-109
      case HB_K_INVERSE_R: *out = 1.0 / r; break;
      case HB_K_LOG_R: *out = std::log(r); break;
      case HB_K_HELMHOLTZ3D_RE: *out = std::cos(r) / r; break;
      case HB_K_HELMHOLTZ3D_IM: *out = std::sin(r) / r; break;
      case HB_K_HANKEL_H12_RE: *out = hb::bessel_j2(r); break;  // bessel.hpp:129-135
      case HB_K_HANKEL_H12_IM: *out = hb::bessel_y2(r); break;  // bessel.hpp:137-144
      case HB_K_R: *out = r; break;
      case HB_K_SIN_R: *out = std::sin(r); break;
      case HB_K_INV_SQRT_1_PLUS_R: *out = 1.0 / std::sqrt(1.0 + r); break;
      case HB_K_EXP_NEG_R: *out = std::exp(-r); break;
      case HB_K_EXP_NEG_R2: *out = std::exp(-(r * r)); break;
      default: throw Error(HB_EUNSUPPORTED, "kernel not available");
    }
  });
}

hb_status hb_rank_matrix(hb_context* ctx, const double* d_A, int64_t m, int64_t n, int64_t ld,
                         const double* tols, int32_t ntol, hb_rank_result* out) {
  if (!ctx) return HB_EINVAL;
  return guarded(ctx, [&] {
    if (m < 1 || n < 1) throw Error(HB_EINVAL, "epsilon_rank: empty matrix");
    if (ld < m || !d_A || !out) throw Error(HB_EINVAL, "bad matrix arguments");
    check_tols(tols, ntol);
    HB_CUDA(cudaSetDevice(ctx->device));
    const int64_t lda = hb::round_up(m, 8);
    double* A = hb::ws<double>(ctx, hb::B_A, (size_t)lda * n);
    HB_CUDA(cudaMemcpy2DAsync(A, lda * 8, d_A, ld * 8, m * 8, n, cudaMemcpyDeviceToDevice, ctx->stream));
    unsigned int* flags = hb::ws<unsigned int>(ctx, hb::B_FLAGS, 4);
    HB_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned int), ctx->stream));
    hb::nonfinite_kernel<<<(unsigned)hb::ceil_div(m * n, 256), 256, 0, ctx->stream>>>(A, m, n, lda, flags);
    HB_LAUNCH_CHECK();
    raise_flags(read_flags(ctx, flags));  // SPEC.md:564 non-finite entries -> numeric error
    float fm = 0, cm = 0;
    hb::rank_matrix_inplace(ctx, A, m, n, lda, tols, ntol, out, &fm, &cm);
    for (int t = 0; t < ntol; ++t) out[t].sec[3] = (fm + cm) * 1e-3;
  });
}

hb_status hb_rank(hb_context* ctx, const hb_kernel* kernel, const hb_pair* pair, const double* tols,
                  int32_t ntol, hb_rank_result* out) {
  if (!ctx || !out) return HB_EINVAL;
  return guarded(ctx, [&] { rank_pair(ctx, kernel, pair, tols, ntol, out); });
}

hb_status hb_rank_complex(hb_context* ctx, const hb_kernel* kernel_re, const hb_kernel* kernel_im,
                          const hb_pair* pair, const double* tols, int32_t ntol, hb_rank_result* out) {
  if (!ctx || !out) return HB_EINVAL;
  return guarded(ctx, [&] { rank_pair_complex(ctx, kernel_re, kernel_im, pair, tols, ntol, out); });
}

hb_status hb_last_sigma(hb_context* ctx, double* host_out, int64_t max, int64_t* count) {
  if (!ctx || !count) return HB_EINVAL;
  return guarded(ctx, [&] {
    const int64_t k = ctx->last_k;
    *count = k;
    if (k == 0 || max <= 0 || !host_out) return;
    HB_CUDA(cudaSetDevice(ctx->device));
    double* d = hb::ws<double>(ctx, hb::B_D, (size_t)k + 1);
    double* e = hb::ws<double>(ctx, hb::B_E, (size_t)k + 1);
    double* o = hb::ws<double>(ctx, hb::B_BV, (size_t)2 * k + 8);
    hb::sigma_all_kernel<<<(unsigned)hb::ceil_div(k * 32, 256), 256, 0, ctx->stream>>>(
        d, e, k, ctx->last_sigma1, o);
    HB_LAUNCH_CHECK();
    const int64_t cnt = std::min(k, max);
    HB_CUDA(cudaMemcpyAsync(host_out, o, cnt * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    HB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

uint64_t hb_problem_seed(uint64_t base, int32_t d, int32_t d_prime, int64_t n) {
  const uint64_t key = ((uint64_t)d << 48) | ((uint64_t)(d_prime + 1) << 40) | (uint64_t)n;
  return hb::splitmix64(base ^ hb::splitmix64(key));
}

hb_status hb_partition(const hb_problem* probs, int64_t n, int32_t nparts, int32_t* owner) {
  if ((!probs && n > 0) || nparts < 1 || (!owner && n > 0) || n < 0) return HB_EINVAL;
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::vector<double> cost(n);
  for (int64_t i = 0; i < n; ++i) cost[i] = problem_cost(probs[i]);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return cost[a] > cost[b]; });
  std::vector<double> load(nparts, 0.0);
  for (int64_t i : order) {
    int best = 0;
    for (int p = 1; p < nparts; ++p)
      if (load[p] < load[best]) best = p;
    owner[i] = best;
    load[best] += cost[i];
  }
  return HB_OK;
}

static hb_context* cached_context(int device, int slot, hb_status* st) {
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    for (auto& e : g_cache)
      if (e.first.first == device && e.first.second == slot) return e.second;
  }
  hb_context* c = nullptr;
  *st = hb_context_create(device, &c);
  if (*st != HB_OK) return nullptr;
  std::lock_guard<std::mutex> lk(g_reg_mu);
  g_cache.push_back({{device, slot}, c});
  return c;
}

void hb_sweep_release(void) {
  std::vector<hb_context*> cs;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    for (auto& e : g_cache) cs.push_back(e.second);
    g_cache.clear();
  }
  for (auto* c : cs) hb_context_destroy(c);
}

static constexpr int64_t kSmallN = 16384;   // above this N a problem is "big" (K >= 2 GB)
static constexpr double kSmallRank = 1000.0; // HB_SOLO_BIG=1 only: solo above this predicted rank
static constexpr int kSubStreams = 4;      // concurrent streams per GPU (HB_SUBSTREAMS)
static constexpr int kMaxBig = 3;          // at most this many N > kSmallN problems in flight
static constexpr double kSoloFrac = 0.3;   // K above this share of device memory runs alone
static constexpr size_t kTrimBytes = size_t(16) << 30;  // after a big problem keep buffers <= this
static constexpr double kBudgetFrac = 0.88;  // admitted workspace, share of device memory

static int sub_streams() {
  static const int n = [] {
    const char* e = getenv("HB_SUBSTREAMS");
    const int v = e ? atoi(e) : kSubStreams;
    return v < 1 ? 1 : (v > 16 ? 16 : v);
  }();
  return n;
}

namespace {
// Device-memory admission shared by every sweep worker on one device (duplicate device entries
// in `devices` share it): the bytes reserved by running problems plus the workspace each stream
// keeps between problems must stay within kBudgetFrac of device memory.
struct DeviceBudget {
  std::mutex mu;
  std::condition_variable cv;
  double reserved = 0.0;  // Σ over streams of max(bytes held, bytes its running problem needs)
  int big_running = 0;
};
DeviceBudget& device_budget(int device) {
  static std::mutex m;
  static std::vector<std::pair<int, std::unique_ptr<DeviceBudget>>> all;
  std::lock_guard<std::mutex> lk(m);
  for (auto& e : all)
    if (e.first == device) return *e.second;
  all.emplace_back(device, std::make_unique<DeviceBudget>());
  return *all.back().second;
}

double held_bytes(const hb_context* c) {
  double s = 0.0;
  for (const auto& b : c->bufs) s += (double)b.cap;
  return s;
}

// Predicted peak workspace of one problem (rank_pair + rank_matrix_inplace): K, the
// certification copy of R_kᵀ (k ≈ 1.6 p̂), the k x k triangle, the sketch, V and W, with the
// 1/8 growth headroom of ws().
double problem_bytes(const hb_problem& p) {
  const double m = (double)p.pair.n_target, n = (double)p.pair.n_source;
  const double np = std::max(m, n);
  const double kh = std::min(std::min(m, n), 1.6 * predicted_rank(p.pair.target.d, p.pair.d_prime,
                                                                   (int64_t)np) + 128.0);
  const double lda = (double)hb::round_up((int64_t)m, 8);
  const double b = 8.0 * (lda * n + n * kh + kh * kh + np * 4.0 * 128.0 + 128.0 * m + 3.0 * 120.0 * np);
  return 1.125 * b + 64.0 * 1024 * 1024;
}
}  // namespace

hb_status hb_sweep_ex(const hb_problem* probs, int64_t n, const int32_t* devices, int32_t ndev,
                      hb_rank_result* out, int32_t* status_out, hb_sweep_opts* opts) {
  bool bad = n < 0 || (n > 0 && (!probs || !out)) || ndev < 1 || ndev > HB_MAX_DEVICES || !devices;
  for (int64_t i = 0; !bad && i < n; ++i) bad = probs[i].ntol < 1 || probs[i].ntol > HB_MAX_TOLS;
  if (bad) {  // report the failure per problem too, so a caller reading statuses sees it
    if (status_out)
      for (int64_t i = 0; i < n; ++i) status_out[i] = HB_EINVAL;
    return HB_EINVAL;
  }
  std::vector<int64_t> offset(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) offset[i + 1] = offset[i] + probs[i].ntol;
  std::vector<int32_t> owner(n);
  hb_partition(probs, n, ndev, owner.data());
  std::vector<hb_status> st(n, HB_OK);
  std::vector<double> cost(n);
  for (int64_t i = 0; i < n; ++i) cost[i] = problem_cost(probs[i]);
  std::vector<int> slot(ndev, 0);
  for (int w = 0; w < ndev; ++w)
    for (int v = 0; v < w; ++v)
      if (devices[v] == devices[w]) slot[w]++;
  auto worker = [&](int w) {
    hb_status cs = HB_OK;
    hb_context* c = cached_context(devices[w], slot[w], &cs);
    if (!c) {
      for (int64_t i = 0; i < n; ++i)
        if (owner[i] == w) st[i] = cs;
      return;
    }
    if (opts) c->profiling = opts->profiling != 0;
    std::vector<int64_t> mine;
    for (int64_t i = 0; i < n; ++i)
      if (owner[i] == w) mine.push_back(i);
    std::stable_sort(mine.begin(), mine.end(), [&](int64_t a, int64_t b) { return cost[a] > cost[b]; });
    cudaSetDevice(c->device);
    cudaEventRecord(c->ev[5], c->stream);
    DeviceBudget& bud = device_budget(c->device);
    const double budget = kBudgetFrac * (double)c->total_mem;
    // All problems share kSubStreams concurrent streams fed from one queue in cost order (LPT),
    // each stream's cooperative grids capped to a share of the SMs (the caps sum to <= #SMs, so
    // co-resident grid barriers cannot deadlock).  Big problems (N > kSmallN: K alone >= 2 GB)
    // are admitted at most kMaxBig at a time AND only while the device budget holds their
    // predicted workspace (problem_bytes) next to what the other streams hold or reserve; a
    // stream that finished a big problem frees its > kTrimBytes buffers.  Only a problem whose K
    // alone exceeds kSoloFrac of device memory runs by itself, first, with the whole GPU.
    // HB_SOLO_BIG=1 restores the round-1 policy (every problem with N > HB_SMALL_N or predicted
    // rank > HB_SMALL_RANK solo), for comparisons.
    static const int64_t small_n = [] {
      const char* e = getenv("HB_SMALL_N");
      return e ? (int64_t)atoll(e) : kSmallN;
    }();
    static const double small_rank = [] {
      const char* e = getenv("HB_SMALL_RANK");
      return e ? atof(e) : kSmallRank;
    }();
    static const bool solo_big = [] {
      const char* e = getenv("HB_SOLO_BIG");
      return e && atoi(e) != 0;
    }();
    auto np_of = [&](int64_t i) { return std::max(probs[i].pair.n_target, probs[i].pair.n_source); };
    auto is_big = [&](int64_t i) { return np_of(i) > small_n; };
    std::vector<int64_t> small;  // the shared queue, costliest first
    bool ran_solo = false;
    for (int64_t i : mine) {
      const hb_problem& p = probs[i];
      const int64_t np = np_of(i);
      const double k_bytes = 8.0 * (double)hb::round_up(p.pair.n_target, 8) * (double)p.pair.n_source;
      const bool solo = solo_big ? (np > small_n || predicted_rank(p.pair.target.d, p.pair.d_prime, np) > small_rank)
                                 : k_bytes > kSoloFrac * (double)c->total_mem;
      if (!solo) {
        small.push_back(i);
        continue;
      }
      {  // a solo problem waits until no other worker of this device holds a big reservation
        std::unique_lock<std::mutex> lk(bud.mu);
        bud.cv.wait(lk, [&] { return bud.big_running == 0; });
        bud.big_running++;
        bud.reserved += problem_bytes(p);
      }
      st[i] = hb_rank(c, &p.kernel, &p.pair, p.tols, p.ntol, out + offset[i]);
      ran_solo = true;
      {
        std::lock_guard<std::mutex> lk(bud.mu);
        bud.big_running--;
        bud.reserved -= problem_bytes(p);
      }
      bud.cv.notify_all();
    }
    if (ran_solo) {  // the main context only records events from here on: give its K back
      try {
        hb::context_trim(c, size_t(64) << 20);
      } catch (const hb::Error&) {
      }
    }
    std::vector<hb_context*> subs;
    if (!small.empty()) {
      cudaEvent_t ready;
      if (getenv("HB_TIMELINE")) cudaEventCreate(&ready);
      else cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
      cudaEventRecord(ready, c->stream);
      const int nsub = (int)std::min<size_t>(sub_streams(), small.size());
      // two-ended queue: the first nsub - nback streams take the costliest remaining problem, the
      // last nback streams the cheapest (latency-bound small problems start at t = 0 instead of
      // forming a tail after the large ones); HB_BACK_STREAMS, default 0
      static const int back_env = [] {
        const char* e = getenv("HB_BACK_STREAMS");
        return e ? std::max(0, atoi(e)) : 0;
      }();
      const int nback = std::min(back_env, nsub - 1);
      int64_t q_front = 0, q_back = (int64_t)small.size() - 1;
      static const int max_big = [] {  // HB_MAX_BIG: experiments
        const char* e = getenv("HB_MAX_BIG");
        return e ? std::max(1, atoi(e)) : kMaxBig;
      }();
      // per-stream reservation (bytes) in the device budget; guarded by bud.mu
      std::vector<double> res(nsub, 0.0);
      std::vector<hb_context*> sctx(nsub, nullptr);
      // take the next problem from the preferred end (else the other end); a big one only while
      // fewer than kMaxBig run and its workspace fits the device budget next to everything the
      // other streams hold — unless no big problem runs at all (progress).  Waits when nothing
      // can be admitted (or returns -2 when `wait` is false).  Lock order: bud.mu only.
      auto take_ex = [&](int s, bool from_back, bool wait) -> int64_t {
        std::unique_lock<std::mutex> lk(bud.mu);
        for (;;) {
          if (q_front > q_back) return -1;
          const int64_t a = from_back ? q_back : q_front, b = from_back ? q_front : q_back;
          const double held = sctx[s] ? held_bytes(sctx[s]) : 0.0;
          for (int64_t idx : {a, b}) {
            const hb_problem& p = probs[small[idx]];
            const double need = std::max(held, problem_bytes(p));
            if (is_big(small[idx])) {
              if (bud.big_running >= max_big) continue;
              if (bud.big_running > 0 && bud.reserved - res[s] + need > budget) continue;
              bud.big_running++;
            }
            bud.reserved += need - res[s];
            res[s] = need;
            if (idx == q_front) q_front++;
            else q_back--;
            return idx;
          }
          if (!wait) return -2;
          bud.cv.wait(lk);
        }
      };
      // after a problem: drop the reservation to what the stream keeps
      auto finished = [&](int s, int64_t q) {
        {
          std::lock_guard<std::mutex> lk(bud.mu);
          if (is_big(small[q])) bud.big_running--;
          const double keep = sctx[s] ? held_bytes(sctx[s]) : 0.0;
          bud.reserved += keep - res[s];
          res[s] = keep;
        }
        bud.cv.notify_all();
      };
      std::vector<hb_status> sctx_st(nsub, HB_OK);
      for (int s = 0; s < nsub; ++s)  // cached stream contexts: their kept workspace counts from the start
        sctx[s] = cached_context(devices[w], 1000 + slot[w] * 16 + s, &sctx_st[s]);
      std::vector<int64_t> first_q(nsub);  // stream 0 starts with the costliest problem
      for (int s = 0; s < nsub; ++s) first_q[s] = take_ex(s, s >= nsub - nback, false);
      std::vector<std::thread> sth;
      std::mutex sub_mu;
      std::vector<std::string> trace_lines;
      const double sweep_t0 = hb::host_now();
      auto sub_worker = [&](int s) {
        const hb_status ss = sctx_st[s];
        hb_context* sc = sctx[s];
        const bool from_back = s >= nsub - nback;
        auto take = [&] { return take_ex(s, from_back, true); };
        int64_t q0 = first_q[s] == -2 ? take() : first_q[s];
        if (!sc) {
          for (int64_t q = q0; q >= 0; q = take()) {
            st[small[q]] = ss;
            finished(s, q);
          }
          return;
        }
        {
          std::lock_guard<std::mutex> lk(sub_mu);
          subs.push_back(sc);
        }
        // stream 0 runs the costliest small problem (the critical path of the group) at high
        // stream priority with 35% of the SMs for its cooperative grids; the others share the
        // rest (caps sum to <= num_sms, so co-resident barriers cannot deadlock)
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        static const bool no_prio = getenv("HB_NO_PRIORITY") != nullptr;  // experiments
        if (no_prio) hi = lo;
        try {
          hb::context_set_priority(sc, (s == 0 && nsub > 1) ? hi : lo);
        } catch (const hb::Error&) {
        }
        static const double crit_share = [] {  // SM share of the critical stream's coop grids
          const char* e = getenv("HB_CRIT_SHARE");
          const double v = e ? atof(e) : 0.35;
          return v < 0.1 ? 0.1 : (v > 0.9 ? 0.9 : v);
        }();
        const int half = std::max(1, (int)(c->num_sms * crit_share));
        sc->coop_sms = nsub == 1 ? c->num_sms
                                 : (s == 0 ? half : std::max(1, (c->num_sms - half) / (nsub - 1)));
        sc->profiling = c->profiling;
        cudaStreamWaitEvent(sc->stream, ready, 0);
        static const bool timeline = getenv("HB_TIMELINE") != nullptr;
        for (int64_t q = q0; q >= 0; q = take()) {
          const hb_problem& p = probs[small[q]];
          cudaEvent_t e0 = nullptr, e1 = nullptr;
          if (timeline) {
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, sc->stream);
          }
          const bool ht = hb::host_trace_enabled();
          const hb::HostTrace h0 = hb::host_trace();
          const double t0 = ht ? hb::host_now() : 0.0;
          st[small[q]] = hb_rank(sc, &p.kernel, &p.pair, p.tols, p.ntol, out + offset[small[q]]);
          if (is_big(small[q]) || st[small[q]] == HB_ENOMEM) {
            // give the pool back the big buffers before the next admission
            try {
              hb::context_trim(sc, kTrimBytes);
            } catch (const hb::Error&) {
            }
          }
          finished(s, q);
          if (ht) {
            const hb::HostTrace& h1 = hb::host_trace();
            char buf[256];
            snprintf(buf, sizeof buf,
                     "[hosttrace] stream %d N=%lld d'=%d start %.2f wall %.2f sync %.2f (n %ld max %.2f) "
                     "coop %.2f (max %.2f) call %.2f @%s gap %.2f @%s ms\n",
                     s, (long long)p.pair.n_target, p.pair.d_prime, (t0 - sweep_t0) * 1e3,
                     (hb::host_now() - t0) * 1e3, (h1.sync_s - h0.sync_s) * 1e3, h1.n_sync - h0.n_sync,
                     h1.max_sync_s * 1e3, (h1.launch_s - h0.launch_s) * 1e3, h1.max_launch_s * 1e3,
                     h1.max_call_s * 1e3, h1.max_call_at, h1.max_gap_s * 1e3, h1.max_gap_at);
            hb::host_trace().max_call_s = hb::host_trace().max_gap_s = 0.0;
            hb::host_trace().max_sync_s = 0.0;
            hb::host_trace().max_launch_s = 0.0;
            std::lock_guard<std::mutex> lk(sub_mu);
            trace_lines.push_back(buf);
          }
          if (timeline) {  // HB_TIMELINE=1: per-problem device span on its sub-stream (stderr)
            cudaEventRecord(e1, sc->stream);
            cudaEventSynchronize(e1);
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, ready, e0);
            cudaEventElapsedTime(&b, ready, e1);
            fprintf(stderr, "[timeline] stream %d N=%lld d=%d d'=%d start %.2f end %.2f ms\n", s,
                    (long long)p.pair.n_target, p.pair.target.d, p.pair.d_prime, a, b);
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
          }
        }
        cudaEventRecord(sc->ev[5], sc->stream);
      };
      for (int s = 0; s < nsub; ++s) sth.emplace_back(sub_worker, s);
      for (auto& t : sth) t.join();
      for (auto& l : trace_lines) fputs(l.c_str(), stderr);
      for (auto* sc : subs) cudaStreamWaitEvent(c->stream, sc->ev[5], 0);
      cudaEventDestroy(ready);
      {  // this sweep's streams no longer reserve anything; what they keep is accounted when a
         // later sweep's stream takes its first problem
        std::lock_guard<std::mutex> lk(bud.mu);
        for (int s = 0; s < nsub; ++s) bud.reserved -= res[s];
      }
      bud.cv.notify_all();
    }
    // device span of this worker: first event to last completion on its streams
    cudaEvent_t end;
    cudaEventCreate(&end);
    cudaEventRecord(end, c->stream);
    cudaEventSynchronize(end);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[5], end);
    cudaEventDestroy(end);
    if (opts) opts->device_seconds[w] = ms * 1e-3;
  };
  std::vector<std::thread> th;
  for (int w = 1; w < ndev; ++w) th.emplace_back(worker, w);
  worker(0);
  for (auto& t : th) t.join();
  hb_status first = HB_OK;
  for (int64_t i = 0; i < n; ++i) {
    if (status_out) status_out[i] = st[i];
    if (first == HB_OK && st[i] != HB_OK) first = st[i];
  }
  return first;
}

hb_status hb_sweep(const hb_problem* probs, int64_t n, const int32_t* devices, int32_t ndev,
                   hb_rank_result* out, int32_t* status_out) {
  return hb_sweep_ex(probs, n, devices, ndev, out, status_out, nullptr);
}

}  // extern "C"

#include "hb_debug.h"

namespace {
void check_aca_args(const hb_kernel* kernel, const double* x, int64_t nt, const double* y, int64_t ns,
                    int32_t d, const hb_block* b) {
  check_kernel(kernel);
  if (!x || !y || !b) throw Error(HB_EINVAL, "aca: NULL argument");
  if (d < 1 || d > 8) throw Error(HB_EINVAL, "aca: bad dimension");
  if (b->rows == 0 || b->cols == 0) throw Error(HB_EINVAL, "aca::compress: empty block");  // aca.hpp:174-175
  if (b->rows < 0 || b->cols < 0 || b->row_begin < 0 || b->col_begin < 0 || b->row_begin + b->rows > nt ||
      b->col_begin + b->cols > ns)
    throw Error(HB_EINVAL, "aca: block outside the point sets");
}
}  // namespace

extern "C" hb_status hb_aca_compress(hb_context* ctx, const hb_kernel* kernel, const double* d_tgt, int64_t nt,
                                     const double* d_src, int64_t ns, int32_t d, const hb_block* blocks,
                                     int64_t nblocks, double eps, int64_t max_rank, hb_aca_factor** out) {
  if (!ctx || !out) return HB_EINVAL;
  return guarded(ctx, [&] {
    if (!(eps > 0)) throw Error(HB_EINVAL, "aca::compress: epsilon must be positive");   // aca.hpp:172
    if (max_rank < 1) throw Error(HB_EINVAL, "aca::compress: max_rank must be >= 1");  // aca.hpp:173
    if (nblocks < 1 || !blocks) throw Error(HB_EINVAL, "aca: no blocks");
    for (int64_t i = 0; i < nblocks; ++i) check_aca_args(kernel, d_tgt, nt, d_src, ns, d, blocks + i);
    for (int64_t i = 0; i < nblocks; ++i) out[i] = nullptr;
    HB_CUDA(cudaSetDevice(ctx->device));
    hb::aca_compress(ctx, *kernel, d_tgt, nt, d_src, ns, d, blocks, nblocks, eps, max_rank, out);
  });
}

extern "C" hb_status hb_aca_factor_info(const hb_aca_factor* f, int32_t* rank, int32_t* met, int64_t* mem) {
  if (!f) return HB_EINVAL;
  if (rank) *rank = f->rank;
  if (met) *met = f->met;
  if (mem)  // aca.hpp:58-61
    *mem = 2 * (int64_t)f->rank * f->rank * (int64_t)sizeof(double) + 2 * (int64_t)f->rank * (int64_t)sizeof(int64_t);
  return HB_OK;
}

extern "C" hb_status hb_aca_factor_copy(const hb_aca_factor* f, int64_t* sigma, int64_t* tau, double* L, double* U) {
  if (!f) return HB_EINVAL;
  return guarded(nullptr, [&] {
    const size_t r = (size_t)f->rank;
    if (sigma && r) std::memcpy(sigma, f->sigma.data(), r * sizeof(int64_t));
    if (tau && r) std::memcpy(tau, f->tau.data(), r * sizeof(int64_t));
    HB_CUDA(cudaSetDevice(f->device));
    if (L && r) HB_CUDA(cudaMemcpy(L, f->L, r * r * sizeof(double), cudaMemcpyDeviceToHost));
    if (U && r) HB_CUDA(cudaMemcpy(U, f->U, r * r * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

extern "C" hb_status hb_aca_apply(hb_context* ctx, const hb_aca_factor* f, const hb_kernel* kernel,
                                  const double* d_tgt, int64_t nt, const double* d_src, int64_t ns, int32_t d,
                                  const hb_block* block, const double* d_q, double* d_b) {
  if (!ctx || !f) return HB_EINVAL;
  return guarded(ctx, [&] {
    check_aca_args(kernel, d_tgt, nt, d_src, ns, d, block);
    if (!d_q || !d_b) throw Error(HB_EINVAL, "aca::apply: NULL vector");
    for (int32_t k = 0; k < f->rank; ++k)
      if (f->sigma[(size_t)k] < block->row_begin || f->sigma[(size_t)k] >= block->row_begin + block->rows ||
          f->tau[(size_t)k] < block->col_begin || f->tau[(size_t)k] >= block->col_begin + block->cols)
        throw Error(HB_EINVAL, "aca::apply: factor pivots outside the block");
    HB_CUDA(cudaSetDevice(ctx->device));
    hb::aca_apply(ctx, f, *kernel, d_tgt, nt, d_src, ns, d, *block, d_q, d_b);
  });
}

extern "C" void hb_aca_factor_destroy(hb_aca_factor* f) {
  if (!f) return;
  cudaSetDevice(f->device);
  delete f;
}

extern "C" hb_status hb_debug_dgemm_async(hb_context* ctx, int32_t transA, int64_t M, int64_t N,
                                          int64_t K, double alpha, const double* A, int64_t lda,
                                          const double* B, int64_t ldb, double beta, double* C,
                                          int64_t ldc, int32_t reps) {
  if (!ctx) return HB_EINVAL;
  return guarded(ctx, [&] {
    if (M < 0 || N < 0 || K < 0) throw Error(HB_EINVAL, "negative size");
    HB_CUDA(cudaSetDevice(ctx->device));
    hb::GemmArgs g{};
    g.M = M; g.N = N; g.K = K; g.alpha = alpha; g.A = A; g.lda = lda; g.transA = transA != 0;
    g.B = B; g.ldb = ldb; g.beta = beta; g.C = C; g.ldc = ldc;
    const int64_t wse = 8ll << 20;
    double* sk = hb::ws<double>(ctx, hb::B_SPLITK, wse);
    for (int r = 0; r < reps; ++r) hb::launch_dgemm(g, sk, wse, ctx->num_sms, ctx->stream);
  });
}

extern "C" hb_status hb_debug_dgemm(hb_context* ctx, int32_t transA, int64_t M, int64_t N, int64_t K,
                                    double alpha, const double* A, int64_t lda, const double* B,
                                    int64_t ldb, double beta, double* C, int64_t ldc) {
  hb_status s = hb_debug_dgemm_async(ctx, transA, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, 1);
  if (s != HB_OK) return s;
  return guarded(ctx, [&] { HB_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

extern "C" hb_status hb_debug_dgemm_fro(hb_context* ctx, int32_t transA, int64_t M, int64_t N, int64_t K,
                                        double alpha, const double* A, int64_t lda, const double* B,
                                        int64_t ldb, double beta, double* C, int64_t ldc, int64_t fro_row0,
                                        double* fro_out) {
  if (!ctx || !fro_out) return HB_EINVAL;
  return guarded(ctx, [&] {
    if (M < 0 || N < 0 || K < 0) throw Error(HB_EINVAL, "negative size");
    HB_CUDA(cudaSetDevice(ctx->device));
    const int64_t cnt = hb::gemm_fro_count(M, N, K, ctx->num_sms);
    double* parts = hb::ws<double>(ctx, hb::B_FRO, (size_t)cnt);
    double* sum = hb::ws<double>(ctx, hb::B_FROSUM, 8);
    hb::GemmArgs g{};
    g.M = M; g.N = N; g.K = K; g.alpha = alpha; g.A = A; g.lda = lda; g.transA = transA != 0;
    g.B = B; g.ldb = ldb; g.beta = beta; g.C = C; g.ldc = ldc;
    g.fro_partials = parts;
    g.fro_row0 = fro_row0;
    const int64_t wse = 8ll << 20;
    double* sk = hb::ws<double>(ctx, hb::B_SPLITK, wse);
    hb::launch_dgemm(g, sk, wse, ctx->num_sms, ctx->stream);
    hb::sum_kernel<<<1, 1024, 0, ctx->stream>>>(parts, cnt, sum);
    HB_LAUNCH_CHECK();
    HB_CUDA(cudaMemcpyAsync(fro_out, sum, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    HB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

