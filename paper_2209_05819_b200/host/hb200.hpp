// hb200.hpp — C++ host mirror of the reference interface for the rank-reveal path, over the C ABI
// (include/hb.h).  Same names, argument meaning and error behaviour as the reference headers, so
// a caller of hodlr::KernelSpec / HyperCube / InteractionClass / (SPEC) pair_geometry,
// epsilon_rank, rank_table can switch to hb200:: with the device doing the work.
//
//   hb200::KernelId / KernelSpec / kernel_from_string / kernel_name / eval_radial
//        <- hodlr::KernelId, KernelSpec, kernel_from_string, kernel_name, eval_radial
//           (/root/reference/proj/include/hodlr/kernel.hpp:19-157)
//   hb200::HyperCube, InteractionClass   <- hodlr::HyperCube, InteractionClass (geometry.hpp:15-104)
//   hb200::BoxIndex, classify_pair       <- hodlr::BoxIndex, classify_pair (geometry.hpp:66-71, 106-118)
//   hb200::assemble_dense                <- hodlr::assemble_dense (kernel.hpp:168-181), host
//                                           PointSets in, host column-major Matrix out
//   hb200::HMatrix, BuildReport, AdmissibilityPolicy
//        <- hodlr::HMatrix::initialize / matvec (hmatrix.hpp:19-179, cluster_tree.hpp:17-29)
//   hb200::chebyshev_nodes, interpolation_decay, fit_decay_rate, v_d_constant
//        <- chebyshev.hpp:16-23, 139-193
//   hb200::fit_growth                    <- SPEC fit_growth
//   hb200::pair_geometry, epsilon_rank, rank_table, RankRecord, write_csv
//        <- SPEC rankbench module (CSV schema SPEC.md:613)
// Exceptions follow the reference: std::invalid_argument (HB_EINVAL), std::length_error
// (HB_ECAP), std::domain_error (HB_EDOMAIN), std::runtime_error (HB_ESINGULAR and device
// errors).  KernelId::Custom (a std::function) cannot run on the device: EUNSUPPORTED ->
// std::invalid_argument with an explanatory message.
#pragma once

#include <cstdint>
#include <optional>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hb.h"

namespace hb200 {

inline void check(hb_status s, const char* where, const hb_context* ctx = nullptr) {
  if (s == HB_OK) return;
  std::string msg = std::string(where) + ": " + hb_status_string(s);
  const char* detail = hb_last_error(ctx);
  if (detail && *detail) msg += std::string(" (") + detail + ")";
  switch (s) {
    case HB_EINVAL:
    case HB_EUNSUPPORTED: throw std::invalid_argument(msg);
    case HB_ECAP: throw std::length_error(msg);
    case HB_EDOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}

enum class KernelId {
  InverseR, LogR, Helmholtz3DReal, Helmholtz3DImag, HankelH12Real, HankelH12Imag, R, SinR,
  InvSqrt1PlusR, ExpNegR, ExpNegR2, Custom,
};

struct KernelSpec {
  KernelId id = KernelId::Custom;
  std::optional<double> diagonal_value;

  static KernelSpec catalog(KernelId id) {  // kernel.hpp:40-67
    if (id == KernelId::Custom)
      throw std::invalid_argument("KernelSpec::catalog: Custom has no catalog entry");
    KernelSpec s;
    s.id = id;
    switch (id) {
      case KernelId::Helmholtz3DImag:
      case KernelId::InvSqrt1PlusR:
      case KernelId::ExpNegR:
      case KernelId::ExpNegR2: s.diagonal_value = 1.0; break;
      default: s.diagonal_value = 0.0; break;
    }
    return s;
  }
  bool singular_at_origin() const {
    return id == KernelId::InverseR || id == KernelId::LogR || id == KernelId::Helmholtz3DReal ||
           id == KernelId::HankelH12Imag || (id == KernelId::Custom && !diagonal_value);
  }
  hb_kernel to_c() const {
    hb_kernel k{};
    k.id = static_cast<int32_t>(id);
    k.has_diag = diagonal_value.has_value();
    k.diag = diagonal_value.value_or(0.0);
    return k;
  }
};

inline const std::vector<std::pair<std::string, KernelId>>& kernel_names() {
  static const std::vector<std::pair<std::string, KernelId>> t = {
      {"one_over_r", KernelId::InverseR}, {"log_r", KernelId::LogR},
      {"helmholtz3d_re", KernelId::Helmholtz3DReal}, {"helmholtz3d_im", KernelId::Helmholtz3DImag},
      {"hankel_h12_re", KernelId::HankelH12Real}, {"hankel_h12_im", KernelId::HankelH12Imag},
      {"r", KernelId::R}, {"sin_r", KernelId::SinR}, {"inv_sqrt_1_plus_r", KernelId::InvSqrt1PlusR},
      {"exp_neg_r", KernelId::ExpNegR}, {"exp_neg_r2", KernelId::ExpNegR2}};
  return t;
}

inline KernelSpec kernel_from_string(const std::string& name) {  // kernel.hpp:112-129
  for (const auto& [key, id] : kernel_names())
    if (name == key) return KernelSpec::catalog(id);
  throw std::invalid_argument("unknown kernel id: " + name);
}

inline std::string kernel_name(const KernelSpec& spec) {
  for (const auto& [key, id] : kernel_names())
    if (spec.id == id) return key;
  return "custom";
}

inline double eval_radial(const KernelSpec& spec, double r) {  // kernel.hpp:149-157
  const hb_kernel k = spec.to_c();
  double out = 0.0;
  check(hb_eval_radial_host(&k, r, &out), "eval_radial");
  return out;
}

struct HyperCube {  // geometry.hpp:15-64
  std::vector<double> lower;
  double side = 1.0;
  HyperCube() = default;
  HyperCube(std::vector<double> lower_corner, double side_length)
      : lower(std::move(lower_corner)), side(side_length) {
    if (!(side > 0.0)) throw std::invalid_argument("HyperCube: side must be positive");
    if (lower.empty() || lower.size() > 8) throw std::invalid_argument("HyperCube: 1 <= d <= 8");
  }
  int dim() const { return static_cast<int>(lower.size()); }
  hb_cube to_c() const {
    hb_cube c{};
    c.d = dim();
    for (int k = 0; k < dim(); ++k) c.lower[k] = lower[k];
    c.side = side;
    return c;
  }
};

struct InteractionClass {  // geometry.hpp:77-104
  enum class Kind { SelfBlock, SharedSurface, FarField };
  Kind kind = Kind::SelfBlock;
  int surface_dim = -1;
  static InteractionClass self_block() { return {Kind::SelfBlock, -1}; }
  static InteractionClass shared_surface(int d_prime) { return {Kind::SharedSurface, d_prime}; }
  static InteractionClass far_field() { return {Kind::FarField, -1}; }
  bool is_self() const { return kind == Kind::SelfBlock; }
  bool is_far() const { return kind == Kind::FarField; }
  bool is_vertex() const { return kind == Kind::SharedSurface && surface_dim == 0; }
  bool shares_surface(int d_prime) const { return kind == Kind::SharedSurface && surface_dim == d_prime; }
  friend bool operator==(const InteractionClass& a, const InteractionClass& b) {
    return a.kind == b.kind && (a.kind != Kind::SharedSurface || a.surface_dim == b.surface_dim);
  }
  // hb_pair.d_prime encoding: HB_DPRIME_SELF (-2), HB_DPRIME_FAR (-1) or d'
  int32_t dprime() const { return is_self() ? HB_DPRIME_SELF : (is_far() ? HB_DPRIME_FAR : surface_dim); }
  static InteractionClass from_c(hb_interaction ic) {
    if (ic.kind == HB_IC_SELF) return self_block();
    if (ic.kind == HB_IC_FAR) return far_field();
    return shared_surface(ic.surface_dim);
  }
  std::string name() const {
    switch (kind) {
      case Kind::SelfBlock: return "self";
      case Kind::FarField: return "far";
      default: return "surface:" + std::to_string(surface_dim);
    }
  }
  static InteractionClass parse(const std::string& s) {
    if (s == "far") return far_field();
    if (s == "self") return self_block();
    if (s.rfind("surface:", 0) == 0) return shared_surface(std::stoi(s.substr(8)));
    if (s == "vertex") return shared_surface(0);
    throw std::invalid_argument("unknown interaction: " + s);
  }
};

// BoxIndex (geometry.hpp:66-71): level + per-axis grid coordinate in [0, 2^level).
struct BoxIndex {
  int level = 0;
  std::vector<int32_t> grid;
  int dim() const { return static_cast<int>(grid.size()); }
};

// classify_pair (geometry.hpp:106-118): self / far (any offset >= 2) / surface:#zero offsets.
inline InteractionClass classify_pair(const BoxIndex& a, const BoxIndex& b) {
  if (a.grid.size() != b.grid.size())
    throw std::invalid_argument("classify_pair: boxes have different dimensions");
  hb_interaction ic{};
  check(hb_classify_pair(a.dim(), a.level, a.grid.data(), b.level, b.grid.data(), &ic), "classify_pair");
  return InteractionClass::from_c(ic);
}

// The same for two cubes of one uniform subdivision (equal sides, integer offsets).
inline InteractionClass classify_pair(const HyperCube& a, const HyperCube& b) {
  const hb_cube ca = a.to_c(), cb = b.to_c();
  hb_interaction ic{};
  check(hb_classify_cubes(&ca, &cb, &ic), "classify_pair");
  return InteractionClass::from_c(ic);
}

enum class PointMode { Uniform = HB_POINTS_UNIFORM, GridInterior = HB_POINTS_GRID_INTERIOR,
                       GridClosed = HB_POINTS_GRID_CLOSED };

// SPEC pair_geometry: target cube [0,1]^d; source = target + o with
// o = (2,0,..,0) far-field or d-d' leading ones for a d'-dimensional shared surface.
struct PairGeometry {
  int d = 1;
  InteractionClass interaction;
  HyperCube target, source;
  int64_t n = 0;
  PointMode mode = PointMode::Uniform;
  uint64_t seed = 0;
  hb_pair to_c() const {
    hb_pair p{};
    p.target = target.to_c();
    p.source = source.to_c();
    p.d_prime = interaction.dprime();
    p.point_mode = static_cast<int32_t>(mode);
    p.n_target = n;
    p.n_source = n;
    p.seed = seed;
    return p;
  }
};

inline PairGeometry pair_geometry(int d, InteractionClass inter, int64_t n,
                                  PointMode mode = PointMode::Uniform, uint64_t seed = 0) {
  if (d < 1 || d > 8) throw std::invalid_argument("pair_geometry: 1 <= d <= 8");
  if (inter.kind == InteractionClass::Kind::SelfBlock)
    throw std::invalid_argument("pair_geometry: self interaction is not a cube pair");
  if (!inter.is_far() && (inter.surface_dim < 0 || inter.surface_dim > d - 1))
    throw std::invalid_argument("pair_geometry: invalid d'");
  std::vector<double> o(d, 0.0);
  if (inter.is_far()) o[0] = 2.0;
  else
    for (int k = 0; k < d - inter.surface_dim; ++k) o[k] = 1.0;
  PairGeometry g;
  g.d = d;
  g.interaction = inter;
  g.target = HyperCube(std::vector<double>(d, 0.0), 1.0);
  g.source = HyperCube(o, 1.0);
  g.n = n;
  g.mode = mode;
  g.seed = seed;
  return g;
}

inline uint64_t problem_seed(uint64_t base, int d, const InteractionClass& inter, int64_t n) {
  return hb_problem_seed(base, d, inter.dprime(), n);
}

// SPEC RankRecord + certification data.
struct RankRecord {
  std::string kernel;
  int d = 0;
  InteractionClass interaction;
  int64_t N = 0;
  double epsilon = 0.0;
  int rank = 0;
  int rank_lo = 0, rank_hi = 0, k_factored = 0;
  double sigma1 = 0.0, sigma_r = 0.0, sigma_r1 = 0.0, gap = 0.0;
  double seconds = 0.0;
  double fp_band = 0.0;  // sqrt(N)·u·‖A‖_F / thr: gap < fp_band means rounding could move the count
};

// RAII device context (one per device and host thread).
class Device {
 public:
  explicit Device(int device = 0) { check(hb_context_create(device, &ctx_), "hb_context_create"); }
  ~Device() { hb_context_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  hb_context* get() const { return ctx_; }

 private:
  hb_context* ctx_ = nullptr;
};

// PointSet (types.hpp:14-15): column-major, points are rows -> coordinate k of point i at k*n + i.
struct PointSet {
  int64_t n = 0;
  int d = 0;
  std::vector<double> soa;
};

// Matrix (types.hpp:11): column-major rows x cols.
struct Matrix {
  int64_t rows = 0, cols = 0;
  std::vector<double> data;
  double operator()(int64_t i, int64_t j) const { return data[(size_t)(j * rows + i)]; }
};

// assemble_dense (kernel.hpp:168-181): K(i, j) = F(‖targets_i − sources_j‖), assembled on the
// device from host point sets, returned as a host column-major Matrix.  Same exceptions:
// empty set / dimension mismatch -> invalid_argument, T·N > entry_cap -> length_error,
// r == 0 on a singular kernel without a diagonal value -> runtime_error.
inline Matrix assemble_dense(Device& dev, const KernelSpec& spec, const PointSet& targets,
                             const PointSet& sources, int64_t entry_cap = 400'000'000) {
  if (targets.n == 0 || sources.n == 0) throw std::invalid_argument("assemble_dense: empty point set");
  if (targets.d != sources.d) throw std::invalid_argument("assemble_dense: point dimensions differ");
  Matrix K;
  K.rows = targets.n;
  K.cols = sources.n;
  K.data.resize((size_t)(targets.n * sources.n));
  const hb_kernel ck = spec.to_c();
  check(hb_assemble_dense_host(dev.get(), &ck, targets.soa.data(), targets.n, sources.soa.data(),
                               sources.n, targets.d, K.data.data(), K.rows, entry_cap),
        "assemble_dense", dev.get());
  return K;
}

// SPEC epsilon_rank of one generated block: count of σ_k > eps·σ₁.
inline std::vector<RankRecord> epsilon_rank(Device& dev, const KernelSpec& k, const PairGeometry& g,
                                            const std::vector<double>& eps) {
  if (eps.empty() || eps.size() > HB_MAX_TOLS) throw std::invalid_argument("need 1..4 tolerances");
  const hb_kernel ck = k.to_c();
  const hb_pair cp = g.to_c();
  std::vector<hb_rank_result> out(eps.size());
  check(hb_rank(dev.get(), &ck, &cp, eps.data(), (int32_t)eps.size(), out.data()), "epsilon_rank",
        dev.get());
  std::vector<RankRecord> recs;
  for (size_t t = 0; t < eps.size(); ++t) {
    RankRecord r;
    r.kernel = kernel_name(k); r.d = g.d; r.interaction = g.interaction; r.N = g.n;
    r.epsilon = eps[t]; r.rank = out[t].rank; r.rank_lo = out[t].rank_lo; r.rank_hi = out[t].rank_hi;
    r.k_factored = out[t].k_factored; r.sigma1 = out[t].sigma1; r.sigma_r = out[t].sigma_r;
    r.sigma_r1 = out[t].sigma_r1; r.gap = out[t].gap; r.seconds = out[t].sec[3];
    r.fp_band = out[t].fp_band;
    recs.push_back(r);
  }
  return recs;
}

// ε-rank of the complex block K_re + i·K_im (the paper's F3 / F4 columns, PAPER.md:121-131;
// e.g. Helmholtz3DReal + i·Helmholtz3DImag = e^{ir}/r, HankelH12Real + i·HankelH12Imag = H_2^(1)).
inline std::vector<RankRecord> epsilon_rank_complex(Device& dev, const KernelSpec& re, const KernelSpec& im,
                                                    const PairGeometry& g, const std::vector<double>& eps) {
  if (eps.empty() || eps.size() > HB_MAX_TOLS) throw std::invalid_argument("need 1..4 tolerances");
  const hb_kernel cr = re.to_c(), ci = im.to_c();
  const hb_pair cp = g.to_c();
  std::vector<hb_rank_result> out(eps.size());
  check(hb_rank_complex(dev.get(), &cr, &ci, &cp, eps.data(), (int32_t)eps.size(), out.data()),
        "epsilon_rank_complex", dev.get());
  std::vector<RankRecord> recs;
  for (size_t t = 0; t < eps.size(); ++t) {
    RankRecord r;
    r.kernel = kernel_name(re) + "+i*" + kernel_name(im); r.d = g.d; r.interaction = g.interaction;
    r.N = g.n; r.epsilon = eps[t]; r.rank = out[t].rank; r.rank_lo = out[t].rank_lo;
    r.rank_hi = out[t].rank_hi; r.k_factored = out[t].k_factored; r.sigma1 = out[t].sigma1;
    r.sigma_r = out[t].sigma_r; r.sigma_r1 = out[t].sigma_r1; r.gap = out[t].gap;
    r.seconds = out[t].sec[3];
    recs.push_back(r);
  }
  return recs;
}

// SPEC epsilon_rank(matrix, epsilon) on a device matrix (column-major m x n, leading dim ld).
inline int epsilon_rank(Device& dev, const double* d_matrix, int64_t m, int64_t n, int64_t ld,
                        double eps) {
  hb_rank_result r{};
  check(hb_rank_matrix(dev.get(), d_matrix, m, n, ld, &eps, 1, &r), "epsilon_rank", dev.get());
  return r.rank;
}

// SPEC fit_growth: rank(N) against constant / a + b ln N / a N^c.
struct GrowthFit {
  std::string best;  // "constant" | "log" | "power"
  double constant = 0, log_a = 0, log_b = 0, pow_a = 0, pow_c = 0, rss[3] = {0, 0, 0}, max_min_ratio = 0;
};
inline GrowthFit fit_growth(const std::vector<RankRecord>& recs) {
  std::vector<int64_t> ns;
  std::vector<double> rk;
  for (const auto& r : recs) {
    ns.push_back(r.N);
    rk.push_back((double)r.rank);
  }
  hb_growth_fit f{};
  check(hb_fit_growth(ns.data(), rk.data(), (int32_t)ns.size(), &f), "fit_growth");
  static const char* names[3] = {"constant", "log", "power"};
  GrowthFit g;
  g.best = names[f.best];
  g.constant = f.constant; g.log_a = f.log_a; g.log_b = f.log_b; g.pow_a = f.pow_a; g.pow_c = f.pow_c;
  for (int k = 0; k < 3; ++k) g.rss[k] = f.rss[k];
  g.max_min_ratio = f.max_min_ratio;
  return g;
}

// SPEC rank_table: one record per (kernel, N), problems spread over the
// given devices by hb_sweep (LPT partition, one worker thread per device).
inline std::vector<RankRecord> rank_table(const std::vector<KernelSpec>& kernels,
                                          const InteractionClass& inter, int d,
                                          const std::vector<int64_t>& n_list, double epsilon,
                                          const std::vector<int>& devices = {0},
                                          PointMode mode = PointMode::Uniform, uint64_t base_seed = 0,
                                          std::vector<hb_status>* statuses = nullptr) {
  std::vector<hb_problem> probs;
  std::vector<RankRecord> recs;
  for (const auto& k : kernels)
    for (int64_t n : n_list) {
      const uint64_t seed = mode == PointMode::Uniform ? problem_seed(base_seed, d, inter, n) : base_seed;
      const PairGeometry g = pair_geometry(d, inter, n, mode, seed);
      hb_problem p{};
      p.kernel = k.to_c();
      p.pair = g.to_c();
      p.tols[0] = epsilon;
      p.ntol = 1;
      probs.push_back(p);
      RankRecord r;
      r.kernel = kernel_name(k); r.d = d; r.interaction = inter; r.N = n; r.epsilon = epsilon;
      recs.push_back(r);
    }
  std::vector<hb_rank_result> out(probs.size());
  std::vector<int32_t> st(probs.size(), 0);
  std::vector<int32_t> devs(devices.begin(), devices.end());
  hb_sweep(probs.data(), (int64_t)probs.size(), devs.data(), (int32_t)devs.size(), out.data(), st.data());
  for (size_t i = 0; i < probs.size(); ++i) {
    auto& r = recs[i];
    r.rank = out[i].rank; r.rank_lo = out[i].rank_lo; r.rank_hi = out[i].rank_hi;
    r.k_factored = out[i].k_factored; r.sigma1 = out[i].sigma1; r.sigma_r = out[i].sigma_r;
    r.sigma_r1 = out[i].sigma_r1; r.gap = out[i].gap; r.seconds = out[i].sec[3];
    if (statuses) statuses->push_back(static_cast<hb_status>(st[i]));
  }
  return recs;
}

// CSV schema of SPEC.md:613 (+ certification columns).
inline void write_csv_header(std::ostream& os) {
  os << "kernel,d,interaction,dprime,N,epsilon,rank,seconds,rank_lo,rank_hi,k_factored,sigma1,gap\n";
}
inline void write_csv_row(std::ostream& os, const RankRecord& r) {
  os << r.kernel << ',' << r.d << ',' << r.interaction.name() << ','
     << (r.interaction.is_far() ? -1 : r.interaction.surface_dim) << ',' << r.N << ',' << r.epsilon
     << ',' << r.rank << ',' << r.seconds << ',' << r.rank_lo << ',' << r.rank_hi << ','
     << r.k_factored << ',' << r.sigma1 << ',' << r.gap << '\n';
}

// ---- ACA (aca.hpp:16-213) on device point sets --------------------------------------------------
// BlockSpec: K(I, J) over SoA device point sets (coordinate k of point i at k*n + i).
struct BlockSpec {  // aca.hpp:16-28
  const KernelSpec* kernel = nullptr;
  const double* targets = nullptr;  // device, d x nt
  const double* sources = nullptr;  // device, d x ns
  int64_t nt = 0, ns = 0;
  int d = 0;
  int64_t row_begin = 0, rows = 0, col_begin = 0, cols = 0;
  hb_block to_c() const { return hb_block{row_begin, rows, col_begin, cols}; }
};

// ACAFactor (aca.hpp:50-62): pivot ids and r x r LU factors (host copies; the device handle
// stays alive for apply()).
struct ACAFactor {
  std::vector<int64_t> sigma, tau;
  std::vector<double> L, U;  // column-major rank x rank
  int rank = 0;
  bool tolerance_met = true;
  std::shared_ptr<hb_aca_factor> handle;
  int64_t memory_bytes() const {  // aca.hpp:58-61
    return 2 * (int64_t)rank * rank * (int64_t)sizeof(double) + 2 * (int64_t)rank * (int64_t)sizeof(int64_t);
  }
};

// compress (aca.hpp:171-198) of several blocks of the same point sets in one call.
inline std::vector<ACAFactor> compress(Device& dev, const std::vector<BlockSpec>& blocks, double epsilon,
                                       int64_t max_rank) {
  if (blocks.empty()) return {};
  const BlockSpec& b0 = blocks.front();
  if (!b0.kernel) throw std::invalid_argument("aca::compress: BlockSpec without a kernel");
  std::vector<hb_block> cb;
  for (const auto& b : blocks) {
    if (b.kernel != b0.kernel || b.targets != b0.targets || b.sources != b0.sources)
      throw std::invalid_argument("aca::compress: blocks of one call share kernel and point sets");
    cb.push_back(b.to_c());
  }
  const hb_kernel ck = b0.kernel->to_c();
  std::vector<hb_aca_factor*> raw(blocks.size(), nullptr);
  check(hb_aca_compress(dev.get(), &ck, b0.targets, b0.nt, b0.sources, b0.ns, b0.d, cb.data(),
                        (int64_t)cb.size(), epsilon, max_rank, raw.data()),
        "aca::compress", dev.get());
  std::vector<ACAFactor> out;
  for (hb_aca_factor* h : raw) {
    ACAFactor f;
    f.handle = std::shared_ptr<hb_aca_factor>(h, hb_aca_factor_destroy);
    int32_t r = 0, met = 0;
    check(hb_aca_factor_info(h, &r, &met, nullptr), "aca::compress");
    f.rank = r;
    f.tolerance_met = met != 0;
    f.sigma.resize(r);
    f.tau.resize(r);
    f.L.resize((size_t)r * r);
    f.U.resize((size_t)r * r);
    check(hb_aca_factor_copy(h, f.sigma.data(), f.tau.data(), f.L.data(), f.U.data()), "aca::compress");
    out.push_back(std::move(f));
  }
  return out;
}

inline ACAFactor compress(Device& dev, const BlockSpec& block, double epsilon, int64_t max_rank) {
  return compress(dev, std::vector<BlockSpec>{block}, epsilon, max_rank).front();
}

// apply (aca.hpp:202-213): b = K(I, τ) U⁻¹ L⁻¹ K(σ, J) q for device vectors q (cols), b (rows).
inline void apply(Device& dev, const ACAFactor& f, const BlockSpec& block, const double* d_q, double* d_b) {
  const hb_kernel ck = block.kernel->to_c();
  const hb_block cb = block.to_c();
  check(hb_aca_apply(dev.get(), f.handle.get(), &ck, block.targets, block.nt, block.sources, block.ns,
                     block.d, &cb, d_q, d_b),
        "aca::apply", dev.get());
}

// ---- HODLRdD operator (hmatrix.hpp) ----------------------------------------------------------
enum class AdmissibilityPolicy { WeakDD = HB_POLICY_WEAKDD, Strong = HB_POLICY_STRONG, WeakAll = HB_POLICY_WEAKALL };
using BuildReport = hb_build_report;  // hmatrix.hpp:19-26

// HMatrix::initialize + matvec on the device: the tree, block structure, dense leaf / near blocks
// and ACA factors live on the device of `dev` (which must outlive the operator).
class HMatrix {
 public:
  static std::pair<HMatrix, BuildReport> initialize(Device& dev, const PointSet& points, const HyperCube& domain,
                                                    const KernelSpec& kernel, AdmissibilityPolicy policy,
                                                    int64_t n_max, double epsilon, int64_t max_rank = 1 << 14,
                                                    int64_t dense_entry_cap = 400'000'000) {
    HMatrix h;
    h.n_ = points.n;
    const hb_kernel ck = kernel.to_c();
    const hb_cube cd = domain.to_c();
    BuildReport rep{};
    hb_hmatrix* raw = nullptr;
    check(hb_hmatrix_build(dev.get(), &ck, points.soa.data(), points.n, points.d, &cd, (int32_t)policy, n_max,
                           epsilon, max_rank, dense_entry_cap, &raw, &rep),
          "HMatrix::initialize", dev.get());
    h.h_.reset(raw, [](hb_hmatrix* p) { hb_hmatrix_destroy(p); });
    h.dev_ = dev.get();
    return {std::move(h), rep};
  }
  int64_t size() const { return n_; }
  // b = K q in the original point ordering (hmatrix.hpp:133-179)
  std::vector<double> matvec(const std::vector<double>& q) const {
    if ((int64_t)q.size() != n_) throw std::invalid_argument("HMatrix::matvec: length mismatch");
    std::vector<double> b((size_t)n_);
    check(hb_hmatrix_matvec(h_.get(), q.data(), b.data(), 1), "HMatrix::matvec", dev_);
    return b;
  }
  int64_t original_id(int64_t tree_id) const {  // ClusterTree::original_id
    std::vector<int64_t> o((size_t)n_);
    check(hb_hmatrix_tree_order(h_.get(), o.data()), "HMatrix::original_id");
    return o.at((size_t)tree_id);
  }

 private:
  std::shared_ptr<hb_hmatrix> h_;
  hb_context* dev_ = nullptr;
  int64_t n_ = 0;
};

// ---- Chebyshev interpolation bound check (chebyshev.hpp:16-23, 139-193) ---------------------
inline std::vector<double> chebyshev_nodes(int p) {
  std::vector<double> y((size_t)std::max(p + 1, 1));
  check(hb_chebyshev_nodes(p, y.data()), "chebyshev_nodes");
  return y;
}
inline std::vector<std::pair<int, double>> interpolation_decay(Device& dev, const KernelSpec& spec,
                                                               const PointSet& targets, const HyperCube& cube,
                                                               const std::vector<int>& p_list) {
  const hb_kernel ck = spec.to_c();
  const hb_cube cc = cube.to_c();
  std::vector<int32_t> ps(p_list.begin(), p_list.end());
  std::vector<double> err(ps.size());
  check(hb_interpolation_decay(dev.get(), &ck, targets.soa.data(), targets.n, &cc, ps.data(), (int32_t)ps.size(),
                               err.data()),
        "interpolation_decay", dev.get());
  std::vector<std::pair<int, double>> out;
  for (size_t i = 0; i < ps.size(); ++i) out.emplace_back(ps[i], err[i]);
  return out;
}
inline double fit_decay_rate(const std::vector<std::pair<int, double>>& decay) {
  std::vector<int32_t> p;
  std::vector<double> e;
  for (const auto& [pp, ee] : decay) {
    p.push_back(pp);
    e.push_back(ee);
  }
  double rho = 0.0;
  check(hb_fit_decay_rate(p.data(), e.data(), (int32_t)p.size(), &rho), "fit_decay_rate");
  return rho;
}
inline double v_d_constant(int d, double rho) {
  double v = 0.0;
  check(hb_v_d_constant(d, rho, &v), "v_d_constant");
  return v;
}

}  // namespace hb200

