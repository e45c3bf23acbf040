// ref_wrap.cpp -- TEST INFRASTRUCTURE ONLY.  extern "C" wrapper that compiles the reference's
// own headers (kernel.hpp, aca.hpp, bessel.hpp, geometry.hpp, chebyshev.hpp, cluster_tree.hpp,
// hmatrix.hpp, types.hpp) from where they lie under
// /root/reference/proj/include, against the from-scratch Eigen subset in oracle/eigen_shim,
// into oracle/_ref/libhb_ref.so.  No reference source is copied into this repository.
// It is the second oracle: tests pin the C restatement (hb_oracle.c) against it, and
// tests/golden/make_aca_golden.py freezes its outputs as fixtures for the GPU box (where
// /root/reference does not exist).
#include <cstdint>
#include <cstring>
#include <stdexcept>

#include "hodlr/aca.hpp"
#include "hodlr/chebyshev.hpp"
#include "hodlr/geometry.hpp"
#include "hodlr/hmatrix.hpp"
#include "hodlr/kernel.hpp"

using namespace hodlr;

namespace {
// status codes of include/hb.h
enum { OK = 0, EINVAL_ = 1, EDOMAIN_ = 2, ECAP_ = 3, ESINGULAR_ = 4, EUNSUPPORTED_ = 5 };

KernelSpec spec_of(int id, int has_diag, double diag) {
  KernelSpec s = KernelSpec::catalog(static_cast<KernelId>(id));  // kernel.hpp:42-67
  if (has_diag)
    s.diagonal_value = diag;
  else
    s.diagonal_value.reset();
  return s;
}

PointSet soa_to_pointset(const double* soa, int64_t n, int d) {
  PointSet p(n, d);  // column-major N x d == SoA
  std::memcpy(p.data(), soa, sizeof(double) * (size_t)(n * d));
  return p;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return OK;
  } catch (const std::invalid_argument&) {
    return EINVAL_;
  } catch (const std::length_error&) {
    return ECAP_;
  } catch (const std::domain_error&) {
    return EDOMAIN_;
  } catch (const std::runtime_error&) {
    return ESINGULAR_;
  } catch (...) {
    return EUNSUPPORTED_;
  }
}
}  // namespace

extern "C" {

double hbr_eval_radial(int id, int has_diag, double diag, double r, int* status) {
  double out = 0.0;
  *status = guarded([&] { out = eval_radial(spec_of(id, has_diag, diag), r); });
  return out;
}

double hbr_j2(double x) { return bessel::j2(x); }
double hbr_y2(double x) { return bessel::y2(x); }

// hodlr::assemble_dense (kernel.hpp:168-181) -> K column-major T x N.
int hbr_assemble_dense(int id, int has_diag, double diag, const double* x_soa, int64_t T,
                       const double* y_soa, int64_t N, int d, double* K, int64_t entry_cap) {
  return guarded([&] {
    const KernelSpec s = spec_of(id, has_diag, diag);
    const Matrix k = assemble_dense(s, soa_to_pointset(x_soa, T, d), soa_to_pointset(y_soa, N, d),
                                    entry_cap);
    std::memcpy(K, k.data(), sizeof(double) * (size_t)(T * N));
  });
}

// hodlr::compress (aca.hpp:171-198) on BlockSpec(kernel, targets, rb, rows, sources, cb, cols)
// (aca.hpp:26-28), and optionally hodlr::apply (aca.hpp:202-213) to q (length cols) -> b (rows).
// Outputs: sigma/tau (global ids), L/U column-major r x r, capacity `cap` pivots.
int hbr_aca_compress(int id, int has_diag, double diag, const double* x_soa, int64_t nt,
                     const double* y_soa, int64_t ns, int d, int64_t rb, int64_t rows, int64_t cb,
                     int64_t cols, double eps, int64_t max_rank, int64_t cap, int64_t* sigma,
                     int64_t* tau, double* L, double* U, int32_t* rank, int32_t* met,
                     const double* q, double* b) {
  return guarded([&] {
    const KernelSpec s = spec_of(id, has_diag, diag);
    const PointSet X = soa_to_pointset(x_soa, nt, d), Y = soa_to_pointset(y_soa, ns, d);
    const BlockSpec blk(s, X, rb, rows, Y, cb, cols);
    const ACAFactor f = compress(blk, eps, max_rank);
    if (f.rank > cap) throw std::length_error("hbr_aca_compress: capacity");
    *rank = f.rank;
    *met = f.tolerance_met ? 1 : 0;
    for (int k = 0; k < f.rank; ++k) {
      sigma[k] = f.sigma[(size_t)k];
      tau[k] = f.tau[(size_t)k];
    }
    for (int j = 0; j < f.rank; ++j)
      for (int i = 0; i < f.rank; ++i) {
        L[i + (int64_t)j * f.rank] = f.L(i, j);
        U[i + (int64_t)j * f.rank] = f.U(i, j);
      }
    if (q && b) {
      Vector qq(cols);
      for (int64_t j = 0; j < cols; ++j) qq(j) = q[j];
      const Vector bb = apply(f, blk, qq);
      for (int64_t i = 0; i < rows; ++i) b[i] = bb(i);
    }
  });
}

// hodlr::classify_pair (geometry.hpp:109-118) on two BoxIndex values; kind 0 self, 1 shared
// surface (surface_dim = d'), 2 far (hb.h HB_IC_*).
int hbr_classify_pair(int d, int level_a, const int32_t* grid_a, int level_b, const int32_t* grid_b,
                      int32_t* kind, int32_t* surface_dim) {
  return guarded([&] {
    BoxIndex a, b;
    a.level = level_a;
    b.level = level_b;
    a.grid = Eigen::ArrayXi::Zero(d);
    b.grid = Eigen::ArrayXi::Zero(d);
    for (int k = 0; k < d; ++k) {
      a.grid(k) = grid_a[k];
      b.grid(k) = grid_b[k];
    }
    const InteractionClass ic = classify_pair(a, b);
    *kind = ic.is_self() ? 0 : (ic.is_far() ? 2 : 1);
    *surface_dim = ic.surface_dim;
  });
}

// hodlr::box_grid / box_id (geometry.hpp:123-141): z-order box id <-> per-axis grid.
int hbr_box_grid(int d, int level, int64_t id, int32_t* grid) {
  return guarded([&] {
    const Eigen::ArrayXi g = box_grid(d, level, id);
    for (int k = 0; k < d; ++k) grid[k] = g(k);
  });
}

// ---- chebyshev.hpp ------------------------------------------------------------------------
int hbr_chebyshev_nodes(int p, double* out) {
  return guarded([&] {
    const Vector y = chebyshev_nodes(p);
    for (Index i = 0; i < y.size(); ++i) out[i] = y(i);
  });
}

int hbr_lagrange_weights(const double* nodes, int m, double y, double* out) {
  return guarded([&] {
    Vector nd(m);
    for (int i = 0; i < m; ++i) nd(i) = nodes[i];
    const Vector w = lagrange_weights(nd, y);
    for (int i = 0; i < m; ++i) out[i] = w(i);
  });
}

// interpolation_decay (chebyshev.hpp:151-177): max |K - U V| over the sample grid per degree.
int hbr_interpolation_decay(int id, int has_diag, double diag, const double* x_soa, int64_t T, int d,
                            const double* lower, double side, const int32_t* p_list, int np,
                            double* err_out) {
  return guarded([&] {
    const KernelSpec s = spec_of(id, has_diag, diag);
    Point lo(d);
    for (int a = 0; a < d; ++a) lo(a) = lower[a];
    const HyperCube cube(lo, side);
    std::vector<int> ps(p_list, p_list + np);
    const auto dec = interpolation_decay(s, soa_to_pointset(x_soa, T, d), cube, ps);
    for (int i = 0; i < np; ++i) err_out[i] = dec[(size_t)i].second;
  });
}

int hbr_fit_decay_rate(const int32_t* p, const double* err, int n, double* rho) {
  return guarded([&] {
    std::vector<std::pair<int, double>> dec;
    for (int i = 0; i < n; ++i) dec.emplace_back(p[i], err[i]);
    *rho = fit_decay_rate(dec);
  });
}

int hbr_v_d_constant(int d, double rho, double* out) {
  return guarded([&] { *out = v_d_constant(d, rho); });
}

// ---- cluster_tree.hpp / hmatrix.hpp ---------------------------------------------------------
// HMatrix::initialize (hmatrix.hpp:50-126) + matvec (hmatrix.hpp:133-179) on nq vectors
// (column-major N x nq), single-threaded.  report: [max_block_rank, num_low_rank_blocks,
// num_dense_entries, num_tolerance_failures, memory_bytes, depth].  perm: tree -> original id.
int hbr_hmatrix_matvec(int id, int has_diag, double diag, const double* pts_soa, int64_t N, int d,
                       const double* lower, double side, int policy, int64_t n_max, double eps,
                       int64_t max_rank, const double* q, int nq, double* b, int64_t* report,
                       int64_t* perm) {
  return guarded([&] {
    const KernelSpec s = spec_of(id, has_diag, diag);
    Point lo(d);
    for (int a = 0; a < d; ++a) lo(a) = lower[a];
    const HyperCube dom(lo, side);
    HMatrixOptions opts;
    opts.max_rank = max_rank;
    auto [h, rep] = HMatrix::initialize(soa_to_pointset(pts_soa, N, d), dom, s,
                                        static_cast<AdmissibilityPolicy>(policy), n_max, eps, opts);
    for (int c = 0; c < nq; ++c) {
      Vector qq(N);
      for (int64_t i = 0; i < N; ++i) qq(i) = q[i + c * N];
      const Vector bb = h.matvec(qq);
      for (int64_t i = 0; i < N; ++i) b[i + c * N] = bb(i);
    }
    report[0] = rep.max_block_rank;
    report[1] = rep.num_low_rank_blocks;
    report[2] = rep.num_dense_entries;
    report[3] = rep.num_tolerance_failures;
    report[4] = rep.memory_bytes;
    report[5] = h.tree().depth();
    if (perm)
      for (int64_t t = 0; t < N; ++t) perm[t] = h.tree().original_id(t);
  });
}

}  // extern "C"
