// Device-side entry rule shared by k2 (assembly) and the ACA kernels: F(r) of
// KernelSpec::operator() (kernel.hpp:93-109) and eval_radial's r == 0 rule (kernel.hpp:149-157),
// with r = ||x - y||_2 as a left-to-right sum of separately rounded squares (kernel.hpp:179).
#pragma once
#include "common.cuh"
#include "bessel_dd.cuh"

namespace hb {

template <int KID>
__device__ __forceinline__ double radial(double r) {
  if (KID == HB_K_INVERSE_R) return __ddiv_rn(1.0, r);
  if (KID == HB_K_LOG_R) return log(r);
  if (KID == HB_K_HELMHOLTZ3D_RE) return __ddiv_rn(cos(r), r);
  if (KID == HB_K_HELMHOLTZ3D_IM) return __ddiv_rn(sin(r), r);
  if (KID == HB_K_HANKEL_H12_RE) return bessel_j2(r);
  if (KID == HB_K_HANKEL_H12_IM) return bessel_y2(r);
  if (KID == HB_K_R) return r;
  if (KID == HB_K_SIN_R) return sin(r);
  if (KID == HB_K_INV_SQRT_1_PLUS_R) return __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(1.0, r)));
  if (KID == HB_K_EXP_NEG_R) return exp(-r);
  if (KID == HB_K_EXP_NEG_R2) return exp(-__dmul_rn(r, r));
  return 0.0;
}

// Runtime kernel id (ACA evaluates one row / column per pivot; the switch is not the bound).
__device__ __forceinline__ double radial_rt(int id, double r) {
  switch (id) {
    case HB_K_INVERSE_R: return radial<HB_K_INVERSE_R>(r);
    case HB_K_LOG_R: return radial<HB_K_LOG_R>(r);
    case HB_K_HELMHOLTZ3D_RE: return radial<HB_K_HELMHOLTZ3D_RE>(r);
    case HB_K_HELMHOLTZ3D_IM: return radial<HB_K_HELMHOLTZ3D_IM>(r);
    case HB_K_HANKEL_H12_RE: return radial<HB_K_HANKEL_H12_RE>(r);
    case HB_K_HANKEL_H12_IM: return radial<HB_K_HANKEL_H12_IM>(r);
    case HB_K_R: return radial<HB_K_R>(r);
    case HB_K_SIN_R: return radial<HB_K_SIN_R>(r);
    case HB_K_INV_SQRT_1_PLUS_R: return radial<HB_K_INV_SQRT_1_PLUS_R>(r);
    case HB_K_EXP_NEG_R: return radial<HB_K_EXP_NEG_R>(r);
    case HB_K_EXP_NEG_R2: return radial<HB_K_EXP_NEG_R2>(r);
    default: return 0.0;
  }
}

// Kernel descriptor as the device sees it.
struct DevKernel {
  int id;
  int has_diag;
  int singular;  // singular at r == 0 without a diagonal value (kernel.hpp:76-89)
  double diag;
};

// eval_radial(spec, ||x_i - y_j||) for SoA point sets (coordinate k of point i at k*nx + i).
// *bad |= 1 on r == 0 for a singular kernel without a diagonal (runtime_error in the reference).
__device__ __forceinline__ double entry_soa(const DevKernel& K, const double* __restrict__ x,
                                            int64_t nx, int64_t i, const double* __restrict__ y,
                                            int64_t ny, int64_t j, int d, unsigned int* bad) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    const double df = __dsub_rn(x[(int64_t)k * nx + i], y[(int64_t)k * ny + j]);
    const double sq = __dmul_rn(df, df);
    s = (k == 0) ? sq : __dadd_rn(s, sq);
  }
  const double r = __dsqrt_rn(s);
  if (r == 0.0) {
    if (K.has_diag) return K.diag;
    if (K.singular) {
      *bad |= 1u;
      return 0.0;
    }
  }
  return radial_rt(K.id, r);
}

}  // namespace hb
