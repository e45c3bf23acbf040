// Device J2 / Y2 (hodlr::bessel::j2 / y2, bessel.hpp:25-144) for the HankelH12Real / Imag
// kernels (kernel.hpp:26-27, 100-101).  The reference sums the x <= 19 ascending series in
// __float128 (113-bit) because the alternating series loses ~e^x ulps to cancellation; the GPU
// has no binary128, so the same series run in double-double (106-bit, error-free transforms on
// the FP64 pipe: two-sum / fma two-product).  The x > 19 Hankel asymptotic expansion (long double
// in the reference) runs in double-double for P, Q and uses cos/sin(x − (2ν+1)π/4) expanded with
// the exact constants ±√2/2.  Results agree with the reference to ~1 ulp on the series branch;
// on the asymptotic branch to ~2e-16 · sqrt(2/(πx)) absolute (tests/test_gpu_entries.py).
#pragma once
#include <cuda_runtime.h>

#include <cmath>

// __host__ __device__: the host build (hb_eval_radial_host) runs the same double-double code;
// x86-64 host code has no FMA contraction, fma() is the libm correctly rounded one.
#ifdef __CUDA_ARCH__
#define HB_DADD(a, b) __dadd_rn(a, b)
#define HB_DSUB(a, b) __dsub_rn(a, b)
#define HB_DMUL(a, b) __dmul_rn(a, b)
#define HB_DDIV(a, b) __ddiv_rn(a, b)
#define HB_FMA(a, b, c) __fma_rn(a, b, c)
#else
#define HB_DADD(a, b) ((a) + (b))
#define HB_DSUB(a, b) ((a) - (b))
#define HB_DMUL(a, b) ((a) * (b))
#define HB_DDIV(a, b) ((a) / (b))
#define HB_FMA(a, b, c) std::fma(a, b, c)
#endif
#define HB_HD __host__ __device__

namespace hb {

struct ddv {
  double hi, lo;
};

HB_HD inline ddv dd_two_sum(double a, double b) {
  const double s = HB_DADD(a, b);
  const double bb = HB_DSUB(s, a);
  const double e = HB_DADD(HB_DSUB(a, HB_DSUB(s, bb)), HB_DSUB(b, bb));
  return {s, e};
}
HB_HD inline ddv dd_quick(double a, double b) {  // |a| >= |b|
  const double s = HB_DADD(a, b);
  return {s, HB_DSUB(b, HB_DSUB(s, a))};
}
HB_HD inline ddv dd_prod(double a, double b) {
  const double p = HB_DMUL(a, b);
  return {p, HB_FMA(a, b, -p)};
}
HB_HD inline ddv dd_add(ddv a, ddv b) {
  ddv s = dd_two_sum(a.hi, b.hi);
  const ddv t = dd_two_sum(a.lo, b.lo);
  s.lo = HB_DADD(s.lo, t.hi);
  s = dd_quick(s.hi, s.lo);
  s.lo = HB_DADD(s.lo, t.lo);
  return dd_quick(s.hi, s.lo);
}
HB_HD inline ddv dd_neg(ddv a) { return {-a.hi, -a.lo}; }
HB_HD inline ddv dd_sub(ddv a, ddv b) { return dd_add(a, dd_neg(b)); }
HB_HD inline ddv dd_mul(ddv a, ddv b) {
  ddv p = dd_prod(a.hi, b.hi);
  p.lo = HB_FMA(a.hi, b.lo, p.lo);
  p.lo = HB_FMA(a.lo, b.hi, p.lo);
  return dd_quick(p.hi, p.lo);
}
HB_HD inline ddv dd_mul_d(ddv a, double b) {
  ddv p = dd_prod(a.hi, b);
  p.lo = HB_FMA(a.lo, b, p.lo);
  return dd_quick(p.hi, p.lo);
}
HB_HD inline ddv dd_div(ddv a, ddv b) {
  const double q1 = HB_DDIV(a.hi, b.hi);
  ddv r = dd_sub(a, dd_mul_d(b, q1));
  const double q2 = HB_DDIV(r.hi, b.hi);
  r = dd_sub(r, dd_mul_d(b, q2));
  const double q3 = HB_DDIV(r.hi, b.hi);
  return dd_add(dd_quick(q1, q2), ddv{q3, 0.0});
}
HB_HD inline ddv dd_div_d(ddv a, double b) { return dd_div(a, ddv{b, 0.0}); }
HB_HD inline ddv dd_d(double a) { return {a, 0.0}; }

constexpr double kDdPiHi = 3.141592653589793, kDdPiLo = 1.2246467991473532e-16;
constexpr double kDdLn2Hi = 0.6931471805599453, kDdLn2Lo = 2.3190468138462996e-17;
constexpr double kDdGammaHi = 0.5772156649015329, kDdGammaLo = -4.942915152430645e-18;

// exp(x) in double-double: x = k ln2 + r, |r| <= ln2/2, Taylor to 1e-33.
HB_HD inline ddv dd_exp(ddv x) {
  const double k = std::rint(HB_DDIV(x.hi, kDdLn2Hi));
  const ddv r = dd_sub(x, dd_mul_d(ddv{kDdLn2Hi, kDdLn2Lo}, k));
  ddv term = dd_d(1.0), s = dd_d(1.0);
  for (int n = 1; n < 40; ++n) {
    term = dd_div_d(dd_mul(term, r), (double)n);
    s = dd_add(s, term);
    if (std::fabs(term.hi) < 1e-34 * std::fabs(s.hi)) break;
  }
  return {std::scalbn(s.hi, (int)k), std::scalbn(s.lo, (int)k)};
}
// log(a) for a double a > 0: Newton step on exp from the double log.
HB_HD inline ddv dd_log(double a) {
  const double y = std::log(a);
  const ddv e = dd_exp(dd_d(-y));             // exp(-y)
  const ddv t = dd_sub(dd_mul_d(e, a), dd_d(1.0));  // a exp(-y) - 1
  return dd_add(dd_d(y), t);                  // log a = y + log(1 + t) ≈ y + t − t²/2
}

// bessel.hpp:45-56 (J_nu ascending series), nu = 0, 1, 2.
HB_HD inline ddv dd_j_series(int nu, double x) {
  const ddv h = dd_d(0.5 * x), h2 = dd_prod(h.hi, h.hi);
  ddv term = dd_d(1.0);
  for (int k = 1; k <= nu; ++k) term = dd_mul(term, dd_div_d(h, (double)k));
  ddv s = term;
  const ddv mh2 = dd_neg(h2);
  for (int m = 1; m < 400; ++m) {
    term = dd_mul(term, dd_div_d(mh2, (double)m * (double)(m + nu)));
    s = dd_add(s, term);
    if (m > 4 && std::fabs(term.hi) < 1e-32 * std::fabs(s.hi)) break;
  }
  return s;
}

// bessel.hpp:59-86 (Y0, Y1 ascending series, harmonic-number form)
HB_HD inline void dd_y01_series(double x, ddv& y0, ddv& y1) {
  const ddv pi{kDdPiHi, kDdPiLo};
  const ddv h = dd_d(0.5 * x), h2 = dd_prod(h.hi, h.hi);
  const ddv lg = dd_add(dd_log(h.hi), ddv{kDdGammaHi, kDdGammaLo});
  const ddv j0 = dd_j_series(0, x), j1 = dd_j_series(1, x);
  ddv s = dd_d(0.0), term = dd_d(1.0), hk = dd_d(0.0);
  for (int k = 1; k < 400; ++k) {
    term = dd_mul(term, dd_div_d(h2, (double)k * (double)k));
    hk = dd_add(hk, dd_div_d(dd_d(1.0), (double)k));
    const ddv c = dd_mul((k % 2) ? term : dd_neg(term), hk);
    s = dd_add(s, c);
    if (k > 4 && std::fabs(c.hi) < 1e-32 * std::fabs(s.hi)) break;
  }
  const ddv two_pi = dd_div(dd_d(2.0), pi);
  y0 = dd_mul(two_pi, dd_add(dd_mul(lg, j0), s));
  ddv s1 = dd_d(0.0), t1 = dd_d(1.0), ha = dd_d(0.0), hb = dd_d(1.0);
  for (int k = 0; k < 400; ++k) {
    if (k > 0) {
      t1 = dd_mul(t1, dd_div_d(h2, (double)k * (double)(k + 1)));
      ha = dd_add(ha, dd_div_d(dd_d(1.0), (double)k));
      hb = dd_add(hb, dd_div_d(dd_d(1.0), (double)(k + 1)));
    }
    const ddv c = dd_mul((k % 2) ? dd_neg(t1) : t1, dd_add(ha, hb));
    s1 = dd_add(s1, c);
    if (k > 4 && std::fabs(c.hi) < 1e-32 * std::fabs(s1.hi)) break;
  }
  // y1 = (2/π) lg j1 − 2/(π x) − h/π s1
  y1 = dd_sub(dd_sub(dd_mul(dd_mul(two_pi, lg), j1), dd_div(dd_d(2.0), dd_mul_d(pi, x))),
              dd_mul(dd_div(h, pi), s1));
}

// bessel.hpp:89-107, P and Q truncated at the smallest term (double-double for long double)
HB_HD inline void dd_asym_pq(int nu, double x, double& p, double& q) {
  const double mu = 4.0 * nu * nu;
  const ddv x2 = dd_mul_d(dd_prod(x, x), 64.0);
  ddv ps = dd_d(1.0), qs = dd_div(dd_d(mu - 1.0), dd_d(8.0 * x));
  ddv tp = dd_d(1.0), tq = qs;
  for (int k = 1; k < 40; ++k) {
    const double a = 4.0 * k - 3, b = 4.0 * k - 1, c = 4.0 * k + 1;
    const ddv np_num = dd_neg(dd_mul(dd_d(mu - a * a), dd_d(mu - b * b)));
    const ddv nq_num = dd_neg(dd_mul(dd_d(mu - b * b), dd_d(mu - c * c)));
    const ddv ntp = dd_div(dd_mul(tp, np_num), dd_mul_d(x2, (2.0 * k - 1) * (2.0 * k)));
    const ddv ntq = dd_div(dd_mul(tq, nq_num), dd_mul_d(x2, (2.0 * k) * (2.0 * k + 1)));
    if (std::fabs(ntp.hi) >= std::fabs(tp.hi) || std::fabs(ntq.hi) >= std::fabs(tq.hi)) break;
    ps = dd_add(ps, ntp);
    qs = dd_add(qs, ntq);
    tp = ntp;
    tq = ntq;
    if (std::fabs(ntp.hi) < 1e-24 && std::fabs(ntq.hi) < 1e-24) break;
  }
  p = ps.hi;
  q = qs.hi;
}

// sqrt(2/(πx)) [P cos χ − Q sin χ] (J) or [P sin χ + Q cos χ] (Y), χ = x − (2ν+1)π/4,
// cos χ / sin χ from sincos(x) and the exact ±√2/2 of (2ν+1)π/4 (bessel.hpp:111-125)
HB_HD inline double dd_asymptotic(int nu, double x, bool y) {
  double p, q;
  dd_asym_pq(nu, x, p, q);
  double sx, cx;
  sx = std::sin(x);
  cx = std::cos(x);
  const double r2 = 0.7071067811865476;
  // (2ν+1)π/4 for ν = 0, 1, 2: cos = +, −, −; sin = +, +, −  (times √2/2)
  const double cc = (nu == 0) ? r2 : -r2, sc = (nu == 2) ? -r2 : r2;
  const ddv cchi = dd_add(dd_mul_d(dd_d(cx), cc), dd_mul_d(dd_d(sx), sc));  // cos x cos c + sin x sin c
  const ddv schi = dd_sub(dd_mul_d(dd_d(sx), cc), dd_mul_d(dd_d(cx), sc));  // sin x cos c − cos x sin c
  const ddv v = y ? dd_add(dd_mul_d(schi, p), dd_mul_d(cchi, q)) : dd_sub(dd_mul_d(cchi, p), dd_mul_d(schi, q));
  return HB_DMUL(std::sqrt(HB_DDIV(2.0, HB_DMUL(3.141592653589793, x))), v.hi);
}

HB_HD inline double bessel_j2(double x) {  // bessel.hpp:129-135
  if (x == 0.0) return 0.0;
  if (x <= 19.0) return dd_j_series(2, x).hi;
  return dd_asymptotic(2, x, false);
}

HB_HD inline double bessel_y2(double x) {  // bessel.hpp:137-144
  if (x <= 19.0) {
    ddv y0, y1;
    dd_y01_series(x, y0, y1);
    return dd_sub(dd_mul(dd_div(dd_d(2.0), dd_d(x)), y1), y0).hi;
  }
  return HB_DSUB(HB_DMUL(HB_DDIV(2.0, x), dd_asymptotic(1, x, true)), dd_asymptotic(0, x, true));
}

}  // namespace hb
