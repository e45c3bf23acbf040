/*
 * hb_oracle.c -- CPU ORACLE, TEST INFRASTRUCTURE ONLY (see hb_oracle.h for the citations and
 * the rule on who may call it).  Compiled with -ffp-contract=off so that every multiply and
 * add rounds separately, exactly as the device kernel pins it with __dmul_rn/__dadd_rn.
 */
#include "hb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

uint64_t hbo_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static int64_t int_root(int64_t n, int d) {
  /* exact integer d-th root or -1 */
  int64_t r = (int64_t)llround(pow((double)n, 1.0 / d));
  for (int64_t c = (r > 2 ? r - 2 : 1); c <= r + 2; ++c) {
    int64_t p = 1;
    for (int k = 0; k < d; ++k) p *= c;
    if (p == n) return c;
  }
  return -1;
}

int hbo_points(int d, const double* lower, double side, int64_t n, int mode, uint64_t seed,
               int role, double* out) {
  if (d < 1 || d > 8 || n < 1 || !(side > 0.0)) return HBO_EINVAL; /* geometry.hpp:22 */
  if (mode == HBO_UNIFORM) {
    const uint64_t stream = hbo_splitmix64(seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(role + 1)));
    for (int k = 0; k < d; ++k)
      for (int64_t i = 0; i < n; ++i) {
        const uint64_t bits = hbo_splitmix64(stream + (uint64_t)i * 8u + (uint64_t)k);
        const double u = ((double)(bits >> 12) + 0.5) * 0x1p-52; /* exact, in (0,1) */
        const double s = side * u;
        out[(int64_t)k * n + i] = lower[k] + s;
      }
    return HBO_OK;
  }
  if (mode != HBO_GRID_INTERIOR && mode != HBO_GRID_CLOSED) return HBO_EINVAL;
  const int64_t m = int_root(n, d);
  if (m < 1) return HBO_EINVAL; /* N must be a perfect d-th power */
  if (mode == HBO_GRID_CLOSED && m < 2) return HBO_EINVAL;
  for (int64_t i = 0; i < n; ++i) {
    int64_t rest = i;
    for (int k = 0; k < d; ++k) {
      const int64_t g = rest % m;
      rest /= m;
      const double t = (mode == HBO_GRID_INTERIOR) ? (double)(g + 1) / (double)(m + 1)
                                                   : (double)g / (double)(m - 1);
      const double s = side * t;
      out[(int64_t)k * n + i] = lower[k] + s;
    }
  }
  return HBO_OK;
}

double hbo_distance(int d, const double* x, int64_t i, int64_t nx, const double* y, int64_t j,
                    int64_t ny) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    const double df = x[(int64_t)k * nx + i] - y[(int64_t)k * ny + j];
    const double sq = df * df;
    s = (k == 0) ? sq : s + sq;
  }
  return sqrt(s);
}


/* ---------------------------------------------------------------------------------------------
 * J2 / Y2 (bessel.hpp:25-144): x <= 19 ascending series summed in __float128 (bessel.hpp:
 * 16-18, 43-85), x > 19 Hankel asymptotic P/Q in long double truncated at the smallest term
 * (bessel.hpp:88-125).  Restated with the same operation order.
 * ------------------------------------------------------------------------------------------- */
#include <quadmath.h>
typedef __float128 wide_t;
static wide_t wabs_q(wide_t x) { return x < 0 ? -x : x; }

static wide_t jser_q(int nu, wide_t x) { /* bessel.hpp:45-56 */
  const wide_t h = x / 2, h2 = h * h;
  wide_t term = 1;
  for (int k = 1; k <= nu; ++k) term *= h / k;
  wide_t s = term;
  for (int m = 1; m < 400; ++m) {
    term *= -h2 / ((wide_t)m * (wide_t)(m + nu));
    s += term;
    if (m > 4 && wabs_q(term) < (wide_t)1e-32 * wabs_q(s)) break;
  }
  return s;
}

static void y01_q(wide_t x, wide_t* y0, wide_t* y1) { /* bessel.hpp:59-86 */
  const wide_t pi = M_PIq;
  const wide_t gam = strtoflt128("0.577215664901532860606512090082402431", NULL);
  const wide_t h = x / 2, h2 = h * h;
  const wide_t lg = logq(h) + gam;
  const wide_t j0 = jser_q(0, x), j1 = jser_q(1, x);
  wide_t s = 0, term = 1, hk = 0;
  for (int k = 1; k < 400; ++k) {
    term *= h2 / ((wide_t)k * (wide_t)k);
    hk += (wide_t)1 / k;
    const wide_t c = (k % 2 ? term : -term) * hk;
    s += c;
    if (k > 4 && wabs_q(c) < (wide_t)1e-32 * wabs_q(s)) break;
  }
  *y0 = (2 / pi) * (lg * j0 + s);
  wide_t s1 = 0, t1 = 1, ha = 0, hb = 1;
  for (int k = 0; k < 400; ++k) {
    if (k > 0) {
      t1 *= h2 / ((wide_t)k * (wide_t)(k + 1));
      ha += (wide_t)1 / k;
      hb += (wide_t)1 / (k + 1);
    }
    const wide_t c = (k % 2 ? -t1 : t1) * (ha + hb);
    s1 += c;
    if (k > 4 && wabs_q(c) < (wide_t)1e-32 * wabs_q(s1)) break;
  }
  *y1 = (2 / pi) * lg * j1 - 2 / (pi * x) - h / pi * s1;
}

static void asym_pq(int nu, double x, double* p, double* q) { /* bessel.hpp:89-107 */
  const long double mu = 4.0L * nu * nu, x2 = 64.0L * (long double)x * (long double)x;
  long double ps = 1.0L, qs = (mu - 1) / (8.0L * x);
  long double tp = 1.0L, tq = qs;
  for (int k = 1; k < 40; ++k) {
    const long double a = 4.0L * k - 3, b = 4.0L * k - 1, c = 4.0L * k + 1;
    const long double ntp = tp * -((mu - a * a) * (mu - b * b)) / ((2.0L * k - 1) * (2.0L * k) * x2);
    const long double ntq = tq * -((mu - b * b) * (mu - c * c)) / ((2.0L * k) * (2.0L * k + 1) * x2);
    if (fabsl(ntp) >= fabsl(tp) || fabsl(ntq) >= fabsl(tq)) break;
    ps += ntp;
    qs += ntq;
    tp = ntp;
    tq = ntq;
    if (fabsl(ntp) < 1e-24L && fabsl(ntq) < 1e-24L) break;
  }
  *p = (double)ps;
  *q = (double)qs;
}

static const long double kQPi = 0.785398163397448309615660845819875721L;

static double asym(int nu, double x, int y) { /* bessel.hpp:111-125 */
  double p, q;
  asym_pq(nu, x, &p, &q);
  const long double chi = (long double)x - (2 * nu + 1) * kQPi;
  const long double v = y ? (p * sinl(chi) + q * cosl(chi)) : (p * cosl(chi) - q * sinl(chi));
  return sqrt(2.0 / (M_PI * x)) * (double)v;
}

double hbo_j2(double x) { /* bessel.hpp:129-135 (x >= 0) */
  if (x == 0) return 0.0;
  if (x <= 19.0) return (double)jser_q(2, (wide_t)x);
  return asym(2, x, 0);
}

double hbo_y2(double x) { /* bessel.hpp:137-144 (x > 0) */
  if (x <= 19.0) {
    wide_t y0, y1;
    y01_q((wide_t)x, &y0, &y1);
    return (double)((2 / (wide_t)x) * y1 - y0);
  }
  return (2.0 / x) * asym(1, x, 1) - asym(0, x, 1);
}

/* kernel.hpp:46-61 catalog singularity; used when no diagonal value is supplied. */
static int singular_at_origin(int id) { return id == 0 || id == 1 || id == 2 || id == 5; }

double hbo_eval_radial(int id, int has_diag, double diag, double r, int* status) {
  if (r == 0.0) { /* kernel.hpp:150-155 */
    if (has_diag) return diag;
    if (singular_at_origin(id)) { *status = HBO_ESINGULAR; return 0.0; }
  }
  switch (id) { /* kernel.hpp:93-109 */
    case 0: return 1.0 / r;
    case 1: return log(r);
    case 2: return cos(r) / r;
    case 3: return sin(r) / r;
    case 4: return hbo_j2(r);
    case 5: return hbo_y2(r);
    case 6: return r;
    case 7: return sin(r);
    case 8: return 1.0 / sqrt(1.0 + r);
    case 9: return exp(-r);
    case 10: return exp(-(r * r));
    default: *status = HBO_EUNSUPPORTED; return 0.0; /* Custom: std::function, not on this path */
  }
}

typedef struct {
  int id, has_diag;
  double diag;
  const double *x, *y;
  int64_t T, N, ldk;
  int d;
  double* K;
  int64_t lo, hi; /* row range */
  int status;
} job_t;

static void* run_rows(void* p) {
  job_t* j = (job_t*)p;
  for (int64_t i = j->lo; i < j->hi; ++i)
    for (int64_t c = 0; c < j->N; ++c) {
      const double r = hbo_distance(j->d, j->x, i, j->T, j->y, c, j->N);
      int st = HBO_OK;
      const double v = hbo_eval_radial(j->id, j->has_diag, j->diag, r, &st);
      if (st != HBO_OK && j->status == HBO_OK) j->status = st;
      j->K[c * j->ldk + i] = v;
    }
  return NULL;
}

int hbo_assemble(int id, int has_diag, double diag, const double* x, int64_t T, const double* y,
                 int64_t N, int d, double* K, int64_t ldk, int nthreads, int64_t entry_cap) {
  if (T <= 0 || N <= 0) return HBO_EINVAL;  /* kernel.hpp:171 */
  if (d < 1 || d > 8 || ldk < T) return HBO_EINVAL;
  if (entry_cap > 0 && T > entry_cap / N) return HBO_ECAP; /* kernel.hpp:174-175 */
  if (id < 0 || id > 10) return HBO_EUNSUPPORTED;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > T) nthreads = (int)T;
  job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  const int64_t chunk = (T + nthreads - 1) / nthreads; /* parallel.hpp:20 static chunks */
  for (int w = 0; w < nthreads; ++w) {
    job_t* j = &jobs[w];
    j->id = id; j->has_diag = has_diag; j->diag = diag; j->x = x; j->y = y;
    j->T = T; j->N = N; j->ldk = ldk; j->d = d; j->K = K; j->status = HBO_OK;
    j->lo = w * chunk;
    j->hi = (w + 1) * chunk < T ? (w + 1) * chunk : T;
    if (j->lo > j->hi) j->lo = j->hi;
  }
  for (int w = 1; w < nthreads; ++w) pthread_create(&th[w], NULL, run_rows, &jobs[w]);
  run_rows(&jobs[0]);
  for (int w = 1; w < nthreads; ++w) pthread_join(th[w], NULL);
  int st = HBO_OK;
  for (int w = 0; w < nthreads; ++w)
    if (jobs[w].status != HBO_OK) { st = jobs[w].status; break; }
  free(jobs);
  free(th);
  return st;
}

/* ---------------------------------------------------------------------------------------------
 * ACA restatement (aca.hpp:16-213).  BlockSpec entry(i, j) = eval_radial(||x_{rb+i} -
 * y_{cb+j}||) (aca.hpp:30-33); aca_sweep (aca.hpp:72-162) with its pivot rules (row 0 first,
 * first-maximum argmax over unused columns / rows, zero residual rows skipped), the Frobenius
 * stopping test ||u|| ||v|| <= eps ||A_r||_F with the cross-term update of fro2 (aca.hpp:
 * 120-130), L/U assembly (aca.hpp:150-160); compress (aca.hpp:171-198): re-sweep at eps/10
 * and truncate on a degenerate pivot; apply (aca.hpp:202-213).  Contiguous-vector reductions
 * (norm, dot) use the Eigen SSE2 packet order restated in oracle/eigen_shim/Eigen/Dense.
 * ------------------------------------------------------------------------------------------- */
typedef double (*coeff_fn)(const void* ctx, int64_t i);

static double vec_redux(int64_t n, const double* a, const double* b) {
  /* sum_i a[i]*b[i] (b == NULL: a[i]*a[i]) in Eigen 3.4 LinearVectorizedTraversal order (2-wide) */
#define HBO_C(i) (a[(i)] * (b ? b[(i)] : a[(i)]))
  const int64_t aligned2 = (n / 4) * 4, aligned = (n / 2) * 2;
  if (aligned == 0) {
    double r = HBO_C(0);
    for (int64_t i = 1; i < n; ++i) r = r + HBO_C(i);
    return r;
  }
  double p0 = HBO_C(0), p0b = HBO_C(1);
  if (aligned > 2) {
    double p1 = HBO_C(2), p1b = HBO_C(3);
    for (int64_t i = 4; i < aligned2; i += 4) {
      p0 = p0 + HBO_C(i);
      p0b = p0b + HBO_C(i + 1);
      p1 = p1 + HBO_C(i + 2);
      p1b = p1b + HBO_C(i + 3);
    }
    p0 = p0 + p1;
    p0b = p0b + p1b;
    if (aligned > aligned2) {
      p0 = p0 + HBO_C(aligned2);
      p0b = p0b + HBO_C(aligned2 + 1);
    }
  }
  double r = p0 + p0b;
  for (int64_t i = aligned; i < n; ++i) r = r + HBO_C(i);
  return r;
#undef HBO_C
}

typedef struct {
  int id, has_diag, d;
  double diag;
  const double *x, *y;
  int64_t nt, ns, rb, rows, cb, cols;
  int status;
} hbo_block;

static double blk_entry(hbo_block* b, int64_t i, int64_t j) { /* aca.hpp:30-33 */
  const double r = hbo_distance(b->d, b->x, b->rb + i, b->nt, b->y, b->cb + j, b->ns);
  int st = HBO_OK;
  const double v = hbo_eval_radial(b->id, b->has_diag, b->diag, r, &st);
  if (st != HBO_OK && b->status == HBO_OK) b->status = st;
  return v;
}

typedef struct {
  int64_t rank, cap;
  double *us, *vs; /* rows x cap, cols x cap (column k = u_k / v_k) */
  double* piv;
  int64_t *sigma, *tau; /* block-local indices */
  int met;
} hbo_sweep_t;

static void sweep_free(hbo_sweep_t* s) {
  free(s->us); free(s->vs); free(s->piv); free(s->sigma); free(s->tau);
  memset(s, 0, sizeof(*s));
}

static int sweep_grow(hbo_sweep_t* s, int64_t rows, int64_t cols, int64_t want) {
  if (want <= s->cap) return 0;
  int64_t nc = s->cap ? 2 * s->cap : 16;
  if (nc < want) nc = want;
  double* us = (double*)realloc(s->us, sizeof(double) * (size_t)(rows * nc));
  if (us) s->us = us;
  double* vs = (double*)realloc(s->vs, sizeof(double) * (size_t)(cols * nc));
  if (vs) s->vs = vs;
  double* pv = (double*)realloc(s->piv, sizeof(double) * (size_t)nc);
  if (pv) s->piv = pv;
  int64_t* sg = (int64_t*)realloc(s->sigma, sizeof(int64_t) * (size_t)nc);
  if (sg) s->sigma = sg;
  int64_t* tu = (int64_t*)realloc(s->tau, sizeof(int64_t) * (size_t)nc);
  if (tu) s->tau = tu;
  if (!us || !vs || !pv || !sg || !tu) return -1;
  s->cap = nc;
  return 0;
}

/* aca.hpp:72-148 */
static int aca_sweep(hbo_block* b, double eps, int64_t max_rank, hbo_sweep_t* s) {
  const int64_t m = b->rows, n = b->cols;
  int64_t lim = m < n ? m : n;
  if (max_rank < lim) lim = max_rank;
  char* used_row = (char*)calloc((size_t)m, 1);
  char* used_col = (char*)calloc((size_t)n, 1);
  double* row = (double*)malloc(sizeof(double) * (size_t)n);
  double* u = (double*)malloc(sizeof(double) * (size_t)m);
  double fro2 = 0.0;
  int64_t next_row = 0, rows_left = m;
  int met = 0, rc = 0;
  memset(s, 0, sizeof(*s));
  while (s->rank < lim) {
    const int64_t r = s->rank;
    for (int64_t j = 0; j < n; ++j) row[j] = blk_entry(b, next_row, j);
    for (int64_t k = 0; k < r; ++k) {
      const double c = s->us[k * m + next_row];
      const double* vk = s->vs + k * n;
      for (int64_t j = 0; j < n; ++j) row[j] = row[j] - c * vk[j];
    }
    int64_t piv_col = -1;
    double piv_abs = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      if (used_col[j]) continue;
      const double a = fabs(row[j]);
      if (a > piv_abs) { piv_abs = a; piv_col = j; }
    }
    if (piv_col < 0 || piv_abs == 0.0) { /* aca.hpp:97-107 */
      used_row[next_row] = 1;
      if (--rows_left == 0) { met = 1; break; }
      for (int64_t i = 0; i < m; ++i)
        if (!used_row[i]) { next_row = i; break; }
      continue;
    }
    if (sweep_grow(s, m, n, r + 1)) { rc = -1; break; }
    const double pivot = row[piv_col];
    double* v = s->vs + r * n;
    for (int64_t j = 0; j < n; ++j) v[j] = row[j] / pivot;
    for (int64_t i = 0; i < m; ++i) u[i] = blk_entry(b, i, piv_col);
    for (int64_t k = 0; k < r; ++k) {
      const double c = s->vs[k * n + piv_col];
      const double* uk = s->us + k * m;
      for (int64_t i = 0; i < m; ++i) u[i] = u[i] - c * uk[i];
    }
    s->sigma[r] = next_row;
    s->tau[r] = piv_col;
    s->piv[r] = pivot;
    used_row[next_row] = 1;
    used_col[piv_col] = 1;
    --rows_left;
    const double nu = sqrt(vec_redux(m, u, NULL)), nv = sqrt(vec_redux(n, v, NULL));
    double cross = 0.0;
    for (int64_t k = 0; k < r; ++k)
      cross += vec_redux(m, s->us + k * m, u) * vec_redux(n, s->vs + k * n, v);
    fro2 += 2.0 * cross + nu * nu * nv * nv;
    memcpy(s->us + r * m, u, sizeof(double) * (size_t)m);
    s->rank = r + 1;
    if (nu * nv <= eps * sqrt(fro2 > 0.0 ? fro2 : 0.0)) { met = 1; break; }
    if (rows_left == 0) { met = 1; break; }
    next_row = -1;
    double best = -1.0;
    const double* uu = s->us + r * m;
    for (int64_t i = 0; i < m; ++i) {
      if (used_row[i]) continue;
      const double a = fabs(uu[i]);
      if (a > best) { best = a; next_row = i; }
    }
  }
  s->met = met || s->rank == (m < n ? m : n);
  free(used_row); free(used_col); free(row); free(u);
  return rc;
}

static int degenerate(const hbo_sweep_t* s) { /* aca.hpp:177-181, |diag U| = |pivots| */
  if (s->rank == 0) return 0;
  double mn = fabs(s->piv[0]), mx = mn;
  for (int64_t k = 1; k < s->rank; ++k) {
    const double a = fabs(s->piv[k]);
    if (a < mn) mn = a;
    if (a > mx) mx = a;
  }
  return mn < 1e-14 * mx;
}

/* 0: one sweep, 1: re-swept at eps/10, 2: re-swept and truncated (test introspection) */
int hbo_aca_last_path = 0;

int hbo_aca_compress(int id, int has_diag, double diag, const double* x, int64_t nt,
                     const double* y, int64_t ns, int d, int64_t rb, int64_t rows, int64_t cb,
                     int64_t cols, double eps, int64_t max_rank, int64_t cap, int64_t* sigma,
                     int64_t* tau, double* L, double* U, int32_t* rank, int32_t* met,
                     const double* q, double* bout) {
  if (!(eps > 0)) return HBO_EINVAL;     /* aca.hpp:172 */
  if (max_rank < 1) return HBO_EINVAL;   /* aca.hpp:173 */
  if (rows == 0 || cols == 0) return HBO_EINVAL; /* aca.hpp:174-175 */
  if (id < 0 || id > 10) return HBO_EUNSUPPORTED;
  hbo_block b = {id, has_diag, d, diag, x, y, nt, ns, rb, rows, cb, cols, HBO_OK};
  hbo_sweep_t s;
  hbo_aca_last_path = 0;
  if (aca_sweep(&b, eps, max_rank, &s)) { sweep_free(&s); return HBO_EINVAL; }
  if (b.status == HBO_OK && degenerate(&s)) {
    hbo_aca_last_path = 1;
    sweep_free(&s);
    if (aca_sweep(&b, eps / 10.0, max_rank, &s)) { sweep_free(&s); return HBO_EINVAL; }
  }
  if (b.status != HBO_OK) { sweep_free(&s); return b.status; }
  int64_t r = s.rank;
  const int met_flag = s.met;
  if (degenerate(&s)) { /* aca.hpp:185-196: keep the leading pivots >= 1e-14 max */
    hbo_aca_last_path = 2;
    double mx = 0.0;
    for (int64_t k = 0; k < s.rank; ++k) if (fabs(s.piv[k]) > mx) mx = fabs(s.piv[k]);
    const double cut = 1e-14 * mx;
    r = 0;
    while (r < s.rank && fabs(s.piv[r]) >= cut) ++r;
  }
  if (r > cap) { sweep_free(&s); return HBO_ECAP; }
  const int64_t m = rows, n = cols;
  *rank = (int32_t)r;
  *met = met_flag;
  for (int64_t k = 0; k < r; ++k) { sigma[k] = rb + s.sigma[k]; tau[k] = cb + s.tau[k]; }
  for (int64_t k = 0; k < r; ++k) /* aca.hpp:157-160 */
    for (int64_t a = 0; a < r; ++a) {
      L[a + k * r] = s.us[k * m + s.sigma[a]] / s.piv[k];
      U[k + a * r] = s.piv[k] * s.vs[k * n + s.tau[a]];
    }
  if (q && bout) { /* aca.hpp:202-213 */
    for (int64_t i = 0; i < m; ++i) bout[i] = 0.0;
    if (r > 0) {
      double* t = (double*)malloc(sizeof(double) * (size_t)r);
      double* rowv = (double*)malloc(sizeof(double) * (size_t)n);
      for (int64_t k = 0; k < r; ++k) {
        for (int64_t j = 0; j < n; ++j) rowv[j] = blk_entry(&b, s.sigma[k], j);
        t[k] = vec_redux(n, rowv, q);
      }
      for (int64_t k = 0; k < r; ++k) /* unit lower */
        for (int64_t i = k + 1; i < r; ++i) t[i] = t[i] - L[i + k * r] * t[k];
      for (int64_t k = r - 1; k >= 0; --k) { /* upper */
        t[k] = t[k] / U[k + k * r];
        for (int64_t i = 0; i < k; ++i) t[i] = t[i] - U[i + k * r] * t[k];
      }
      for (int64_t k = 0; k < r; ++k)
        for (int64_t i = 0; i < m; ++i) bout[i] = bout[i] + t[k] * blk_entry(&b, i, s.tau[k]);
      free(t); free(rowv);
    }
  }
  sweep_free(&s);
  return HBO_OK;
}
