/*
 * hb_oracle.c -- CPU ORACLE, TEST INFRASTRUCTURE ONLY (see hb_oracle.h for the citations and
 * the rule on who may call it).  Compiled with -ffp-contract=off so that every multiply and
 * add rounds separately, exactly as the device kernel pins it with __dmul_rn/__dadd_rn.
 */
#include "hb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>

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
    case 6: return r;
    case 7: return sin(r);
    case 8: return 1.0 / sqrt(1.0 + r);
    case 9: return exp(-r);
    case 10: return exp(-(r * r));
    default: *status = HBO_EUNSUPPORTED; return 0.0; /* J2/Y2 and Custom: not on this path */
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
  if (id < 0 || id > 10 || id == 4 || id == 5) return HBO_EUNSUPPORTED;
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
