/*
 * hb_oracle.h -- CPU ORACLE, TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's entry semantics for the rank-reveal hot path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker (or the timed CPU baseline).  The product
 * path (paper_2209_05819_b200/) never links or calls it.
 *
 * Follows:
 *   KernelId order / catalog diagonals      /root/reference/proj/include/hodlr/kernel.hpp:19-67
 *   KernelSpec::operator()(r)               kernel.hpp:93-109
 *   eval_radial (r == 0 handling)           kernel.hpp:149-157
 *   assemble_dense (col-major T x N, cap)   kernel.hpp:168-181
 *   distance = (x - y).norm() of strided    kernel.hpp:179 (rows of a column-major PointSet are
 *     rows -> Eigen DefaultTraversal ->     not unit-stride, so Eigen's redux is a left-to-right
 *     sequential sum of squares)            sum; pinned here with -ffp-contract=off, IEEE sqrt)
 *   HyperCube{lower, side}                  geometry.hpp:15-64
 *   parallel_for static chunking            parallel.hpp:12-29
 *   BlockSpec / aca_sweep / compress / apply aca.hpp:16-213
 * The seeded point generator is this project's own definition (BASELINE.json configs say
 * "uniform fp64 points per cube from seed"); the grid modes follow SURVEY.md A.1.
 */
#ifndef HB_ORACLE_H
#define HB_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: same values as include/hb.h */
enum { HBO_OK = 0, HBO_EINVAL = 1, HBO_EDOMAIN = 2, HBO_ECAP = 3, HBO_ESINGULAR = 4,
       HBO_EUNSUPPORTED = 5 };

/* point modes */
enum { HBO_UNIFORM = 0, HBO_GRID_INTERIOR = 1, HBO_GRID_CLOSED = 2 };

/* Generate n points of cube (lower[0..d), side) into SoA out[k*n + i]. */
int hbo_points(int d, const double* lower, double side, int64_t n, int mode, uint64_t seed,
               int role, double* out_soa);

/* r = ||x_i - y_j||_2 with the pinned summation order. */
double hbo_distance(int d, const double* x_soa, int64_t i, int64_t nx, const double* y_soa,
                    int64_t j, int64_t ny);

/* F(r) incl. the r == 0 rule; *status set on error (ESINGULAR / EUNSUPPORTED). */
double hbo_eval_radial(int kernel_id, int has_diag, double diag, double r, int* status);

/* K(i,j) = F(||x_i - y_j||), column-major, leading dimension ldk >= T; nthreads like
 * parallel_for.  entry_cap <= 0 means no cap. */
int hbo_assemble(int kernel_id, int has_diag, double diag, const double* x_soa, int64_t T,
                 const double* y_soa, int64_t N, int d, double* K, int64_t ldk, int nthreads,
                 int64_t entry_cap);

uint64_t hbo_splitmix64(uint64_t x);

/* bessel::j2 / bessel::y2 (bessel.hpp:129-144), __float128 series / long double asymptotics. */
double hbo_j2(double x);
double hbo_y2(double x);

/* hodlr::compress (aca.hpp:171-198) of the block K(rb:rb+rows, cb:cb+cols) of the kernel over
 * target / source point sets (SoA, nt / ns points), then optionally hodlr::apply (aca.hpp:
 * 202-213) to q (length cols) -> bout (length rows).  Outputs: global pivot ids sigma / tau,
 * L (unit lower) and U (upper) column-major rank x rank, capacity cap pivots. */
int hbo_aca_compress(int id, int has_diag, double diag, const double* x, int64_t nt,
                     const double* y, int64_t ns, int d, int64_t rb, int64_t rows, int64_t cb,
                     int64_t cols, double eps, int64_t max_rank, int64_t cap, int64_t* sigma,
                     int64_t* tau, double* L, double* U, int32_t* rank, int32_t* met,
                     const double* q, double* bout);

#ifdef __cplusplus
}
#endif
#endif
