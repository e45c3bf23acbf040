/*
 * hb.h -- C ABI of the B200-native rank-reveal path (seeded cube-pair kernel assembly + ε-rank).
 *
 * The reference (/root/reference/proj/include/hodlr/) is a header-only C++20 library whose
 * interface for this path is value types + free functions with C++ exceptions.  This header is
 * the drop-in boundary a binding would target (see INTEGRATION.md for the C++ / ctypes stubs):
 * plain C structs, pointers and sizes, status codes instead of exceptions, no torch or CUDA
 * types in any signature (streams are passed as void*).
 *
 * Reference interface each entry point replaces:
 *   hb_kernel              <- hodlr::KernelSpec / KernelId          kernel.hpp:19-32, 37-110
 *   hb_cube                <- hodlr::HyperCube{lower, side}         geometry.hpp:15-64
 *   hb_pair.d_prime        <- hodlr::InteractionClass (far / surface:d')  geometry.hpp:77-104
 *   hb_classify_pair       <- hodlr::classify_pair(BoxIndex, BoxIndex)  geometry.hpp:106-118
 *   hb_classify_cubes      <- classify_pair on two cubes of one uniform subdivision
 *                             (the inverse of box_cube, geometry.hpp:145-151)
 *   hb_generate_points     <- SPEC pair_geometry (X, Y point sets)
 *   hb_assemble            <- hodlr::assemble_dense                 kernel.hpp:168-181
 *   hb_assemble_dense_host <- hodlr::assemble_dense on host PointSets (same call, host buffers,
 *                             entry cap -> HB_ECAP)                  kernel.hpp:168-181
 *   hb_eval_radial_host    <- hodlr::eval_radial (scalar, host)     kernel.hpp:149-157
 *   hb_rank_matrix         <- SPEC epsilon_rank(matrix, epsilon)
 *   hb_rank                <- SPEC pair_geometry -> assemble_dense -> epsilon_rank
 *   hb_rank_complex        <- the paper's complex F3 / F4 tables from the
 *                             reference's real/imaginary kernel pairs (kernel.hpp:22-27)
 *   hb_sweep               <- SPEC rank_table + parallel_for        SPEC.md:570-578, parallel.hpp:12-29
 *   hb_fit_growth          <- SPEC fit_growth (rank vs {1, log N, N^c}) SPEC.md:580-588
 *   hb_chebyshev_nodes     <- hodlr::chebyshev_nodes                chebyshev.hpp:16-23
 *   hb_hmatrix_build       <- hodlr::HMatrix::initialize (tree, block structure, dense leaf /
 *                             near blocks, ACA factors)   hmatrix.hpp:50-126, cluster_tree.hpp:107-229
 *   hb_hmatrix_matvec      <- hodlr::HMatrix::matvec                hmatrix.hpp:133-179
 *   hb_interpolation_decay <- hodlr::interpolation_decay            chebyshev.hpp:151-177
 *   hb_fit_decay_rate      <- hodlr::fit_decay_rate                 chebyshev.hpp:180-193
 *   hb_v_d_constant        <- hodlr::v_d_constant                   chebyshev.hpp:139-147
 *   hb_block               <- hodlr::BlockSpec index ranges         aca.hpp:16-28
 *   hb_aca_factor          <- hodlr::ACAFactor                      aca.hpp:50-62
 *   hb_aca_compress        <- hodlr::compress (aca_sweep)           aca.hpp:72-198
 *   hb_aca_apply           <- hodlr::apply                          aca.hpp:202-213
 * Error mapping (reference exceptions -> status):
 *   std::invalid_argument -> HB_EINVAL   (kernel.hpp:171-173, geometry.hpp:22)
 *   std::length_error     -> HB_ECAP     (kernel.hpp:174-175, entry cap)
 *   std::domain_error / non-finite entries -> HB_EDOMAIN
 *   std::runtime_error r == 0 on a singular kernel without diagonal -> HB_ESINGULAR (kernel.hpp:152-153)
 *   KernelId::Custom (std::function, cannot cross to the device), J2/Y2 -> HB_EUNSUPPORTED
 * No C++ exception ever crosses this ABI.
 *
 * Rank semantics: rank = count of singular values σ_k > tol·σ₁.
 * The device factorisation is a sketch-pivoted blocked Householder QR stopped once the
 * residual ‖A22‖_F ≤ η·tol·σ₁; the rank is then certified from the singular values of the
 * leading k rows of R:  rank_lo = #σ(R_k) > thr  ≤  true rank  ≤  rank_hi = #σ(R_k) > sqrt(thr² − δ²).
 */
#ifndef HB_H
#define HB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HB_OK = 0,
  HB_EINVAL = 1,
  HB_EDOMAIN = 2,
  HB_ECAP = 3,
  HB_ESINGULAR = 4,
  HB_EUNSUPPORTED = 5,
  HB_ENOMEM = 6,
  HB_ECUDA = 7,
  HB_ENCCL = 8
} hb_status;

/* KernelId order of kernel.hpp:19-32. */
enum {
  HB_K_INVERSE_R = 0, HB_K_LOG_R = 1, HB_K_HELMHOLTZ3D_RE = 2, HB_K_HELMHOLTZ3D_IM = 3,
  HB_K_HANKEL_H12_RE = 4, HB_K_HANKEL_H12_IM = 5, HB_K_R = 6, HB_K_SIN_R = 7,
  HB_K_INV_SQRT_1_PLUS_R = 8, HB_K_EXP_NEG_R = 9, HB_K_EXP_NEG_R2 = 10, HB_K_CUSTOM = 11
};

/* Point modes. */
enum { HB_POINTS_UNIFORM = 0, HB_POINTS_GRID_INTERIOR = 1, HB_POINTS_GRID_CLOSED = 2 };

/* KernelSpec: id + optional diagonal value used when r == 0 (kernel.hpp:37-61). */
typedef struct {
  int32_t id;
  int32_t has_diag;
  double diag;
} hb_kernel;

/* HyperCube: lower corner (d <= 8 coordinates) and side (> 0). */
typedef struct {
  int32_t d;
  int32_t reserved;
  double lower[8];
  double side;
} hb_cube;

/* A target/source cube pair with its point clouds.
 * d_prime: HB_DPRIME_FAR (-1) far-field, HB_DPRIME_SELF (-2) the same box, else the dimension of
 * the shared hyper-surface.  The geometry itself is carried by the cubes; when the two cubes are
 * boxes of one uniform subdivision (equal sides, corner offsets integer multiples of the side)
 * d_prime must equal hb_classify_cubes(target, source), else HB_EINVAL. */
#define HB_DPRIME_FAR (-1)
#define HB_DPRIME_SELF (-2)
typedef struct {
  hb_cube target;
  hb_cube source;
  int32_t d_prime;
  int32_t point_mode;
  int64_t n_target;
  int64_t n_source;
  uint64_t seed;
} hb_pair;

/* One rank result per tolerance. */
typedef struct {
  int32_t rank;        /* = rank_lo: #σ(R_k) > tol·σ₁ */
  int32_t rank_lo;
  int32_t rank_hi;     /* #σ(R_k) > sqrt(thr² − δ²); == rank_lo when certified */
  int32_t k_factored;  /* columns of the pivoted QR kept before certification */
  double sigma1;
  double sigma_r;      /* σ_p   (0 if p == 0) */
  double sigma_r1;     /* σ_{p+1} (0 if p == min(m, n)) */
  double gap;          /* min(σ_p/thr − 1, 1 − σ_{p+1}/thr) */
  double resid;        /* δ used for rank_hi: bound on ‖A22‖₂ after k_factored columns */
  double sec[4];       /* device seconds: points+assembly, factorisation, certification, total */
  int32_t certificate; /* 1: rank_lo == rank_hi with δ = ‖A22‖_F (deterministic bound);
                          2: rank_lo == rank_hi with δ = 2·(power-method estimate of ‖A22‖₂),
                             valid with probability >= 1 - 1e-27; 0: bracket open.
                          The bracket is exact-arithmetic: see fp_band for rounding. */
  int32_t reserved;
  double fp_band;      /* sqrt(N)·u·‖A‖_F / thr: the relative size of the Householder QR's backward
                          error at the threshold.  gap < fp_band flags a count that rounding could
                          move (reported, like a boundary tie) */
} hb_rank_result;

#define HB_MAX_TOLS 4
/* One sweep entry: kernel x pair x up to four tolerances. */
typedef struct {
  hb_kernel kernel;
  hb_pair pair;
  double tols[HB_MAX_TOLS];
  int32_t ntol;
  int32_t reserved;
} hb_problem;

typedef struct hb_context hb_context; /* opaque; one per device and host thread */

const char* hb_version(void);
const char* hb_status_string(hb_status s);
/* Last error detail recorded on this context (or the global one if ctx == NULL). */
const char* hb_last_error(const hb_context* ctx);

hb_status hb_context_create(int device, hb_context** out);
void hb_context_destroy(hb_context* ctx);
/* The CUDA stream (cudaStream_t) all work of this context is ordered on. */
void* hb_context_stream(hb_context* ctx);
/* Tuning: block size cap (8..120, multiple of 8) and stop factor η (0 < η <= 0.1). */
hb_status hb_context_set_tuning(hb_context* ctx, int32_t block_max, double eta);
/* Stopping rule: 0 (default) = deterministic only (stop when ‖A22‖_F <= η·tol·σ̂₁); 1 = also
 * stop when a block power estimate gives 2·σ̂(A22) <= η·tol·σ̂₁ (probabilistic certificate);
 * default 0: the residual checks cost more than the columns they save on the BASELINE sweep. */
hb_status hb_context_set_stopping(hb_context* ctx, int32_t spectral);

/* InteractionClass (geometry.hpp:77-104): kind + surface dimension (valid for SURFACE only). */
enum { HB_IC_SELF = 0, HB_IC_SURFACE = 1, HB_IC_FAR = 2 };
typedef struct {
  int32_t kind;
  int32_t surface_dim; /* d' for HB_IC_SURFACE, else -1 */
} hb_interaction;

/* classify_pair (geometry.hpp:109-118) on two BoxIndex values (level, d per-axis grid coords):
 * all offsets 0 -> SELF; any |offset| >= 2 -> FAR; else SURFACE with d' = #zero offsets.
 * Different levels or d < 1 -> HB_EINVAL (the reference's invalid_argument). */
hb_status hb_classify_pair(int32_t d, int32_t level_a, const int32_t* grid_a, int32_t level_b,
                           const int32_t* grid_b, hb_interaction* out);
/* The same classification for two cubes of one uniform subdivision: equal sides and corner
 * offsets that are integer multiples of the side (else HB_EINVAL: not a same-level box pair). */
hb_status hb_classify_cubes(const hb_cube* a, const hb_cube* b, hb_interaction* out);
/* hb_pair.d_prime value of a classification (HB_DPRIME_SELF / HB_DPRIME_FAR / d'). */
int32_t hb_interaction_dprime(hb_interaction ic);

/* k1: seeded / grid points, SoA (coordinate k of point i at k*n + i), device pointers. */
hb_status hb_generate_points(hb_context* ctx, const hb_pair* pair, double* d_tgt_soa,
                             double* d_src_soa);

/* k2: K(i,j) = F(||x_i - y_j||_2), column-major T x N, leading dimension ldk >= T.
 * Device pointers; ordered on the context stream; synchronises to report ESINGULAR/EDOMAIN. */
hb_status hb_assemble(hb_context* ctx, const hb_kernel* kernel, const double* d_tgt_soa, int64_t T,
                      const double* d_src_soa, int64_t N, int32_t d, double* d_K, int64_t ldk);

/* assemble_dense (kernel.hpp:168-181) on HOST buffers: targets T x d and sources N x d point sets
 * in the reference's PointSet layout (column-major, points are rows = SoA), K column-major T x N
 * with leading dimension ldk >= T.  Copies the points to the device, assembles there (k2) and
 * copies K back.  entry_cap > 0 mirrors the reference's cap (T > entry_cap / N -> HB_ECAP); 0 = no
 * cap.  Empty point sets -> HB_EINVAL; r == 0 on a singular kernel without diagonal -> ESINGULAR. */
hb_status hb_assemble_dense_host(hb_context* ctx, const hb_kernel* kernel, const double* tgt_soa,
                                 int64_t T, const double* src_soa, int64_t N, int32_t d,
                                 double* K, int64_t ldk, int64_t entry_cap);

/* Scalar host evaluation of F(r) with the r == 0 rule (kernel.hpp:149-157). */
hb_status hb_eval_radial_host(const hb_kernel* kernel, double r, double* out);

/* ε-rank of a caller-provided device matrix (column-major m x n, leading dimension ld).
 * The matrix is copied into context workspace; the input is not modified. */
hb_status hb_rank_matrix(hb_context* ctx, const double* d_A, int64_t m, int64_t n, int64_t ld,
                         const double* tols, int32_t ntol, hb_rank_result* out);

/* k1 + k2 + k3: generate, assemble and rank one pair (out has ntol entries). */
hb_status hb_rank(hb_context* ctx, const hb_kernel* kernel, const hb_pair* pair,
                  const double* tols, int32_t ntol, hb_rank_result* out);

/* ε-rank of the complex block K_re + i·K_im — the paper's F3 = e^{ir}/r (HB_K_HELMHOLTZ3D_RE/IM)
 * and F4 = H_2^(1)(r) (HB_K_HANKEL_H12_RE/IM) columns; the reference exposes
 * their real and imaginary parts as separate real kernels (kernel.hpp:22-27).  Computed through
 * the real 2m x 2n embedding [[Re, −Im], [Im, Re]], whose singular values are those of K, each
 * twice: rank = count/2; an odd count (a σ pair straddling the threshold) leaves the bracket open
 * (certificate 0).  k_factored and hb_last_sigma refer to the embedding. */
hb_status hb_rank_complex(hb_context* ctx, const hb_kernel* kernel_re, const hb_kernel* kernel_im,
                          const hb_pair* pair, const double* tols, int32_t ntol,
                          hb_rank_result* out);

/* Singular values (descending) of R_k from the last certification on this context.
 * Copies min(max, count) values to host_out; *count = number available. */
hb_status hb_last_sigma(hb_context* ctx, double* host_out, int64_t max, int64_t* count);

/* k4: run n independent problems over ndev devices (LPT partition on a cost model, one worker
 * thread per device).  out: sum of ntol over problems, problem-major.  Per-problem status codes
 * go to status_out (may be NULL); the return value is the first failure or HB_OK. */
hb_status hb_sweep(const hb_problem* probs, int64_t n, const int32_t* devices, int32_t ndev,
                   hb_rank_result* out, int32_t* status_out);

/* SPEC fit_growth: least-squares fits of rank(N) for one kernel / interaction
 * series by the three growth laws of the paper's theorems — constant (far field), a + b·log N
 * (vertex, Theorem 1), a·N^c (d'-surface, Theorem 2: c = d'/d) — each with its residual sum of
 * squares; `best` is the model with the lowest BIC, n·ln(RSS/n + s²) + params·ln n with
 * s = 1e-3·mean(rank) (so exact fits tie towards the simpler law).  Fewer than 4 distinct N ->
 * HB_EINVAL (the fit is refused), as are non-positive N or negative ranks. */
enum { HB_GROWTH_CONSTANT = 0, HB_GROWTH_LOG = 1, HB_GROWTH_POWER = 2 };
typedef struct {
  int32_t best;          /* HB_GROWTH_* */
  int32_t n;             /* points used */
  double constant;       /* constant model: rank = constant */
  double log_a, log_b;   /* log model: rank = log_a + log_b * ln N */
  double pow_a, pow_c;   /* power model: rank = pow_a * N^pow_c */
  double rss[3];         /* residual sum of squares per model */
  double max_min_ratio;  /* max rank / min rank of the series */
} hb_growth_fit;
hb_status hb_fit_growth(const int64_t* N, const double* rank, int32_t n, hb_growth_fit* out);

/* ---- HODLRdD operator (hmatrix.hpp, cluster_tree.hpp) ------------------------------------------
 * AdmissibilityPolicy (cluster_tree.hpp:17-29): which same-level box pairs are compressed. */
enum { HB_POLICY_WEAKDD = 0, HB_POLICY_STRONG = 1, HB_POLICY_WEAKALL = 2 };
/* BuildReport (hmatrix.hpp:19-26) */
typedef struct {
  double init_seconds;
  int64_t memory_bytes;
  int32_t max_block_rank;
  int32_t depth;
  int64_t num_low_rank_blocks;
  int64_t num_dense_entries;
  int64_t num_tolerance_failures;
} hb_build_report;
typedef struct hb_hmatrix hb_hmatrix; /* opaque; keeps using ctx (caller keeps it alive) */
/* HMatrix::initialize: balanced 2^d tree over `domain` (boxes split until <= n_max points; a point
 * on an internal face goes to the lower box), block structure of `policy`, dense leaf self and
 * near-field blocks assembled on the device in one batched launch, admissible blocks compressed
 * by the device ACA (epsilon, max_rank).  Points: host SoA (d x N).  Errors as the reference:
 * epsilon <= 0, n_max < 1, max_rank < 1, N < 1, d != domain.d -> HB_EINVAL; a point outside the
 * domain -> HB_EDOMAIN; dense entries > dense_entry_cap (0: 4e8 default) -> HB_ECAP. */
hb_status hb_hmatrix_build(hb_context* ctx, const hb_kernel* kernel, const double* pts_soa,
                           int64_t N, int32_t d, const hb_cube* domain, int32_t policy,
                           int64_t n_max, double epsilon, int64_t max_rank,
                           int64_t dense_entry_cap, hb_hmatrix** out, hb_build_report* report);
/* b = H q in the original point ordering, for nvec host vectors (column-major N x nvec). */
hb_status hb_hmatrix_matvec(hb_hmatrix* h, const double* q, double* b, int32_t nvec);
/* Same on device vectors (length N), ordered on the context stream, not synchronised. */
hb_status hb_hmatrix_matvec_device(hb_hmatrix* h, const double* d_q, double* d_b);
/* tree id -> original point id (ClusterTree::original_id), N entries. */
hb_status hb_hmatrix_tree_order(const hb_hmatrix* h, int64_t* orig_of_tree);
void hb_hmatrix_destroy(hb_hmatrix* h);

/* ---- Chebyshev interpolation bound check (chebyshev.hpp:125-193) --------------------------------
 * cos(pi k / p), k = 0..p (p + 1 values; p = 0 -> {0}); p < 0 -> HB_EINVAL. */
hb_status hb_chebyshev_nodes(int32_t p, double* out);
/* interpolation_decay: for each degree p_list[i], err_out[i] = max |K(X, S) - U V| over the
 * reference's sample grid S of the cube (m^d interior points, m = 20 reduced until m^d <= 6.25e6),
 * where U V is the tensor Chebyshev interpolant of the kernel along the cube (degree p on every
 * axis).  Targets: host SoA (d x T).  A target touching the cube (dist <= 0) -> HB_EINVAL.
 * Computed on the device: k2 entries for U and K, Lagrange weights per sample, DMMA GEMM. */
hb_status hb_interpolation_decay(hb_context* ctx, const hb_kernel* kernel, const double* tgt_soa,
                                 int64_t T, const hb_cube* cube, const int32_t* p_list,
                                 int32_t np, double* err_out);
/* fit_decay_rate: rho from the least-squares fit log err = log C - p log rho over the positive
 * errors; fewer than two -> HB_EINVAL. */
hb_status hb_fit_decay_rate(const int32_t* p, const double* err, int32_t n, double* rho_out);
/* v_d_constant: V_d of the tensor interpolation bound; d < 1 -> HB_EINVAL, rho <= 1 -> HB_EDOMAIN. */
hb_status hb_v_d_constant(int32_t d, double rho, double* out);

/* ---- profiling: per-phase device time from CUDA events on the context stream (off by
 * default; the events add ~µs per phase) and the process-wide kernel-launch counter ---------- */
enum {
  HB_PH_ASSEMBLY = 0, HB_PH_SKETCH = 1, HB_PH_PIVOT = 2, HB_PH_PANEL = 3, HB_PH_UPDATE = 4,
  HB_PH_DOWNDATE = 5, HB_PH_SIGMA1 = 6, HB_PH_CERT_QR = 7, HB_PH_BIDIAG = 8, HB_PH_BISECT = 9,
  HB_PH_CHASE = 10, /* bulge-chasing share of HB_PH_BIDIAG (stage 2) */
  HB_NPHASE = 11
};
typedef struct {
  double phase_ms[HB_NPHASE];
  double gemm_ms;         /* device time inside the FP64 DMMA GEMM launches (incl. split-K finish) */
  double gemm_flops;      /* sum of 2*M*N*K over those launches */
  uint64_t gemm_launches;
  uint64_t launches;      /* every kernel launch issued by the library (process-wide counter) */
  uint64_t problems;      /* problems completed with profiling on */
} hb_stats;
const char* hb_phase_name(int32_t phase);
hb_status hb_context_set_profiling(hb_context* ctx, int32_t on);
/* ctx == NULL: process-wide totals (all contexts, including hb_sweep workers). */
hb_status hb_stats_get(const hb_context* ctx, hb_stats* out);
hb_status hb_stats_reset(hb_context* ctx);

/* hb_sweep with options.  Workers reuse one cached context per device across calls (workspace
 * stays allocated); device_seconds[w] = device time of worker w's problem list, measured with
 * CUDA events on its stream (first launch to last completion). */
#define HB_MAX_DEVICES 64
typedef struct {
  int32_t profiling;
  int32_t reserved;
  double device_seconds[HB_MAX_DEVICES];
} hb_sweep_opts;
hb_status hb_sweep_ex(const hb_problem* probs, int64_t n, const int32_t* devices, int32_t ndev,
                      hb_rank_result* out, int32_t* status_out, hb_sweep_opts* opts);
/* Free the per-device contexts cached by hb_sweep / hb_sweep_ex. */
void hb_sweep_release(void);

/* LPT assignment used by hb_sweep / multi-process sweeps: owner[i] in [0, nparts).  The weight of
 * a problem is its predicted device time (GEMM-bound part + half of the latency-bound part, from
 * the predicted factorisation width).  Replaces the reference's parallel_for over
 * independent blocks (parallel.hpp:12-29) as the unit of distribution.  Host-only, deterministic. */
hb_status hb_partition(const hb_problem* probs, int64_t n, int32_t nparts, int32_t* owner);

/* ---- ACA: the reference's own rank(ε) factorisation (aca.hpp:16-213) --------------------------
 * Partially pivoted ACA of the kernel block K(I, J), entries recomputed on the fly on the device;
 * pivot rules, stopping test ||u_r|| ||v_r|| <= ε ||A_r||_F, degenerate-pivot re-sweep at ε/10
 * and truncation exactly as aca.hpp.  Errors: ε <= 0, max_rank < 1 or an empty block ->
 * HB_EINVAL (aca.hpp:172-175); block outside the point sets -> HB_EINVAL; r == 0 on a singular
 * kernel without a diagonal value -> HB_ESINGULAR. */
/* BlockSpec: rows [row_begin, row_begin + rows) of the targets x columns [col_begin, col_begin +
 * cols) of the sources (aca.hpp:26-28). */
typedef struct {
  int64_t row_begin;
  int64_t rows;
  int64_t col_begin;
  int64_t cols;
} hb_block;
typedef struct hb_aca_factor hb_aca_factor; /* opaque ACAFactor; L / U stay on the device */

/* compress every block of `blocks` (one factor each in out[0..nblocks)); blocks that fit one CTA
 * run batched in one launch, larger ones on a cooperative group of CTAs.  Point sets are device
 * SoA arrays (nt targets, ns sources, dimension d). */
hb_status hb_aca_compress(hb_context* ctx, const hb_kernel* kernel, const double* d_tgt_soa,
                          int64_t nt, const double* d_src_soa, int64_t ns, int32_t d,
                          const hb_block* blocks, int64_t nblocks, double eps, int64_t max_rank,
                          hb_aca_factor** out);
/* rank, tolerance_met and ACAFactor::memory_bytes (aca.hpp:58-61); any pointer may be NULL. */
hb_status hb_aca_factor_info(const hb_aca_factor* f, int32_t* rank, int32_t* tolerance_met,
                             int64_t* memory_bytes);
/* Host copies: sigma / tau (rank global ids), L / U (rank x rank column-major); NULL skips. */
hb_status hb_aca_factor_copy(const hb_aca_factor* f, int64_t* sigma, int64_t* tau, double* L,
                             double* U);
/* b = K(I, τ) U⁻¹ L⁻¹ K(σ, J) q with device vectors q (block cols) and b (block rows). */
hb_status hb_aca_apply(hb_context* ctx, const hb_aca_factor* f, const hb_kernel* kernel,
                       const double* d_tgt_soa, int64_t nt, const double* d_src_soa, int64_t ns,
                       int32_t d, const hb_block* block, const double* d_q, double* d_b);
void hb_aca_factor_destroy(hb_aca_factor* f);

/* Deterministic per-problem seed = hash(base, d, d', N). */
uint64_t hb_problem_seed(uint64_t base, int32_t d, int32_t d_prime, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
