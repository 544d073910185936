/*
 * gadi_cuda.h — C ABI of the B200-native GADI-IR solver (sm_100a).
 *
 * This is the drop-in boundary for the reference's hot path. Every entry
 * point replaces one piece of the reference's C++ solver API
 * (/root/reference/proj/core/include/gadi/ headers); the citation is on each
 * declaration. Plain pointers and sizes only: no C++ types, no exceptions.
 *
 *   reference                                   here
 *   ------------------------------------------  ------------------------------
 *   gadi_ir_solve(A,b,split,cfg,x0*)            gadi_cuda_create + gadi_cuda_solve
 *     solver.hpp:97-98                            (+ gadi_cuda_history)
 *   class GadiSystem (6 virtuals)               gadi_cuda_residual_uf,
 *     solver.hpp:74-89                            gadi_cuda_true_residual_norm,
 *                                                 gadi_cuda_prepare,
 *                                                 gadi_cuda_set_inner_stop_norm,
 *                                                 gadi_cuda_solve_H, gadi_cuda_solve_S
 *   GadiConfig / InnerSolverSpec                gadi_config / gadi_inner_spec
 *     solver.hpp:17-38, inner_solver.hpp:20-25
 *   SolveReport / SolveStatus                   gadi_report / gadi_status
 *     solver.hpp:44-64
 *   hss_split + regularize                      gadi_cuda_create (HSS, built on the
 *     splitting.hpp:22-47                         device) / gadi_cuda_prepare
 *   explicit_splitting  splitting.hpp:25-26     gadi_cuda_set_split(EXPLICIT, M, N)
 *   build_convdiff3d  problems.hpp:16-42        GADI_PROBLEM_STENCIL7 (matrix free)
 *   fit / predict_alpha  gpr.hpp:72-87          gadi_gpr_fit / gadi_gpr_predict
 *
 * Error convention (reference: solver.hpp:91-92, errors.hpp:9-45): contract and
 * parameter violations return a negative gadi_error (the C++ wrapper rethrows
 * them as ContractViolation / ParameterError); numerical outcomes are never
 * errors, they come back in gadi_report.status exactly as SolveStatus does.
 * Handles are not thread safe: one handle per host thread (the reference's
 * GadiSystem instances are also one-per-solve, solver.cpp:241-245).
 */
#ifndef GADI_CUDA_H_
#define GADI_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GADI_ABI_VERSION 1

/* Precision, precision.hpp:14 (same numeric values). */
typedef enum { GADI_HALF = 0, GADI_SINGLE = 1, GADI_DOUBLE = 2 } gadi_precision;

/* InnerMethod, inner_solver.hpp:15 (same numeric values). LU_DIRECT is the
 * reference's band LU with partial pivoting (band_lu.cpp), factored and
 * applied on the device (gadi_lu.cu) in u_r, bit for bit the reference's; it
 * ignores `accum` (the reference LU rounds every op to u_r) and needs
 * (nb+8)(nb+kl) band values of shared memory per CTA (kl <= ~6000 binary32,
 * ~3000 binary64), else GADI_E_UNSUPPORTED. */
typedef enum { GADI_INNER_LU_DIRECT = 0, GADI_INNER_CG = 1, GADI_INNER_GMRES = 2 } gadi_inner_method;

/* Inner arithmetic (extension). NATIVE = every scalar op rounded once to u_r,
 * dots pairwise in u_r: the reference's semantics (kernels.cpp:33-54,147-177),
 * bitwise reproducible against it. FP32 = u_r storage with binary32
 * arithmetic and binary32 pairwise dot accumulation (the north star's
 * "FP16 storage / FP32 accumulate"); identical to NATIVE when u_r = single. */
typedef enum { GADI_ACCUM_NATIVE = 0, GADI_ACCUM_FP32 = 1 } gadi_accum;

/* SolveStatus, solver.hpp:44-51 (same numeric values). */
typedef enum {
  GADI_CONVERGED = 0,
  GADI_MAX_ITERS = 1,
  GADI_DIVERGED = 2,
  GADI_OVERFLOW_DETECTED = 3,
  GADI_SINGULAR_IN_PRECISION = 4,
  GADI_STALLED = 5
} gadi_status;

/* InnerStatus, inner_solver.hpp:45. */
typedef enum { GADI_INNER_CONVERGED = 0, GADI_INNER_STAGNATED = 1, GADI_INNER_OVERFLOW = 2 } gadi_inner_status;

typedef enum {
  GADI_OK = 0,
  GADI_E_CONTRACT = -1,    /* ContractViolation: shapes, null pointers      */
  GADI_E_PARAM = -2,       /* ParameterError: alpha, omega, precision order */
  GADI_E_UNSUPPORTED = -3, /* a shape / layout this build has no kernel for   */
  GADI_E_FIT = -4,         /* FitError (gpr.hpp:83)                           */
  GADI_E_CUDA = -5,
  GADI_E_NCCL = -6,
  GADI_E_OOM = -7,
  GADI_E_STATE = -8,       /* call order (e.g. solve_H before prepare)        */
  /* gadi_cuda_prepare only: the numerical exceptions GadiSystem::prepare
   * throws for LU_DIRECT (band_lu.cpp:106-108,132-134); gadi_cuda_solve
   * reports them as statuses, as run_gadi_ir does (solver.cpp:74-82). */
  GADI_E_SINGULAR = -9,    /* SingularInPrecision */
  GADI_E_OVERFLOW = -10,   /* OverflowDetected    */
  GADI_E_NO_CONVERGENT_ALPHA = -11, /* NoConvergentAlpha (errors.hpp), alpha_bisection */
  GADI_E_IO = -12          /* IoError (errors.hpp:43-45), MatrixMarket files */
} gadi_error;

/* InnerSolverSpec, inner_solver.hpp:20-25; defaults from gadi_config_default. */
typedef struct {
  int32_t method;          /* gadi_inner_method, default LU_DIRECT */
  double tol_epsilon;      /* default 1e-2 */
  int32_t max_inner_iters; /* default 1000 */
  int32_t restart;         /* default 30 (gmres) */
} gadi_inner_spec;

/* GadiConfig, solver.hpp:17-38, field for field, plus `accum`. */
typedef struct {
  double alpha;            /* 1.0 */
  double omega;            /* 1.0 */
  double xi;               /* 0 -> default_xi(u), solver.cpp:12-18 */
  int32_t u_r, u, u_f;     /* gadi_precision; all DOUBLE by default */
  gadi_inner_spec inner;
  int32_t max_outer_iters; /* 20000 */
  double divergence_factor;/* 1e6 */
  int32_t stall_window;    /* 0 */
  int32_t ones_start;      /* 0 */
  int32_t residual_scaling;/* 1 */
  int32_t accum;           /* gadi_accum, extension: NATIVE */
} gadi_config;

/* SolveReport, solver.hpp:54-64. The history lives in the handle
 * (gadi_cuda_history). RoundingStats collapses to the device overflow count. */
typedef struct {
  int32_t status;             /* gadi_status */
  int32_t outer_iters;
  double final_rres;
  int64_t inner_iter_totals;
  int32_t inner_stagnations;
  int32_t history_len;        /* == outer_iters + 1 */
  int64_t h_iters, s_iters;   /* split of inner_iter_totals (extension) */
  double solve_ms;            /* device time of the solve (CUDA events)   */
  double h_ms, s_ms, outer_ms;/* per-phase device time                    */
  double h2d_bytes, d2h_bytes;/* bytes the facade copied for this call    */
  double e2e_ms;              /* gadi_cuda_solve: host b in -> host x out  */
  int64_t launches;           /* device kernels launched by this call      */
} gadi_report;

typedef enum { GADI_PROBLEM_STENCIL7 = 0, GADI_PROBLEM_CSR = 1, GADI_PROBLEM_BAND = 2 } gadi_problem_kind;

/* Problem description. STENCIL7 is the reference's 3D convection-diffusion
 * operator (problems.cpp:8-43) applied matrix free: grid n^3, row
 * i*n^2 + j*n + k (i slowest), coefficient t2 on the i-1, j-1, k-1
 * neighbours, t1 on the diagonal, t3 on k+1, j+1, i+1; the reference fixes
 * t1 = 6, t2 = -1-r, t3 = -1+r, r = 1/(2n+2) (problems.hpp:16-22); r =
 * beta*h/2 generalises it. CSR takes the reference's SparseMatrix layout
 * (sparse.hpp:17-65): int64 row_ptr/col_idx, binary64 values, column indices
 * strictly increasing per row; host pointers, copied during create. */
typedef struct {
  int32_t kind;            /* gadi_problem_kind */
  int64_t n;               /* STENCIL7: points per direction (N = n^3) */
  double t1, t2, t3;       /* STENCIL7 coefficients */
  int64_t n_rows;          /* CSR */
  int64_t nnz;
  const int64_t* row_ptr;
  const int64_t* col_idx;
  const double* values;
  /* BAND (BASELINE configs[3], generated on the device): n_rows rows, k_off
   * distinct off-diagonal columns per row uniform in [i-band, i+band]\{i}
   * (clipped to [0, n_rows)), values U[-1,1], diagonal 1.1 * sum|off|,
   * splitmix64 stream `seed` (the oracle's orc_band_csr, bit for bit). */
  int64_t band;
  int32_t k_off;
  uint64_t seed;
} gadi_problem_desc;

typedef struct {
  int32_t device;          /* CUDA ordinal */
} gadi_device_opts;

typedef struct gadi_handle gadi_handle;

/* Fills the reference defaults (solver.hpp:17-38, inner_solver.hpp:20-25). */
void gadi_config_default(gadi_config* cfg);
/* default_xi, solver.cpp:12-18. */
double gadi_default_xi(int32_t u);
const char* gadi_status_name(int32_t status);      /* name(SolveStatus), solver.cpp:20-29 */
const char* gadi_last_error(void);                 /* thread-local message of the last error */
int32_t gadi_abi_version(void);

/* Build the device operator: A (binary64, fold order of the reference), the
 * HSS split M = (A+A^T)/2, N = (A-A^T)/2 (splitting.cpp:12-20, pattern union
 * with explicit zeros, sparse.cpp:166-178). Replaces CsrGadiSystem's
 * constructor (solver.cpp:185-186) + hss_split. */
int gadi_cuda_create(const gadi_problem_desc* desc, const gadi_device_opts* opts, gadi_handle** out);
int gadi_cuda_destroy(gadi_handle* h);

/* SplitKind, splitting.hpp:12 (Hss, Explicit; SylvesterAB is gadi_sylv_*). */
typedef enum { GADI_SPLIT_HSS = 0, GADI_SPLIT_EXPLICIT = 1 } gadi_split_kind;
/* A square CSR in the reference's SparseMatrix layout (sparse.hpp:17-65), host pointers. */
typedef struct {
  int64_t n_rows, n_cols, nnz;
  const int64_t* row_ptr;
  const int64_t* col_idx;
  const double* values;
} gadi_csr_desc;
/* The splitting A = M + N the solves use (the `split` argument of
 * gadi_ir_solve, solver.hpp:97-98). A new handle has hss_split(A).
 * EXPLICIT = explicit_splitting(A, M, N) (splitting.cpp:22-35) on a
 * GADI_PROBLEM_CSR handle: GADI_E_CONTRACT on a shape mismatch or when an
 * entry of M + N differs from A's by more than one ulp ("M + N != A"); then
 * prepare forms H = shift_diagonal(M, alpha), S = shift_diagonal(N, alpha)
 * (splitting.cpp:37-47) on the device, each on its own pattern. M and N are
 * copied. HSS (M, N ignored) returns to the HSS split. Drops the prepared
 * inner engine. */
int gadi_cuda_set_split(gadi_handle* h, int32_t kind, const gadi_csr_desc* M, const gadi_csr_desc* N);
int gadi_cuda_dim(const gadi_handle* h, int64_t* n);

/* ---- GadiSystem mirror (solver.hpp:74-89); host vectors of length dim, ----
 * ---- values carried in binary64 exactly like the reference's Vector.   ---- */

/* residual_uf: b - A x entirely in u_f (kernels.cpp:56-69). b is the vector
 * most recently given to gadi_cuda_set_rhs. */
int gadi_cuda_set_rhs(gadi_handle* h, const double* b);
int gadi_cuda_residual_uf(gadi_handle* h, int32_t u_f, const double* x, double* s_out);
/* true_residual_norm: binary64 ||b - A x||_2 (solver.cpp:194-197). */
int gadi_cuda_true_residual_norm(gadi_handle* h, const double* x, double* norm_out);
/* prepare: H = alpha I + M, S = alpha I + N rounded to u_r (splitting.cpp:37-47,
 * inner_solver.cpp:41-45); LU_DIRECT also factors H then S (solver.cpp:204-207)
 * and returns GADI_E_SINGULAR / GADI_E_OVERFLOW where the reference throws. */
int gadi_cuda_prepare(gadi_handle* h, double alpha, double omega, int32_t u_r,
                      const gadi_inner_spec* spec, int32_t accum);
/* Drop the prepared inner engine (operators, work vectors, LU factors): the
 * next solve re-runs prepare, exactly as a fresh gadi_ir_solve /
 * CsrGadiSystem does (solver.cpp:75). A handle otherwise keeps the prepared
 * state across solves with the same (alpha, omega, u_r, inner spec). */
int gadi_cuda_reset(gadi_handle* h);
int gadi_cuda_set_inner_stop_norm(gadi_handle* h, double stop_norm);
/* solve_H: CG on H (inner_solver.cpp:47-83); solve_S: GMRES(restart) on S
 * (inner_solver.cpp:85-194; a CG request degrades to GMRES, solver.cpp:217-221).
 * rhs must be u_r-representable (it is rounded on upload, as round_vec does). */
int gadi_cuda_solve_H(gadi_handle* h, const double* rhs, double* x_out, int32_t* iters,
                      int32_t* inner_status);
int gadi_cuda_solve_S(gadi_handle* h, const double* rhs, double* x_out, int32_t* iters,
                      int32_t* inner_status);

/* ---- facade gadi_ir_solve (solver.hpp:97-98; run_gadi_ir solver.cpp:57-179) ---- */

/* Host buffers: b and x0 (nullable: zeros, or ones if cfg->ones_start) are
 * uploaded, the whole IR loop runs device resident, x is downloaded. */
int gadi_cuda_solve(gadi_handle* h, const gadi_config* cfg, const double* b, const double* x0,
                    double* x_out, gadi_report* rep);
/* Same loop on device-resident binary64 vectors (no host copies). */
int gadi_cuda_solve_device(gadi_handle* h, const gadi_config* cfg, const double* d_b,
                           const double* d_x0, double* d_x, gadi_report* rep);
/* rel_residual_history of the last solve (history[0] = 1); returns the number
 * of entries written (min(len, cap)). */
int gadi_cuda_history(const gadi_handle* h, double* out, int32_t cap);

/* Device kernels this handle has launched so far (bench / driver evidence). */
int64_t gadi_cuda_launch_count(const gadi_handle* h);
/* Stored entries of A and of the H/S union pattern (0 for matrix-free stencils). */
int gadi_cuda_nnz(const gadi_handle* h, int64_t* nnz_a, int64_t* nnz_hs);

/* ---- operator-level kernels (parity tests; each is one device pass) ---- */

/* which: 0 = A (binary64 fold, kernels.cpp:41-54), 1 = H, 2 = S (after
 * prepare; fold in the inner arithmetic). y = Op x, host buffers. */
int gadi_cuda_apply(gadi_handle* h, int32_t which, const double* x, double* y);
/* Pairwise dot in precision p (kernels.cpp:33-39,84-90,173-177) and the
 * max-scaled norm2 in p (kernels.cpp:71-82); device kernels, host buffers. */
int gadi_cuda_dot(int32_t device, int32_t p, const double* x, const double* y, int64_t n,
                  double* out);
int gadi_cuda_norm2(int32_t device, int32_t p, const double* x, int64_t n, double* out);

/* ---- synthetic problem data on the device (bench / large parity runs) ---- */

/* x_true_i = lo + (hi-lo) * u(seed, i), u = splitmix64 counter RNG -> 53-bit
 * uniform in [0,1); b = A x_true with the reference's binary64 fold. Writes
 * device buffers of length dim. */
int gadi_cuda_make_rhs(gadi_handle* h, uint64_t seed, double lo, double hi, double* d_xtrue,
                       double* d_b);

/* ---- sharded solves: z-slabs over several devices (the
 * reference has no distributed path -- this extends gadi_ir_solve,
 * solver.hpp:97-98, to a slab-partitioned stencil) ----
 * Rank r of `world` (a power of two dividing n) owns planes
 * [r n/world, (r+1) n/world) of the n^3 grid: rows [r N/world, (r+1) N/world).
 * Every dot / norm is a collective whose result is the single-device value
 * bit for bit (each slab is an aligned subtree of the pairwise sum; the slab
 * partials are folded in rank order), and every rank takes the same
 * control-flow decisions. A shard's vectors (b, x0, x, make_rhs) are its
 * N/world rows; gadi_cuda_dim returns that count. A group must outlive its
 * handles. */
typedef struct gadi_group gadi_group;
/* ranks = threads of this process (one or several devices): gadi_cuda_solve_group */
int gadi_group_local(int32_t world, gadi_group** out);
/* one rank per process over NCCL: every process passes the same 128-byte id
 * (from gadi_nccl_unique_id on one rank, broadcast by the caller) and then
 * calls gadi_cuda_solve / gadi_cuda_solve_device on its shard collectively */
int gadi_nccl_unique_id(uint8_t* out128);
int gadi_group_nccl(int32_t world, int32_t rank, const uint8_t* id128, gadi_group** out);
/* one rank per process on ONE node over CUDA IPC (peer-mapped staging
 * buffers, interprocess events, a barrier in POSIX shared memory `name`,
 * "/..."; every rank passes the same name): the intra-node transport of
 * bench.py --gpus N. Collective: returns when all `world` ranks have attached. */
int gadi_group_ipc(int32_t world, int32_t rank, const char* name, gadi_group** out);
int gadi_group_destroy(gadi_group* g);
/* the shard of `rank` (GADI_PROBLEM_STENCIL7 only) */
int gadi_cuda_create_shard(const gadi_problem_desc* d, const gadi_device_opts* opts, gadi_group* g,
                           int32_t rank, gadi_handle** out);
/* first global row and row count of a handle's shard (0, dim when unsharded) */
int gadi_cuda_shard_range(const gadi_handle* h, int64_t* first_row, int64_t* n_rows);
/* a local group's sharded solve: one host thread per rank, hs[r] = rank r;
 * device buffers per rank (d_x0 may be NULL); one report per rank (identical
 * status, iteration counts and history on every rank) */
int gadi_cuda_solve_group(gadi_handle* const* hs, int32_t world, const gadi_config* cfg,
                          const double* const* d_b, const double* const* d_x0, double* const* d_x,
                          gadi_report* reps);

/* ---- GPR alpha predictor (gpr.hpp:60-87; fit gpr.cpp:109-149,
 * predict_alpha gpr.cpp:151-169) ---- */
typedef struct {
  int32_t fixed_hypers;   /* 1: use sigma_f2/length/sigma_n2 as given (C5); 0: the
                             reference's 27-point grid search */
  double sigma_f2, length, sigma_n2;
  int32_t has_sigma_n2;   /* grid mode: FitOptions::sigma_n2 (gpr.hpp:72-75) */
  int32_t device;
} gadi_gpr_opts;
typedef struct gadi_gpr gadi_gpr;
/* sizes: system dimensions N_i (inputs are ln N_i, gpr.cpp:114); targets alpha_i. */
int gadi_gpr_fit(const double* sizes, const double* alphas, int32_t m, const gadi_gpr_opts* opts,
                 gadi_gpr** out);
int gadi_gpr_predict(gadi_gpr* g, const double* sizes, int32_t q, double* mean, double* stddev);
int gadi_gpr_params(const gadi_gpr* g, double* sigma_f2, double* length, double* sigma_n2,
                    double* lml, double* target_mean);
/* Device times of the last fit / inverse-factor formation / variance pass
 * (CUDA events, ms), the variance path the last predict took (1 = tcgen05
 * tensor cores with fp16 hi/lo operands, 2 = binary64) and the kernels
 * launched so far (bench / driver evidence). Any pointer may be NULL. */
int gadi_gpr_timings(const gadi_gpr* g, double* fit_ms, double* inverse_ms, double* variance_ms,
                     int32_t* variance_path, int64_t* launches);
int gadi_gpr_destroy(gadi_gpr* g);

/* ---- GPR training-set generation (gpr.hpp:37-58; gpr.cpp:15-68) over the
 * reference's convdiff family: size parameter n -> build_convdiff3d({n})
 * (r = 1/(2n+2), b = A * ones, problems.cpp:8-43), HSS split. Each probe is a
 * full device solve with u_r = u = u_f = fmt; the probes run concurrently
 * (a pool of host threads, one handle and stream each; GADI_TRAIN_WORKERS,
 * default 16) and are chosen in the reference's probe order, so the result is
 * the reference's. ---- */
typedef struct {            /* DichotomySettings, gpr.hpp:37-44 */
  double alpha_lo;          /* 1e-2 */
  double alpha_hi;          /* 1e2 */
  int32_t budget;           /* 21 log-grid probes */
  double train_xi;          /* 1e-8 */
  int32_t max_outer;        /* 1500 */
  gadi_inner_spec inner;    /* InnerSolverSpec{}: lu_direct, 1e-2, 1000, 30 */
} gadi_dichotomy;
void gadi_dichotomy_default(gadi_dichotomy* st);
/* alpha_bisection (gpr.cpp:15-50): the grid alpha with the fewest outer
 * iterations among converged probes (ties: the smaller alpha). Errors:
 * GADI_E_PARAM (bracket, budget < 3), GADI_E_NO_CONVERGENT_ALPHA. */
int gadi_alpha_bisection(int64_t size_param, int32_t fmt, double alpha_lo, double alpha_hi, int32_t budget,
                         const gadi_dichotomy* st, int32_t device, double* alpha, int32_t* iters);
/* generate_training_set (gpr.cpp:52-68): one pair per size parameter, sorted
 * by system dimension size_n = n^3; GADI_E_PARAM on duplicate sizes. Feed
 * size_n / alpha to gadi_gpr_fit. */
int gadi_generate_training_set(const int64_t* size_params, int32_t count, int32_t fmt, const gadi_dichotomy* st,
                               int32_t device, int64_t* size_n, double* alpha, int32_t* iters);

/* ---- MatrixMarket ingest (sparse.hpp:75-76; matrix_market.cpp:22-86) ----
 * gadi_mm_read = read_matrix_market_file: coordinate real/integer,
 * general/symmetric/skew-symmetric, 1-based, duplicates summed; the banner is
 * parsed on the host, the from_triplets assembly (sort, duplicate sums,
 * row_ptr) runs on `device`. The CSR stays owned by the library until
 * gadi_csr_destroy; pass its arrays to gadi_cuda_create (GADI_PROBLEM_CSR).
 * Errors: GADI_E_IO (IoError), GADI_E_CONTRACT (triplet out of range). */
typedef struct gadi_csr gadi_csr;
int gadi_mm_read(const char* path, int32_t device, gadi_csr** out);
int gadi_csr_view(const gadi_csr* m, int64_t* n_rows, int64_t* n_cols, int64_t* nnz, const int64_t** row_ptr,
                  const int64_t** col_idx, const double** values);
int gadi_csr_destroy(gadi_csr* m);
/* write_matrix_market_file: "symmetric" (lower triangle) when A == A^T exactly */
int gadi_mm_write(const char* path, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_idx,
                  const double* values);

/* ---- Sylvester GADI-AB (problems.hpp:44-89; sylvester.cpp): the
 * reference's second GadiSystem, A X + X B = G (X m x n, column-major vec),
 * solved by run_gadi_ir with splitting M = I (x) A, N = B^T (x) I: prepare
 * factors alpha I + A and alpha I + B^T (BandLU in u_r, the inner spec is
 * ignored as in the reference), solve_H runs the column solves, solve_S the
 * row solves, one device thread per column / row. ---- */
typedef struct gadi_sylv gadi_sylv;
/* A (m x m) and B (n x n) in the reference's CSR layout, G (m x n) column-major;
 * host pointers, copied. gadi_ab_solve passes G = -C (sylvester.cpp:125-127). */
int gadi_sylv_create(int64_t m, const int64_t* a_rp, const int64_t* a_ci, const double* a_v, int64_t n,
                     const int64_t* b_rp, const int64_t* b_ci, const double* b_v, const double* G, int32_t device,
                     gadi_sylv** out);
/* run_gadi_ir(SylvesterOperator, cfg, x0); x0 NULL: zeros (ones if ones_start). */
int gadi_sylv_solve(gadi_sylv* s, const gadi_config* cfg, const double* x0, double* x_out, gadi_report* rep);
int gadi_sylv_history(const gadi_sylv* s, double* out, int32_t cap);
int gadi_sylv_destroy(gadi_sylv* s);

#ifdef __cplusplus
}
#endif
#endif /* GADI_CUDA_H_ */
