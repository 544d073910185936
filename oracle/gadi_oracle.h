/*
 * gadi_oracle.h — CPU restatement of the reference's GADI-IR hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker the CUDA path is compared
 * against (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline leg).
 * The product never links or calls it. Every function cites the reference
 * file:line it restates (paths under /root/reference/proj/core/).
 *
 * Pinning: tests/test_oracle_pin.py checks this restatement bit for bit
 * against the reference itself (oracle/_ref/libgadi_ref.so, built from the
 * reference sources by oracle/Makefile.ref) and against the committed golden
 * vectors in tests/golden/ that the same reference produced.
 *
 * Values are carried in binary64 exactly like the reference's Vector; a value
 * "in precision p" is a binary64 that is representable in p. Build with
 * -ffp-contract=off (core/CMakeLists.txt:28-30): one rounding per op.
 */
#ifndef GADI_ORACLE_H_
#define GADI_ORACLE_H_

#include <stdint.h>

#include "../include/gadi_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t n;          /* square */
  int64_t* rp;        /* n+1 */
  int64_t* ci;        /* nnz */
  double* v;          /* nnz */
} orc_csr;

/* ---- precision.hpp:54-87, precision.cpp:38-59 ---- */
double orc_round(double x, int p);

/* ---- counter RNG shared bit-for-bit with the device generators ---- */
uint64_t orc_splitmix64(uint64_t seed, uint64_t i);
double orc_uniform(uint64_t seed, uint64_t i, double lo, double hi);

/* ---- problem generators ---- */
/* build_convdiff3d (problems.cpp:8-43) with coefficients (t1, t2, t3); returns
 * nnz; rp/ci/v must hold n^3+1 / 7n^3 entries. */
int64_t orc_convdiff_csr(int64_t n, double t1, double t2, double t3, int64_t* rp, int64_t* ci,
                         double* v);
/* C4 family (BASELINE configs[3]): per row `k_off` distinct columns uniform in
 * [i-band, i+band]\{i} clipped to [0,N), values U[-1,1], diagonal
 * 1.1 * sum|off|. rp/ci/v hold N+1 / N*(k_off+1). */
int64_t orc_band_csr(int64_t N, int32_t k_off, int64_t band, uint64_t seed, int64_t* rp, int64_t* ci,
                     double* v);
/* x_i = orc_uniform(seed, i, lo, hi); b = A x (binary64 fold, kernels.cpp:41-54). */
void orc_make_rhs(const orc_csr* A, uint64_t seed, double lo, double hi, double* x, double* b);

/* ---- kernels.cpp ---- */
void orc_matvec(const orc_csr* A, const double* x, int p, double* y);                    /* :41-54 */
void orc_residual(const orc_csr* A, const double* x, const double* b, int uf, int ur, double* s); /* :56-69,135-145 */
double orc_dot(const double* x, const double* y, int64_t n, int p);                        /* :84-90 */
double orc_norm2(const double* x, int64_t n, int p);                                       /* :71-82 */
double orc_norm2_64(const double* x, int64_t n);                                           /* :184-194 */
void orc_axpy(double a, const double* x, const double* y, int64_t n, int p, double* z);    /* :147-164 */
void orc_scale(double a, const double* x, int64_t n, int p, double* z);                    /* :166-171 */

/* ---- splitting.cpp:12-20,37-47 + sparse.cpp:104-117,166-183 ---- */
/* H = alpha I + (A+A^T)/2 and S = alpha I + (A-A^T)/2 on the shared union
 * pattern. Call with rpH == NULL to get nnz. */
int64_t orc_regularize(const orc_csr* A, double alpha, int64_t* rpH, int64_t* ciH, double* vH,
                       double* vS);

/* ---- inner_solver.cpp:47-194 ---- */
int orc_krylov(const orc_csr* M, const double* rhs, int method, double eps, int max_inner, int restart,
               int fmt, double stop_norm, double* x, int* iters, int* status);
/* the same with arithmetic format af over storage format fmt (af == fmt is
 * the reference; af = binary32 over binary16 = the device's GADI_ACCUM_FP32) */
int orc_krylov_af(const orc_csr* M, const double* rhs, int method, double eps, int max_inner, int restart,
                  int fmt, int af, double stop_norm, double* x, int* iters, int* status);

/* ---- band_lu.cpp:60-172 (BandLU) + inner_solver.cpp:27-39 ---- */
typedef struct {
  int64_t n, kl, ku, ldab;
  int fmt;
  double* ab;     /* ldab x n, column j at ab + j*ldab, A(i,j) at row kl+ku+i-j */
  int64_t* ipiv;
} orc_blu;
int orc_blu_factor(const orc_csr* A, int fmt, orc_blu* f);
void orc_blu_solve(const orc_blu* f, const double* rhs, double* x);
void orc_blu_free(orc_blu* f);
int orc_lu_solve(const orc_csr* M, const double* rhs, int fmt, double* x);

/* ---- solver.cpp:57-179 + 250-258 (gadi_ir_solve on a CSR system) ---- */
int64_t orc_shift_diagonal(const orc_csr* M, double alpha, int64_t* rp, int64_t* ci, double* v);
int orc_explicit_check(const orc_csr* A, const orc_csr* M, const orc_csr* N);
int orc_solve_split(const orc_csr* A, const orc_csr* Ms, const orc_csr* Ns, const double* b, const double* x0,
                    const gadi_config* cfg, double* x, double* hist, int cap, gadi_report* rep);
int orc_solve(const orc_csr* A, const double* b, const double* x0, const gadi_config* cfg, double* x,
              double* hist, int cap, gadi_report* rep);

/* ---- gpr.cpp:15-50 (alpha_bisection on the convdiff family) ---- */
int orc_alpha_bisection(int64_t n, int fmt, double lo, double hi, int budget, const gadi_dichotomy* st,
                        double* alpha, int* iters);

/* ---- gpr.cpp:72-169 ---- */
/* mode: fixed hypers (opts->fixed_hypers) or the reference's 27-point grid.
 * params out: sigma_f2, length, sigma_n2, target_mean, lml. */
int orc_gpr(const double* sizes, const double* alphas, int m, const gadi_gpr_opts* opts,
            const double* qsizes, int q, double* mean, double* sd, double* params);

#ifdef __cplusplus
}
#endif
#endif
