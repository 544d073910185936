/*
 * gadi_oracle.c — CPU restatement of the reference GADI-IR hot path.
 * TEST INFRASTRUCTURE ONLY (see gadi_oracle.h). Built with
 *   gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared -lm
 * Reference paths are relative to /root/reference/proj/core/.
 */
#include "gadi_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define D 2 /* GADI_DOUBLE */

/* ------------------------------------------------------------------ rounding
 * round_to (precision.hpp:54-87, precision.cpp:38-59): one RNE rounding of a
 * binary64 to binary16 (subnormals kept, |x| >= 65520 -> inf) or binary32.
 * Restated with ilogb/nearbyint instead of the reference's bit trick; pinned
 * bit-exact over all 65,536 encodings + random doubles in test_oracle_pin.py. */
static double round_half(double x) {
  if (isnan(x) || isinf(x) || x == 0.0) return x;
  {
    /* normal binary16 range: round the 52-bit fraction to 10 bits in the
     * integer domain (ties to even); a carry into the exponent is the
     * correctly rounded next binade */
    uint64_t u;
    memcpy(&u, &x, 8);
    const uint64_t sgn = u & 0x8000000000000000ull, mag = u & 0x7fffffffffffffffull;
    const double ax = fabs(x);
    if (ax >= 0x1p-14 && ax < 65520.0) {
      const uint64_t keep = (mag >> 42) & 1u;
      uint64_t m2 = (mag + (((uint64_t)1 << 41) - 1u) + keep) & ~(((uint64_t)1 << 42) - 1u);
      m2 |= sgn;
      double r;
      memcpy(&r, &m2, 8);
      return r;
    }
  }
  double ax = fabs(x);
  if (ax >= 65520.0) return copysign(INFINITY, x);
  int e = ilogb(ax);
  int q = e < -14 ? -24 : e - 10; /* exponent of the binary16 quantum */
  double r = ldexp(nearbyint(ldexp(ax, -q)), q);
  return copysign(r, x);
}

double orc_round(double x, int p) {
  if (p == GADI_HALF) return round_half(x);
  if (p == GADI_SINGLE) return (double)(float)x;
  return x;
}
#define R(x, p) orc_round((x), (p))

static double unit_roundoff(int p) {
  return p == GADI_HALF ? ldexp(1.0, -11) : p == GADI_SINGLE ? ldexp(1.0, -24) : ldexp(1.0, -53);
}

/* ----------------------------------------------------------------------- RNG */
uint64_t orc_splitmix64(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double orc_uniform(uint64_t seed, uint64_t i, double lo, double hi) {
  double u = (double)(orc_splitmix64(seed, i) >> 11) * 0x1p-53;
  return lo + (hi - lo) * u;
}

/* ---------------------------------------------------------------- generators */
/* build_convdiff3d, problems.cpp:8-43: push order i-1, j-1, k-1, diag, k+1,
 * j+1, i+1 (= ascending column). */
int64_t orc_convdiff_csr(int64_t n, double t1, double t2, double t3, int64_t* rp, int64_t* ci,
                         double* v) {
  const int64_t nn = n * n;
  int64_t c = 0;
  rp[0] = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j)
      for (int64_t k = 0; k < n; ++k) {
        const int64_t row = i * nn + j * n + k;
#define PUSH(col, val) (ci[c] = (col), v[c] = (val), ++c)
        if (i > 0) PUSH(row - nn, t2);
        if (j > 0) PUSH(row - n, t2);
        if (k > 0) PUSH(row - 1, t2);
        PUSH(row, t1);
        if (k + 1 < n) PUSH(row + 1, t3);
        if (j + 1 < n) PUSH(row + n, t3);
        if (i + 1 < n) PUSH(row + nn, t3);
#undef PUSH
        rp[row + 1] = c;
      }
  return c;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : x > y;
}

/* The C4 generator (BASELINE configs[3]). Draw j of row i uses
 * counter (i << 20) | j of stream `seed`; values use stream seed ^ VALSALT at
 * counter (i << 8) | slot. Mirrored exactly by the device generator. */
#define VALSALT 0x5851F42D4C957F2Dull
int64_t orc_band_csr(int64_t N, int32_t k_off, int64_t band, uint64_t seed, int64_t* rp, int64_t* ci,
                     double* v) {
  int64_t cols[256];
  int64_t c = 0;
  rp[0] = 0;
  for (int64_t i = 0; i < N; ++i) {
    int cnt = 0;
    for (uint64_t draw = 0; cnt < k_off && draw < (1u << 20); ++draw) {
      uint64_t z = orc_splitmix64(seed, ((uint64_t)i << 20) | draw);
      int64_t off = (int64_t)(z % (uint64_t)(2 * band + 1)) - band;
      int64_t col = i + off;
      if (off == 0 || col < 0 || col >= N) continue;
      int dup = 0;
      for (int t = 0; t < cnt; ++t) dup |= cols[t] == col;
      if (dup) continue;
      cols[cnt++] = col;
    }
    qsort(cols, (size_t)cnt, sizeof(int64_t), cmp_i64);
    double sum = 0.0;
    int64_t diag_pos = -1;
    int slot = 0;
    for (int t = 0; t <= cnt; ++t) {
      if (diag_pos < 0 && (t == cnt || cols[t] > i)) {
        diag_pos = c;
        ci[c] = i;
        v[c] = 0.0;
        ++c;
      }
      if (t == cnt) break;
      double val = orc_uniform(seed ^ VALSALT, ((uint64_t)i << 8) | (uint64_t)slot, -1.0, 1.0);
      ++slot;
      sum += fabs(val);
      ci[c] = cols[t];
      v[c] = val;
      ++c;
    }
    v[diag_pos] = 1.1 * sum;
    rp[i + 1] = c;
  }
  return c;
}

/* ------------------------------------------------------------------- kernels */
/* matvec_impl, kernels.cpp:41-54: per-row fold in stored order. */
void orc_matvec(const orc_csr* A, const double* x, int p, double* y) {
  for (int64_t i = 0; i < A->n; ++i) {
    double acc = 0.0;
    for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) acc = R(acc + R(A->v[k] * x[A->ci[k]], p), p);
    y[i] = acc;
  }
}

/* residual_stage1 + round_vec, kernels.cpp:56-69,135-145. */
void orc_residual(const orc_csr* A, const double* x, const double* b, int uf, int ur, double* s) {
  for (int64_t i = 0; i < A->n; ++i) {
    double acc = b[i];
    for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) acc = R(acc - R(A->v[k] * x[A->ci[k]], uf), uf);
    s[i] = R(acc, ur);
  }
}

/* pairwise_sum, kernels.cpp:33-39: halve with h = n/2, every add rounded. */
static double pairwise(const double* t, int64_t n, int p) {
  if (n == 1) return t[0];
  if (n == 2) return R(t[0] + t[1], p);
  const int64_t h = n / 2;
  return R(pairwise(t, h, p) + pairwise(t + h, n - h, p), p);
}

/* dot_impl, kernels.cpp:84-90. */
double orc_dot(const double* x, const double* y, int64_t n, int p) {
  if (n == 0) return 0.0;
  double* t = (double*)malloc((size_t)n * sizeof(double));
  for (int64_t i = 0; i < n; ++i) t[i] = R(x[i] * y[i], p);
  double s = pairwise(t, n, p);
  free(t);
  return s;
}

static double inf_norm(const double* x, int64_t n) {
  double m = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double a = fabs(x[i]);
    if (m < a) m = a; /* std::max(m, a): NaN never wins */
  }
  return m;
}

static int all_finite(const double* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return 0;
  return 1;
}

/* norm2_impl, kernels.cpp:71-82. */
double orc_norm2(const double* x, int64_t n, int p) {
  double m = inf_norm(x, n);
  if (m == 0.0 || !isfinite(m)) return m;
  double* sq = (double*)malloc((size_t)n * sizeof(double));
  for (int64_t i = 0; i < n; ++i) {
    double q = R(x[i] / m, p);
    sq[i] = R(q * q, p);
  }
  double s = pairwise(sq, n, p);
  free(sq);
  return R(m * R(sqrt(s), p), p);
}

/* norm2_64, kernels.cpp:184-194. */
double orc_norm2_64(const double* x, int64_t n) {
  double m = inf_norm(x, n);
  if (m == 0.0 || !isfinite(m)) return m;
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double q = x[i] / m;
    s += q * q;
  }
  return m * sqrt(s);
}

/* axpy, kernels.cpp:147-164: y + a*x, mul then add each rounded. */
void orc_axpy(double a, const double* x, const double* y, int64_t n, int p, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = R(y[i] + R(a * x[i], p), p);
}

/* scale, kernels.cpp:166-171. */
void orc_scale(double a, const double* x, int64_t n, int p, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = R(a * x[i], p);
}

/* ----------------------------------------------------------------- splitting
 * hss_split (splitting.cpp:12-20) = add(0.5,A,0.5,A^T) and add(0.5,A,-0.5,A^T)
 * with from_triplets' duplicate summation (sparse.cpp:36-58,166-178: pattern
 * union, explicit zeros kept); regularize (splitting.cpp:37-47) =
 * shift_diagonal (sparse.cpp:180-183) = add(1.0, M, alpha, I). Sums of two
 * values are order independent (IEEE addition commutes). */
int64_t orc_regularize(const orc_csr* A, double alpha, int64_t* rpH, int64_t* ciH, double* vH,
                       double* vS) {
  const int64_t n = A->n, nnz = A->rp[n];
  /* transpose (sparse.cpp:104-117): counting sort, rows in ascending order */
  int64_t* trp = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t* tci = (int64_t*)malloc((size_t)(nnz ? nnz : 1) * sizeof(int64_t));
  double* tv = (double*)malloc((size_t)(nnz ? nnz : 1) * sizeof(double));
  int64_t* next = (int64_t*)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  for (int64_t k = 0; k < nnz; ++k) ++trp[A->ci[k] + 1];
  for (int64_t j = 0; j < n; ++j) trp[j + 1] += trp[j];
  for (int64_t j = 0; j < n; ++j) next[j] = trp[j];
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
      int64_t q = next[A->ci[k]]++;
      tci[q] = i;
      tv[q] = A->v[k];
    }
  int64_t c = 0;
  if (rpH) rpH[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t a = A->rp[i], ae = A->rp[i + 1], t = trp[i], te = trp[i + 1];
    int diag_done = 0;
    while (a < ae || t < te || !diag_done) {
      int64_t ca = a < ae ? A->ci[a] : INT64_MAX, ct = t < te ? tci[t] : INT64_MAX;
      int64_t col = ca < ct ? ca : ct;
      if (!diag_done && i <= col) col = i;
      int hasA = ca == col, hasT = ct == col;
      double m, nv;
      int in_pattern = hasA || hasT;
      if (hasA && hasT) {
        m = 0.5 * A->v[a] + 0.5 * tv[t];
        nv = 0.5 * A->v[a] + -0.5 * tv[t];
      } else if (hasA) {
        m = 0.5 * A->v[a];
        nv = 0.5 * A->v[a];
      } else if (hasT) {
        m = 0.5 * tv[t];
        nv = -0.5 * tv[t];
      } else {
        m = nv = 0.0;
      }
      double h = m, s = nv;
      if (col == i) {
        /* shift_diagonal: 1.0*M_ii + alpha*1 (alpha alone when M has no ii) */
        h = in_pattern ? 1.0 * m + alpha : alpha;
        s = in_pattern ? 1.0 * nv + alpha : alpha;
        diag_done = 1;
      }
      if (rpH) {
        ciH[c] = col;
        vH[c] = h;
        vS[c] = s;
      }
      ++c;
      if (hasA) ++a;
      if (hasT) ++t;
    }
    if (rpH) rpH[i + 1] = c;
  }
  free(trp);
  free(tci);
  free(tv);
  free(next);
  return c;
}

/* shift_diagonal (sparse.cpp:180-183) of a general CSR M: add(1.0, M, alpha, I),
 * the pattern of M with the diagonal inserted where M has none (value alpha
 * there, 1.0*M_ii + alpha elsewhere). rp == NULL: count only. */
int64_t orc_shift_diagonal(const orc_csr* M, double alpha, int64_t* rp, int64_t* ci, double* v) {
  int64_t c = 0;
  if (rp) rp[0] = 0;
  for (int64_t i = 0; i < M->n; ++i) {
    int done = 0;
    for (int64_t k = M->rp[i]; k < M->rp[i + 1] || !done;) {
      const int64_t col = k < M->rp[i + 1] ? M->ci[k] : INT64_MAX;
      if (!done && i <= col) {
        if (rp) {
          ci[c] = i;
          v[c] = col == i ? 1.0 * M->v[k] + alpha : alpha;
        }
        if (col == i) ++k;
        done = 1;
      } else {
        if (rp) {
          ci[c] = col;
          v[c] = 1.0 * M->v[k];
        }
        ++k;
      }
      ++c;
    }
    if (rp) rp[i + 1] = c;
  }
  return c;
}

/* explicit_splitting's check (splitting.cpp:22-35): every entry of
 * add(1.0, M, 1.0, N) equals A's entry there (0 where A has none) within one
 * ulp of |a|. Returns 0 or GADI_E_CONTRACT. */
int orc_explicit_check(const orc_csr* A, const orc_csr* M, const orc_csr* N) {
  if (M->n != A->n || N->n != A->n) return GADI_E_CONTRACT;
  for (int64_t i = 0; i < A->n; ++i) {
    int64_t m = M->rp[i], me = M->rp[i + 1], q = N->rp[i], qe = N->rp[i + 1], a = A->rp[i], ae = A->rp[i + 1];
    while (m < me || q < qe) {
      const int64_t cm = m < me ? M->ci[m] : INT64_MAX, cn = q < qe ? N->ci[q] : INT64_MAX;
      const int64_t col = cm < cn ? cm : cn;
      double sum = 0.0;
      if (cm == col && cn == col) sum = 1.0 * M->v[m] + 1.0 * N->v[q];
      else if (cm == col) sum = 1.0 * M->v[m];
      else sum = 1.0 * N->v[q];
      if (cm == col) ++m;
      if (cn == col) ++q;
      while (a < ae && A->ci[a] < col) ++a;
      const double av = (a < ae && A->ci[a] == col) ? A->v[a] : 0.0;
      if (fabs(sum - av) > fabs(av) * 2.220446049250313e-16) return GADI_E_CONTRACT;
    }
  }
  return GADI_OK;
}

/* -------------------------------------------------------------------- krylov
 * The Krylov solvers take a storage format `fmt` (u_r: every vector entry
 * and matrix value is a u_r number) and an arithmetic format `af`. af == fmt
 * is the reference (inner_solver.cpp: every op rounded to u_r). af = binary32
 * with fmt = binary16 restates the device's GADI_ACCUM_FP32 mode (binary16
 * storage, binary32 arithmetic and accumulation; not in the reference): each
 * op is rounded to af, each stored vector entry once more to fmt. */
static void matvec_s(const orc_csr* A, const double* x, int af, int fmt, double* y) {
  orc_matvec(A, x, af, y);
  if (fmt != af)
    for (int64_t i = 0; i < A->n; ++i) y[i] = R(y[i], fmt);
}
static void axpy_s(double a, const double* x, const double* y, int64_t n, int af, int fmt, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = R(R(y[i] + R(a * x[i], af), af), fmt);
}

static void rounded_values(const orc_csr* A, int fmt, orc_csr* out, double* buf) {
  *out = *A;
  for (int64_t k = 0; k < A->rp[A->n]; ++k) buf[k] = R(A->v[k], fmt);
  out->v = buf;
}

/* cg_solve, inner_solver.cpp:47-83. */
static int cg_solve(const orc_csr* A0, const double* rhs, double eps, int max_inner, int fmt, int af,
                    double stop_norm, double* x, int* iters) {
  const int64_t n = A0->n;
  double* vb = (double*)malloc((size_t)A0->rp[n] * sizeof(double) + 8);
  orc_csr A;
  rounded_values(A0, fmt, &A, vb);
  const double target = eps * stop_norm;
  double* r = (double*)malloc((size_t)n * 8);
  double* p = (double*)malloc((size_t)n * 8);
  double* Ap = (double*)malloc((size_t)n * 8);
  for (int64_t i = 0; i < n; ++i) {
    x[i] = 0.0;
    r[i] = R(rhs[i], fmt);
    p[i] = r[i];
  }
  double rs = orc_dot(r, r, n, af);
  int status = GADI_INNER_STAGNATED, it;
  int done = 0;
  for (it = 0; it < max_inner; ++it) {
    if (orc_norm2_64(r, n) <= target) {
      *iters = it;
      status = GADI_INNER_CONVERGED;
      done = 1;
      break;
    }
    matvec_s(&A, p, af, fmt, Ap);
    const double pap = orc_dot(p, Ap, n, af);
    if (pap == 0.0 || !isfinite(pap)) break;
    const double a = R(rs / pap, af);
    axpy_s(a, p, x, n, af, fmt, x);
    axpy_s(-a, Ap, r, n, af, fmt, r);
    const double rs_new = orc_dot(r, r, n, af);
    if (!isfinite(rs_new) || !all_finite(r, n)) {
      *iters = it + 1;
      status = GADI_INNER_OVERFLOW;
      done = 1;
      break;
    }
    const double beta = R(rs_new / rs, af);
    axpy_s(beta, p, r, n, af, fmt, p);
    rs = rs_new;
  }
  if (!done) {
    *iters = max_inner;
    status = all_finite(x, n) ? GADI_INNER_STAGNATED : GADI_INNER_OVERFLOW;
  }
  free(vb);
  free(r);
  free(p);
  free(Ap);
  return status;
}

/* the fused mode's basis scaling: round_fmt(round_af(round_af(a) * x)) (scale_rn<T, true> on the device) */
static void scale_af(double a, const double* x, int64_t n, int af, int fmt, double* z) {
  const double aa = R(a, af);
  for (int64_t i = 0; i < n; ++i) z[i] = R(R(aa * x[i], af), fmt);
}

/* gmres_solve, inner_solver.cpp:85-194. */
static int gmres_solve(const orc_csr* A0, const double* rhs, double eps, int max_inner, int restart,
                       int fmt, int af, double stop_norm, double* x, int* iters) {
  const int64_t n = A0->n;
  double* vb = (double*)malloc((size_t)A0->rp[n] * sizeof(double) + 8);
  orc_csr A;
  rounded_values(A0, fmt, &A, vb);
  const double target = eps * stop_norm;
  const int m = restart > 1 ? restart : 1;
  /* The GADI_ACCUM_FP32 extension mode (af != fmt; not in the reference) runs the
   * Arnoldi step as the device's fused passes do: classical Gram-Schmidt (all
   * dots of a step from the same w, then ONE update pass w -= sum h_i v_i in af
   * with a single rounding to fmt), the norms beta and h(j+1, j) as sqrt(dot(., .))
   * in af, and the
   * basis scaling v = w / h as a product in af (scale_af).
   * The reference's modified Gram-Schmidt and max-scaled norm2
   * (inner_solver.cpp:121-126) stay as they are for af == fmt. */
  const int fused = af != fmt && !getenv("ORC_GMRES_MGS");
  double* V = (double*)malloc((size_t)(m + 1) * (size_t)n * 8);
  double* r = (double*)malloc((size_t)n * 8);
  double* w = (double*)malloc((size_t)n * 8);
  double* Hc = (double*)calloc((size_t)(m + 1) * (size_t)m, 8);
  double* cs = (double*)calloc((size_t)m, 8);
  double* sn = (double*)calloc((size_t)m, 8);
  double* g = (double*)calloc((size_t)m + 1, 8);
  double* y = (double*)calloc((size_t)m + 1, 8);
#define HC(i, j) Hc[(size_t)(i) * (size_t)m + (size_t)(j)]
  for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
  int total = 0, status = -1;
  while (total < max_inner) {
    orc_residual(&A, x, rhs, af, fmt, r);
    if (!all_finite(r, n)) {
      status = GADI_INNER_OVERFLOW;
      break;
    }
    const double beta = fused ? R(sqrt(orc_dot(r, r, n, af)), af) : orc_norm2(r, n, af);
    if (orc_norm2_64(r, n) <= target) {
      status = GADI_INNER_CONVERGED;
      break;
    }
    if (beta == 0.0) break;
    int nv = 1;
    if (fused) scale_af(1.0 / beta, r, n, af, fmt, V);
    else orc_scale(1.0 / beta, r, n, fmt, V);
    memset(Hc, 0, (size_t)(m + 1) * (size_t)m * 8);
    memset(cs, 0, (size_t)m * 8);
    memset(sn, 0, (size_t)m * 8);
    memset(g, 0, (size_t)(m + 1) * 8);
    g[0] = beta;
    int j = 0, happy = 0;
    for (; j < m && total < max_inner; ++j, ++total) {
      matvec_s(&A, V + (size_t)j * n, af, fmt, w);
      double h1;
      if (fused) { /* classical Gram-Schmidt: every h_ij from the same w, one update pass */
        for (int i = 0; i <= j; ++i) HC(i, j) = orc_dot(w, V + (size_t)i * n, n, af);
        for (int64_t e = 0; e < n; ++e) {
          double acc = w[e];
          for (int i = 0; i <= j; ++i) acc = R(acc + R(-HC(i, j) * V[(size_t)i * n + e], af), af);
          w[e] = R(acc, fmt);
        }
        h1 = R(sqrt(orc_dot(w, w, n, af)), af);
      } else {
        for (int i = 0; i <= j; ++i) {
          const double h = orc_dot(w, V + (size_t)i * n, n, af);
          HC(i, j) = h;
          axpy_s(-h, V + (size_t)i * n, w, n, af, fmt, w);
        }
        h1 = orc_norm2(w, n, af);
      }
      HC(j + 1, j) = h1;
      if (!isfinite(h1)) {
        status = GADI_INNER_OVERFLOW;
        goto out;
      }
      if (h1 != 0.0) {
        if (fused) scale_af(1.0 / h1, w, n, af, fmt, V + (size_t)nv * n);
        else orc_scale(1.0 / h1, w, n, fmt, V + (size_t)nv * n);
        ++nv;
      }
      for (int i = 0; i < j; ++i) {
        const double t1 = R(R(cs[i] * HC(i, j), af) + R(sn[i] * HC(i + 1, j), af), af);
        const double t2 = R(R(cs[i] * HC(i + 1, j), af) - R(sn[i] * HC(i, j), af), af);
        HC(i, j) = t1;
        HC(i + 1, j) = t2;
      }
      const double a = HC(j, j), b = HC(j + 1, j);
      const double denom = R(hypot(a, b), af);
      if (denom == 0.0) {
        happy = 1;
        ++j;
        ++total;
        break;
      }
      cs[j] = R(a / denom, af);
      sn[j] = R(b / denom, af);
      HC(j, j) = denom;
      HC(j + 1, j) = 0.0;
      const double gj = g[j];
      g[j] = R(cs[j] * gj, af);
      g[j + 1] = R(-sn[j] * gj, af);
      if (fabs(g[j + 1]) <= target || h1 == 0.0) {
        happy = 1;
        ++j;
        ++total;
        break;
      }
    }
    for (int i = j - 1; i >= 0; --i) {
      double acc = g[i];
      for (int k = i + 1; k < j; ++k) acc = R(acc - R(HC(i, k) * y[k], af), af);
      y[i] = R(acc / HC(i, i), af);
    }
    for (int i = 0; i < j; ++i) axpy_s(y[i], V + (size_t)i * n, x, n, af, fmt, x);
    if (!all_finite(x, n)) {
      status = GADI_INNER_OVERFLOW;
      break;
    }
    if (happy) {
      orc_residual(&A, x, rhs, af, fmt, r);
      if (orc_norm2_64(r, n) <= target) {
        status = GADI_INNER_CONVERGED;
        break;
      }
    }
  }
out:
  if (status < 0) status = all_finite(x, n) ? GADI_INNER_STAGNATED : GADI_INNER_OVERFLOW;
  *iters = total;
#undef HC
  free(vb);
  free(V);
  free(r);
  free(w);
  free(Hc);
  free(cs);
  free(sn);
  free(g);
  free(y);
  return status;
}

/* krylov_solve, inner_solver.cpp:198-204. */
int orc_krylov_af(const orc_csr* M, const double* rhs, int method, double eps, int max_inner, int restart,
                  int fmt, int af, double stop_norm, double* x, int* iters, int* status) {
  if (method == GADI_INNER_CG)
    *status = cg_solve(M, rhs, eps, max_inner, fmt, af, stop_norm, x, iters);
  else
    *status = gmres_solve(M, rhs, eps, max_inner, restart, fmt, af, stop_norm, x, iters);
  return 0;
}
int orc_krylov(const orc_csr* M, const double* rhs, int method, double eps, int max_inner, int restart,
               int fmt, double stop_norm, double* x, int* iters, int* status) {
  return orc_krylov_af(M, rhs, method, eps, max_inner, restart, fmt, fmt, stop_norm, x, iters, status);
}


/* ------------------------------------------------------------------ band LU
 * BandLU (band_lu.cpp:60-199): LAPACK-style band storage with kl extra
 * superdiagonals of fill, partial pivoting, every scalar op of the
 * elimination and the triangular solves rounded once to fmt. Values are
 * carried in binary64: a*b of two binary16/32 numbers is exact in binary64,
 * a-b of binary16 numbers is exact too, and the remaining roundings through
 * binary64 are innocuous (53 >= 2p+2), so R(a op b) equals the reference's
 * float-domain policies (band_lu.cpp:12-56) bit for bit. */
#define AT(f, i, j) (f)->ab[(j) * (f)->ldab + ((f)->kl + (f)->ku + (i) - (j))]

static double lu_tiny(int fmt) { /* format(fmt).min_normal */
  return fmt == GADI_HALF ? 0x1p-14 : fmt == GADI_SINGLE ? 0x1p-126 : 0x1p-1022;
}

/* lower/upper_bandwidth, sparse.cpp:142-154 */
static void bandwidths(const orc_csr* A, int64_t* kl, int64_t* ku) {
  int64_t l = 0, u = 0;
  for (int64_t i = 0; i < A->n; ++i)
    if (A->rp[i] < A->rp[i + 1]) {
      if (i - A->ci[A->rp[i]] > l) l = i - A->ci[A->rp[i]];
      if (A->ci[A->rp[i + 1] - 1] - i > u) u = A->ci[A->rp[i + 1] - 1] - i;
    }
  *kl = l;
  *ku = u;
}

/* BandLU::BandLU + factor, band_lu.cpp:60-135. Returns 0, or the SolveStatus
 * the reference's exception maps to in run_gadi_ir (solver.cpp:74-82):
 * GADI_SINGULAR_IN_PRECISION (pivot below min_normal, :106-108) or
 * GADI_OVERFLOW_DETECTED (non-finite factor entry, :132-134). */
int orc_blu_factor(const orc_csr* A, int fmt, orc_blu* f) {
  const int64_t n = A->n;
  memset(f, 0, sizeof(*f));
  f->n = n;
  f->fmt = fmt;
  bandwidths(A, &f->kl, &f->ku);
  f->ldab = 2 * f->kl + f->ku + 1;
  f->ab = (double*)calloc((size_t)(f->ldab * n), 8);
  f->ipiv = (int64_t*)calloc((size_t)n, 8);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) AT(f, i, A->ci[k]) = R(A->v[k], fmt);
  const double tiny = lu_tiny(fmt);
  const int64_t band_cols = f->kl + f->ku;
  for (int64_t j = 0; j < n; ++j) {
    const int64_t ilast = n - 1 < j + f->kl ? n - 1 : j + f->kl;
    int64_t p = j;
    double pmax = fabs(AT(f, j, j));
    for (int64_t i = j + 1; i <= ilast; ++i) {
      const double v = fabs(AT(f, i, j));
      if (v > pmax) {
        pmax = v;
        p = i;
      }
    }
    if (pmax < tiny) return GADI_SINGULAR_IN_PRECISION;
    f->ipiv[j] = p;
    const int64_t klast = n - 1 < j + band_cols ? n - 1 : j + band_cols;
    if (p != j)
      for (int64_t k = j; k <= klast; ++k) {
        const double t = AT(f, j, k);
        AT(f, j, k) = AT(f, p, k);
        AT(f, p, k) = t;
      }
    const double piv = AT(f, j, j);
    for (int64_t i = j + 1; i <= ilast; ++i) AT(f, i, j) = R(AT(f, i, j) / piv, fmt);
    for (int64_t k = j + 1; k <= klast; ++k) {
      const double ajk = AT(f, j, k);
      if (ajk == 0.0) continue;
      for (int64_t i = j + 1; i <= ilast; ++i) AT(f, i, k) = R(AT(f, i, k) - R(AT(f, i, j) * ajk, fmt), fmt);
    }
  }
  for (int64_t t = 0; t < f->ldab * n; ++t)
    if (!isfinite(f->ab[t])) return GADI_OVERFLOW_DETECTED;
  return 0;
}

/* BandLU::solve_impl, band_lu.cpp:137-172. */
void orc_blu_solve(const orc_blu* f, const double* rhs, double* x) {
  const int64_t n = f->n, kl = f->kl, ubw = f->kl + f->ku;
  const int fmt = f->fmt;
  for (int64_t i = 0; i < n; ++i) x[i] = R(rhs[i], fmt);
  for (int64_t j = 0; j < n; ++j) {
    if (f->ipiv[j] != j) {
      const double t = x[j];
      x[j] = x[f->ipiv[j]];
      x[f->ipiv[j]] = t;
    }
    const double xj = x[j];
    if (xj == 0.0) continue;
    const int64_t ilast = n - 1 < j + kl ? n - 1 : j + kl;
    for (int64_t i = j + 1; i <= ilast; ++i) x[i] = R(x[i] - R(AT(f, i, j) * xj, fmt), fmt);
  }
  for (int64_t j = n - 1; j >= 0; --j) {
    const double xj = R(x[j] / AT(f, j, j), fmt);
    x[j] = xj;
    if (xj != 0.0) {
      const int64_t ifirst = j - ubw > 0 ? j - ubw : 0;
      for (int64_t i = ifirst; i < j; ++i) x[i] = R(x[i] - R(AT(f, i, j) * xj, fmt), fmt);
    }
  }
}

void orc_blu_free(orc_blu* f) {
  free(f->ab);
  free(f->ipiv);
  memset(f, 0, sizeof(*f));
}

/* factorize + solve_factored (inner_solver.cpp:27-39) in one call: x = M \ rhs
 * in fmt; returns 0 or the factorization's status (see orc_blu_factor). */
int orc_lu_solve(const orc_csr* M, const double* rhs, int fmt, double* x) {
  orc_blu f;
  const int st = orc_blu_factor(M, fmt, &f);
  if (st == 0) orc_blu_solve(&f, rhs, x);
  orc_blu_free(&f);
  return st;
}
#undef AT

/* -------------------------------------------------------------------- solver */
/* run_gadi_ir (solver.cpp:57-179) over CsrGadiSystem (solver.cpp:183-246).
 * Ms/Ns NULL: the HSS split of A (hss_split); else explicit_splitting(A, Ms, Ns)
 * (splitting.cpp:22-35), H = shift_diagonal(Ms), S = shift_diagonal(Ns). */
int orc_solve_split(const orc_csr* A, const orc_csr* Ms, const orc_csr* Ns, const double* b, const double* x0,
                    const gadi_config* cfg, double* x, double* hist, int cap, gadi_report* rep) {
  const int64_t n = A->n;
  if (Ms && orc_explicit_check(A, Ms, Ns) != GADI_OK) return GADI_E_CONTRACT;
  /* validate, solver.cpp:33-40 */
  if (!(cfg->alpha > 0.0)) return GADI_E_PARAM;
  if (!(cfg->omega >= 0.0 && cfg->omega < 2.0)) return GADI_E_PARAM;
  if (cfg->xi < 0.0) return GADI_E_PARAM;
  if (cfg->max_outer_iters < 1) return GADI_E_PARAM;
  const double uu = unit_roundoff(cfg->u), uf = unit_roundoff(cfg->u_f), ur = unit_roundoff(cfg->u_r);
  if (!(uu <= uf && uf <= ur)) return GADI_E_PARAM;
  if (cfg->inner.method < 0 || cfg->inner.method > 2) return GADI_E_PARAM;
  const double xi = cfg->xi > 0.0 ? cfg->xi : (cfg->u == D ? 1e-26 : cfg->u == GADI_SINGLE ? 1e-8 : 1e-4);
  const int ur_p = cfg->u_r, u_p = cfg->u;
  /* inner arithmetic: u_r (the reference), or binary32 over binary16 storage
   * under GADI_ACCUM_FP32 (gadi_cuda.h; the device's h32 engine) */
  const int af_p = (cfg->accum == GADI_ACCUM_FP32 && ur_p == GADI_HALF) ? GADI_SINGLE : ur_p;

  memset(rep, 0, sizeof(*rep));
  rep->status = GADI_MAX_ITERS;
  rep->final_rres = 1.0;
  int hl = 0;
#define PUSH_HIST(v) (hl < cap ? (hist[hl] = (v)) : 0, ++hl)
  PUSH_HIST(1.0);

  double* s = (double*)malloc((size_t)n * 8);
  double* rhat = (double*)malloc((size_t)n * 8);
  double* z = (double*)malloc((size_t)n * 8);
  double* pz = (double*)malloc((size_t)n * 8);
  double* yv = (double*)malloc((size_t)n * 8);
  int64_t nnzH = Ms ? orc_shift_diagonal(Ms, cfg->alpha, NULL, NULL, NULL)
                    : orc_regularize(A, cfg->alpha, NULL, NULL, NULL, NULL);
  orc_csr H = {n, (int64_t*)malloc((size_t)(n + 1) * 8), (int64_t*)malloc((size_t)nnzH * 8 + 8),
               (double*)malloc((size_t)nnzH * 8 + 8)};
  orc_csr S = H;
  if (Ms) {
    const int64_t nnzS = orc_shift_diagonal(Ns, cfg->alpha, NULL, NULL, NULL);
    S.rp = (int64_t*)malloc((size_t)(n + 1) * 8);
    S.ci = (int64_t*)malloc((size_t)nnzS * 8 + 8);
    S.v = (double*)malloc((size_t)nnzS * 8 + 8);
  } else {
    S.v = (double*)malloc((size_t)nnzH * 8 + 8);
  }

  for (int64_t i = 0; i < n; ++i) x[i] = R(x0 ? x0[i] : (cfg->ones_start ? 1.0 : 0.0), u_p);
  double last = 1.0;
  /* true_residual_norm, solver.cpp:194-197 */
#define TRUE_NORM(out)                        \
  do {                                        \
    orc_residual(A, x, b, D, D, s);           \
    out = orc_norm2_64(s, n);                 \
  } while (0)
  double nt0;
  TRUE_NORM(nt0);
  if (nt0 == 0.0) {
    rep->status = GADI_CONVERGED;
    rep->final_rres = 0.0;
    goto done;
  }
  if (Ms) { /* prepare, solver.cpp:199-208 */
    orc_shift_diagonal(Ms, cfg->alpha, H.rp, H.ci, H.v);
    orc_shift_diagonal(Ns, cfg->alpha, S.rp, S.ci, S.v);
  } else {
    orc_regularize(A, cfg->alpha, H.rp, H.ci, H.v, S.v);
  }
  const int lu = cfg->inner.method == GADI_INNER_LU_DIRECT;
  orc_blu fH, fS;
  memset(&fH, 0, sizeof(fH));
  memset(&fS, 0, sizeof(fS));
  if (lu) { /* prepare: factorize H then S in u_r (solver.cpp:204-207); a throw -> status (:74-82) */
    int st = orc_blu_factor(&H, ur_p, &fH);
    if (st == 0) st = orc_blu_factor(&S, ur_p, &fS);
    if (st != 0) {
      rep->status = st;
      orc_blu_free(&fH);
      orc_blu_free(&fS);
      goto done;
    }
  }

  int e = 0;
  /* rounded_scaled_residual, solver.cpp:86-92 + scaling_exponent :48-53 */
#define RSR()                                                                         \
  do {                                                                                \
    orc_residual(A, x, b, cfg->u_f, D, s);                                            \
    e = 0;                                                                            \
    if (cfg->residual_scaling) {                                                      \
      double m_ = inf_norm(s, n);                                                     \
      if (m_ != 0.0 && isfinite(m_)) e = ilogb(m_);                                   \
    }                                                                                 \
    for (int64_t i_ = 0; i_ < n; ++i_) rhat[i_] = R(e != 0 ? ldexp(s[i_], -e) : s[i_], ur_p); \
  } while (0)
  RSR();
  const double g0 = ldexp(orc_norm2_64(rhat, n), e);
  double stop_norm = ldexp(g0, -e);
  const double p_rounded = R((2.0 - cfg->omega) * cfg->alpha, ur_p);
  const int s_method = cfg->inner.method == GADI_INNER_CG ? GADI_INNER_GMRES : cfg->inner.method;

  double best = 1.0;
  int best_iter = 0;
  for (int k = 0;; ++k) {
    const double rres = last;
    rep->final_rres = rres;
    rep->outer_iters = k;
    const double gn = ldexp(orc_norm2_64(rhat, n), e);
    const int guard = gn * gn <= g0 * g0 * xi;
    const int truem = rres * rres <= xi;
    if (guard && truem) { rep->status = GADI_CONVERGED; break; }
    if (guard) { rep->status = GADI_STALLED; break; }
    if (!isfinite(rres)) { rep->status = GADI_OVERFLOW_DETECTED; break; }
    if (rres > cfg->divergence_factor) { rep->status = GADI_DIVERGED; break; }
    if (cfg->stall_window > 0) {
      if (rres < best * (1.0 - 1e-3)) {
        best = rres;
        best_iter = k;
      } else if (k - best_iter >= cfg->stall_window) {
        rep->status = GADI_STALLED;
        break;
      }
    }
    if (k >= cfg->max_outer_iters) { rep->status = GADI_MAX_ITERS; break; }

    int it = 0, st = 0;
    if (lu) { /* inner_solve LuDirect (solver.cpp:226-231): no iterations, Overflow if non-finite */
      orc_blu_solve(&fH, rhat, z);
      st = all_finite(z, n) ? GADI_INNER_CONVERGED : GADI_INNER_OVERFLOW;
    } else
      orc_krylov_af(&H, rhat, cfg->inner.method, cfg->inner.tol_epsilon, cfg->inner.max_inner_iters,
                    cfg->inner.restart, ur_p, af_p, stop_norm, z, &it, &st);
    rep->inner_iter_totals += it;
    rep->h_iters += it;
    if (st == GADI_INNER_OVERFLOW) { rep->status = GADI_OVERFLOW_DETECTED; break; }
    if (st == GADI_INNER_STAGNATED) ++rep->inner_stagnations;
    orc_scale(p_rounded, z, n, ur_p, pz);
    if (lu) {
      it = 0;
      orc_blu_solve(&fS, pz, yv);
      st = all_finite(yv, n) ? GADI_INNER_CONVERGED : GADI_INNER_OVERFLOW;
    } else
      orc_krylov_af(&S, pz, s_method, cfg->inner.tol_epsilon, cfg->inner.max_inner_iters,
                    cfg->inner.restart, ur_p, af_p, stop_norm, yv, &it, &st);
    rep->inner_iter_totals += it;
    rep->s_iters += it;
    if (st == GADI_INNER_OVERFLOW) { rep->status = GADI_OVERFLOW_DETECTED; break; }
    if (st == GADI_INNER_STAGNATED) ++rep->inner_stagnations;
    if (e != 0)
      for (int64_t i = 0; i < n; ++i) yv[i] = ldexp(yv[i], e);
    orc_axpy(1.0, yv, x, n, u_p, x);
    if (!all_finite(x, n)) {
      double tn;
      TRUE_NORM(tn);
      last = tn / nt0;
      PUSH_HIST(last);
      rep->outer_iters = k + 1;
      rep->final_rres = last;
      rep->status = GADI_OVERFLOW_DETECTED;
      break;
    }
    RSR();
    stop_norm = ldexp(g0, -e);
    double tn;
    TRUE_NORM(tn);
    last = tn / nt0;
    PUSH_HIST(last);
  }
  orc_blu_free(&fH);
  orc_blu_free(&fS);
done:
  rep->history_len = hl;
  free(s);
  free(rhat);
  free(z);
  free(pz);
  free(yv);
  if (Ms) {
    free(S.rp);
    free(S.ci);
  }
  free(H.rp);
  free(H.ci);
  free(H.v);
  free(S.v);
  return GADI_OK;
#undef PUSH_HIST
#undef TRUE_NORM
#undef RSR
}

int orc_solve(const orc_csr* A, const double* b, const double* x0, const gadi_config* cfg, double* x,
              double* hist, int cap, gadi_report* rep) {
  return orc_solve_split(A, NULL, NULL, b, x0, cfg, x, hist, cap, rep);
}


/* ------------------------------------------------------- training set (GPR)
 * alpha_bisection (gpr.cpp:15-50) over the convdiff family (problems.cpp:8-43,
 * r = 1/(2n+2), b = A * ones): budget log-spaced probes, each a solve with
 * u_r = u = u_f = fmt; the fewest outer iterations among converged probes
 * wins (strict <: ties keep the smaller alpha). Returns 0, GADI_E_PARAM or
 * GADI_E_NO_CONVERGENT_ALPHA. */
int orc_alpha_bisection(int64_t n, int fmt, double lo, double hi, int budget, const gadi_dichotomy* st,
                        double* alpha, int* iters) {
  if (!(lo > 0.0) || !(hi > lo)) return GADI_E_PARAM;
  if (budget < 3) return GADI_E_PARAM;
  const int64_t N = n * n * n;
  const double r = 1.0 / (2.0 * (double)n + 2.0);
  int64_t* rp = (int64_t*)malloc((size_t)(N + 1) * 8);
  int64_t* ci = (int64_t*)malloc((size_t)(7 * N) * 8);
  double* v = (double*)malloc((size_t)(7 * N) * 8);
  double* b = (double*)malloc((size_t)N * 8);
  double* ones = (double*)malloc((size_t)N * 8);
  double* x = (double*)malloc((size_t)N * 8);
  orc_convdiff_csr(n, 6.0, -1.0 - r, -1.0 + r, rp, ci, v);
  orc_csr A = {N, rp, ci, v};
  for (int64_t i = 0; i < N; ++i) ones[i] = 1.0;
  orc_matvec(&A, ones, D, b);
  const double ratio = hi / lo;
  double best_alpha = 0.0;
  long long best = 0x7fffffffffffffffLL;
  for (int i = 0; i < budget; ++i) {
    const double a = lo * pow(ratio, (double)i / (double)(budget - 1));
    gadi_config cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.alpha = a;
    cfg.omega = 1.0;
    cfg.xi = st->train_xi;
    cfg.u_r = cfg.u = cfg.u_f = fmt;
    cfg.inner = st->inner;
    cfg.max_outer_iters = st->max_outer;
    cfg.divergence_factor = 1e6;
    cfg.residual_scaling = 1;
    gadi_report rep;
    double h1;
    orc_solve(&A, b, NULL, &cfg, x, &h1, 1, &rep);
    if (rep.status == GADI_CONVERGED && (long long)rep.outer_iters < best) {
      best = rep.outer_iters;
      best_alpha = a;
    }
  }
  free(rp);
  free(ci);
  free(v);
  free(b);
  free(ones);
  free(x);
  if (best_alpha == 0.0) return GADI_E_NO_CONVERGENT_ALPHA;
  *alpha = best_alpha;
  *iters = (int)best;
  return 0;
}

/* ----------------------------------------------------------------------- GPR */
typedef struct {
  double lml, sf, ell, sn;
  double* L;     /* row-major lower factor, m x m */
  double* kinvy; /* m */
} gp_cand;

/* try_fit, gpr.cpp:84-105 (Eigen LLT restated: right-looking Cholesky). */
static int try_fit(const double* x, const double* y, int m, double sf, double ell, double sn,
                   gp_cand* out) {
  double* L = out->L;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      const double d = (x[i] - x[j]) / ell;
      L[(size_t)i * m + j] = sf * exp(-0.5 * d * d);
    }
  const double jit = sn + 1e-12 * (sf > 1.0 ? sf : 1.0);
  for (int i = 0; i < m; ++i) L[(size_t)i * m + i] += jit;
  for (int j = 0; j < m; ++j) {
    double dsum = L[(size_t)j * m + j];
    for (int k = 0; k < j; ++k) dsum -= L[(size_t)j * m + k] * L[(size_t)j * m + k];
    if (!(dsum > 0.0) || !isfinite(dsum)) return 0;
    const double ljj = sqrt(dsum);
    L[(size_t)j * m + j] = ljj;
    for (int i = j + 1; i < m; ++i) {
      double s = L[(size_t)i * m + j];
      for (int k = 0; k < j; ++k) s -= L[(size_t)i * m + k] * L[(size_t)j * m + k];
      L[(size_t)i * m + j] = s / ljj;
    }
  }
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) L[(size_t)i * m + j] = 0.0;
  double* a = out->kinvy;
  for (int i = 0; i < m; ++i) {
    double acc = y[i];
    for (int k = 0; k < i; ++k) acc -= L[(size_t)i * m + k] * a[k];
    a[i] = acc / L[(size_t)i * m + i];
  }
  for (int i = m - 1; i >= 0; --i) {
    double acc = a[i];
    for (int k = i + 1; k < m; ++k) acc -= L[(size_t)k * m + i] * a[k];
    a[i] = acc / L[(size_t)i * m + i];
  }
  double logdet = 0.0, ya = 0.0;
  for (int i = 0; i < m; ++i) logdet += log(L[(size_t)i * m + i]);
  for (int i = 0; i < m; ++i) ya += y[i] * a[i];
  const double lml = -0.5 * ya - logdet - 0.5 * (double)m * log(2.0 * M_PI);
  if (!isfinite(lml)) return 0;
  out->lml = lml;
  out->sf = sf;
  out->ell = ell;
  out->sn = sn;
  return 1;
}

int orc_gpr(const double* sizes, const double* alphas, int m, const gadi_gpr_opts* opts,
            const double* qsizes, int q, double* mean, double* sd, double* params) {
  if (m < 3) return GADI_E_FIT; /* gpr.cpp:110 */
  double* x = (double*)malloc((size_t)m * 8);
  double* y = (double*)malloc((size_t)m * 8);
  double mu = 0.0, tmin = INFINITY;
  for (int i = 0; i < m; ++i) {
    if (!(alphas[i] > 0.0)) {
      free(x);
      free(y);
      return GADI_E_FIT;
    }
    x[i] = log(sizes[i]);
    mu += alphas[i];
    if (alphas[i] < tmin) tmin = alphas[i];
  }
  mu /= (double)m;
  double var = 0.0;
  for (int i = 0; i < m; ++i) {
    y[i] = alphas[i] - mu;
    var += y[i] * y[i];
  }
  var = var / (double)m;
  if (var < 1e-8) var = 1e-8;
  const double span = x[m - 1] - x[0];
  double spacing = span / (double)(m - 1);
  if (spacing < 1e-3) spacing = 1e-3;

  gp_cand best = {-INFINITY, 0, 0, 0, (double*)malloc((size_t)m * m * 8), (double*)malloc((size_t)m * 8)};
  gp_cand cand = {-INFINITY, 0, 0, 0, (double*)malloc((size_t)m * m * 8), (double*)malloc((size_t)m * 8)};
  if (opts && opts->fixed_hypers) {
    if (try_fit(x, y, m, opts->sigma_f2, opts->length, opts->sigma_n2, &cand)) {
      gp_cand t = best;
      best = cand;
      cand = t;
    }
  } else {
    const double sfs[3] = {0.25 * var, 1.0 * var, 4.0 * var};
    const double ells[3] = {0.5 * spacing, 1.0 * spacing, 2.0 * spacing};
    double sns[3] = {1e-10 * var, 1e-8 * var, 1e-6 * var};
    int nsn = 3;
    if (opts && opts->has_sigma_n2) {
      sns[0] = opts->sigma_n2;
      nsn = 1;
    }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        for (int c = 0; c < nsn; ++c)
          if (try_fit(x, y, m, sfs[a], ells[b], sns[c], &cand) && cand.lml > best.lml) {
            gp_cand t = best;
            best = cand;
            cand = t;
          }
  }
  int rc = GADI_OK;
  if (!isfinite(best.lml)) {
    rc = GADI_E_FIT;
  } else {
    double* ks = (double*)malloc((size_t)m * 8);
    for (int t = 0; t < q; ++t) {
      const double xq = log(qsizes[t]);
      double mn = mu;
      for (int i = 0; i < m; ++i) {
        const double d = (xq - x[i]) / best.ell;
        ks[i] = best.sf * exp(-0.5 * d * d);
      }
      double kd = 0.0;
      for (int i = 0; i < m; ++i) kd += ks[i] * best.kinvy[i];
      mn += kd;
      double vn = 0.0;
      for (int i = 0; i < m; ++i) { /* v = L^-1 k (in place) */
        double acc = ks[i];
        for (int k = 0; k < i; ++k) acc -= best.L[(size_t)i * m + k] * ks[k];
        ks[i] = acc / best.L[(size_t)i * m + i];
      }
      for (int i = 0; i < m; ++i) vn += ks[i] * ks[i];
      double v = best.sf + best.sn - vn;
      if (v < 0.0) v = 0.0;
      if (mn < tmin / 10.0) mn = tmin / 10.0;
      mean[t] = mn;
      sd[t] = sqrt(v);
    }
    free(ks);
    params[0] = best.sf;
    params[1] = best.ell;
    params[2] = best.sn;
    params[3] = mu;
    params[4] = best.lml;
  }
  free(best.L);
  free(best.kinvy);
  free(cand.L);
  free(cand.kinvy);
  free(x);
  free(y);
  return rc;
}

/* x_i = U(seed, i) in [lo, hi); b = A x in binary64 (matvec, kernels.cpp:41-54;
 * the reference builds b = A * x_exact the same way, problems.cpp:44). */
void orc_make_rhs(const orc_csr* A, uint64_t seed, double lo, double hi, double* x, double* b) {
  for (int64_t i = 0; i < A->n; ++i) x[i] = orc_uniform(seed, (uint64_t)i, lo, hi);
  orc_matvec(A, x, D, b);
}
