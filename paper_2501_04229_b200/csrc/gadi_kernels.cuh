// gadi_kernels.cuh — the device kernels of the GADI-IR hot path.
//
// One thread owns one reduction segment (see gadi_common.cuh); every kernel
// that produces a dot product or norm folds it into the same pass that writes
// the vector (SpMV + p.Ap; the two CG axpys + r.r + ||r||_2; GMRES MGS axpy +
// the next Arnoldi dot), and the last block to finish evaluates the top of
// the pairwise tree and the scalar recurrences (alpha, beta, stop tests) on
// the device, so the host never waits inside an inner iteration.
//
// Template parameters: Op (Stencil7 / Csr), T (storage: __half, float,
// double), C (arithmetic: T, or float for binary16 storage with binary32
// accumulation), VEC (elements per thread on the aligned path; 1 = general).
#pragma once

#include "gadi_common.cuh"
#include "gadi_ops.cuh"

namespace gadi {

struct Geo {
  int64_t N;
  int D;     // tree depth of the segments
  int bdim;  // threads per block (power of 2)
  int nblk;  // blocks (power of 2); nblk * bdim = 2^D segments
};

struct Red {
  double* part0;
  double* part1;
  unsigned* ticket;
};

// Device-resident solver state (one per handle).
struct DevState {
  // CG (inner_solver.cpp:47-83)
  int cg_done, cg_status, cg_iters, cg_it, cg_max, cg_flags;
  double cg_rs, cg_pap, cg_a, cg_beta, cg_target;
  // generic reduction outputs
  double red_c, red_d;
  int flags;
  int pad0;
  unsigned long long maxbits;
  // GMRES Arnoldi column, h(0..j+1, j)
  double hcol[72];
  double ycoef[72];
  // outer loop
  double res_ss, res_max, rhat_ss;
  int res_e, xbad;
  int* hdone;  // mapped host flag raised when a CG solve finishes
};

enum : int { INNER_CONVERGED = 0, INNER_STAGNATED = 1, INNER_OVERFLOW = 2 };

__device__ __forceinline__ void cg_finish(DevState* st, int status, int iters) {
  st->cg_done = 1;
  st->cg_status = status;
  st->cg_iters = iters;
  if (st->hdone) {
    *(volatile int*)st->hdone = 1;
    __threadfence_system();
  }
}

// ------------------------------------------------------------ reductions
// Reduce v0 (pairwise in C) and v1 (pairwise in binary64) over the grid.
// Returns true in exactly one thread (thread 0 of the last block), which
// then holds the totals. Every thread of every block must call it.
template <class C0>
__device__ __forceinline__ bool grid_finish(C0 v0, double v1, const Geo& g, const Red& r, C0& t0,
                                            double& t1) {
  __shared__ __align__(8) unsigned char smb0[32 * sizeof(double)];
  __shared__ double sm1[32];
  __shared__ int last;
  C0* sm0 = reinterpret_cast<C0*>(smb0);
  C0 b0 = block_tree(v0, g.bdim, sm0);
  double b1 = block_tree(v1, g.bdim, sm1);
  if (threadIdx.x == 0) {
    r.part0[blockIdx.x] = to_dbl(b0);
    r.part1[blockIdx.x] = b1;
    __threadfence();
    const unsigned t = atomicAdd(r.ticket, 1u);
    last = (t == (unsigned)g.nblk - 1u);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  const int P = g.nblk, B = blockDim.x, tid = threadIdx.x;
  C0 a0;
  double a1;
  int cnt;
  if (P <= B) {
    a0 = tid < P ? from_dbl<C0>(__ldcg(r.part0 + tid)) : Ar<C0>::zero();
    a1 = tid < P ? __ldcg(r.part1 + tid) : 0.0;
    cnt = P;
  } else {
    const int64_t L = P / B;
    const double* p0 = r.part0 + (int64_t)tid * L;
    const double* p1 = r.part1 + (int64_t)tid * L;
    a0 = run_pairwise<C0>(L, [&](int64_t j) { return from_dbl<C0>(__ldcg(p0 + j)); });
    a1 = run_pairwise<double>(L, [&](int64_t j) { return __ldcg(p1 + j); });
    cnt = B;
  }
  a0 = block_tree(a0, cnt, sm0);
  a1 = block_tree(a1, cnt, sm1);
  if (tid == 0) {
    *r.ticket = 0u;
    t0 = a0;
    t1 = a1;
  }
  return tid == 0;
}

// Block-wide OR of f into *dst (one global atomic per block, issued by
// thread 0 before it takes the grid ticket).
__device__ __forceinline__ void or_flags(int* dst, int f) {
  __shared__ int sf;
  if (threadIdx.x == 0) sf = 0;
  __syncthreads();
  if (f) atomicOr(&sf, f);
  __syncthreads();
  if (threadIdx.x == 0 && sf) atomicOr(dst, sf);
}

__device__ __forceinline__ void block_max_abs(unsigned long long* dst, double m) {
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0 && m > 0.0) {
    atomic_max_abs(dst, m);
    __threadfence();
  }
}

// ------------------------------------------------------------ segment I/O
template <class T, int VEC, int G>
__device__ __forceinline__ void load_seg(const T* __restrict__ p, const Seg& s, T (&v)[G]) {
  if constexpr (VEC > 1) {
    ld_vec<T, VEC>(p, s.lo, v);
  } else {
#pragma unroll
    for (int i = 0; i < G; ++i) v[i] = i < s.len ? p[s.lo + i] : from_dbl<T>(0.0);
  }
}
template <class T, int VEC, int G>
__device__ __forceinline__ void store_seg(T* __restrict__ p, const Seg& s, const T (&v)[G]) {
  if constexpr (VEC > 1) {
    st_vec<T, VEC>(p, s.lo, v);
  } else {
#pragma unroll
    for (int i = 0; i < G; ++i)
      if (i < s.len) p[s.lo + i] = v[i];
  }
}
// Operator fold over a segment: aligned = one VEC-wide row fold, general =
// element by element.
template <int VEC, int G, class Op, class X, class Acc, class F>
__device__ __forceinline__ void fold_seg(const Op& op, const X* __restrict__ x, const Seg& s,
                                         Acc (&acc)[G], F f) {
  if constexpr (VEC > 1) {
    op.template fold<VEC>(x, s.lo, acc, f);
  } else {
#pragma unroll
    for (int i = 0; i < G; ++i)
      if (i < s.len) {
        Acc a1[1] = {acc[i]};
        op.template fold<1>(x, s.lo + i, a1, f);
        acc[i] = a1[0];
      }
  }
}

#define GADI_SEG()                                                     \
  constexpr int G = VEC > 1 ? VEC : 4;                                 \
  const int64_t tix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  \
  const Seg s = seg_of<VEC>(tix, g.N, g.D);                            \
  (void)G

template <class C, class T>
struct MatvecF {  // acc + coef * x (kernels.cpp:47-52)
  __device__ __forceinline__ C operator()(C a, C coef, T xv) const {
    return Ar<C>::add(a, Ar<C>::mul(coef, ld_c<T, C>(xv)));
  }
};
template <class C, class T>
struct ResidF {  // acc - coef * x (kernels.cpp:63-66)
  __device__ __forceinline__ C operator()(C a, C coef, T xv) const {
    return Ar<C>::sub(a, Ar<C>::mul(coef, ld_c<T, C>(xv)));
  }
};
template <int P>
struct ResidAF {  // binary64-carried residual rounded to u_f per op
  __device__ __forceinline__ double operator()(double a, double coef, double xv) const {
    return round_p<P>(__dsub_rn(a, round_p<P>(__dmul_rn(coef, xv))));
  }
};
struct MatvecAF {  // b = A x in binary64 (problems.cpp:44)
  __device__ __forceinline__ double operator()(double a, double coef, double xv) const {
    return __dadd_rn(a, __dmul_rn(coef, xv));
  }
};

// ================================================================== CG
// r = p = rhs, x = 0, rs = dot(r, r) (inner_solver.cpp:51-55); initial stop test.
template <class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_cg_init(const T* __restrict__ rhs, T* __restrict__ r,
                                                 T* __restrict__ p, T* __restrict__ x, int max_inner,
                                                 double target, Geo g, Red rd, DevState* st) {
  GADI_SEG();
  T v[G], z[G];
  load_seg<T, VEC, G>(rhs, s, v);
#pragma unroll
  for (int i = 0; i < G; ++i) z[i] = from_dbl<T>(0.0);
  store_seg<T, VEC, G>(r, s, v);
  store_seg<T, VEC, G>(p, s, v);
  store_seg<T, VEC, G>(x, s, z);
  C tc[G];
  double td[G];
#pragma unroll
  for (int i = 0; i < G; ++i) {
    const C c = ld_c<T, C>(v[i]);
    tc[i] = Ar<C>::mul(c, c);
    const double d = to_dbl(v[i]);
    td[i] = d * d;
  }
  C sc = seg_sum<C, G>(tc, s.len);
  double sd = seg_sum<double, G>(td, s.len);
  C rs;
  double ss;
  if (grid_finish(sc, sd, g, rd, rs, ss)) {
    st->cg_rs = to_dbl(rs);
    st->cg_it = 0;
    st->cg_flags = 0;
    st->cg_max = max_inner;
    st->cg_target = target;
    if (max_inner <= 0) {
      cg_finish(st, INNER_STAGNATED, 0);
    } else if (sqrt(ss) <= target) {
      cg_finish(st, INNER_CONVERGED, 0);
    } else {
      st->cg_done = 0;
    }
  }
}

// q = H p, pap = dot(p, q); alpha = rs / pap or break (inner_solver.cpp:62-65).
template <class Op, class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_cg_spmv(Op op, const T* __restrict__ p, T* __restrict__ q,
                                                 Geo g, Red rd, DevState* st) {
  if (*(volatile int*)&st->cg_done) return;
  GADI_SEG();
  C acc[G];
#pragma unroll
  for (int i = 0; i < G; ++i) acc[i] = Ar<C>::zero();
  fold_seg<VEC, G>(op, p, s, acc, MatvecF<C, T>());
  T qv[G], pv[G];
#pragma unroll
  for (int i = 0; i < G; ++i) qv[i] = st_t<T, C>(acc[i]);
  store_seg<T, VEC, G>(q, s, qv);
  load_seg<T, VEC, G>(p, s, pv);
  C tc[G];
#pragma unroll
  for (int i = 0; i < G; ++i) tc[i] = Ar<C>::mul(ld_c<T, C>(pv[i]), ld_c<T, C>(qv[i]));
  C sc = seg_sum<C, G>(tc, s.len);
  C pap;
  double dummy;
  if (grid_finish(sc, 0.0, g, rd, pap, dummy)) {
    const double pd = to_dbl(pap);
    st->cg_pap = pd;
    if (pd == 0.0 || !isfinite(pd)) {
      // `break` -> Stagnated / Overflow with iters = max (:64, :79-81)
      cg_finish(st, (st->cg_flags & 2) ? INNER_OVERFLOW : INNER_STAGNATED, st->cg_max);
    } else {
      st->cg_a = to_dbl(div_c<C>(from_dbl<C>(st->cg_rs), pap));
    }
  }
}

// x += a p; r -= a q; rs' = dot(r, r); ||r||_2 (binary64) for the next stop
// test; overflow checks (inner_solver.cpp:66-77).
template <class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_cg_update(T* __restrict__ x, T* __restrict__ r,
                                                   const T* __restrict__ p, const T* __restrict__ q, Geo g,
                                                   Red rd, DevState* st) {
  if (*(volatile int*)&st->cg_done) return;
  GADI_SEG();
  const C a = from_dbl<C>(st->cg_a);
  const C na = Ar<C>::neg(a);
  T xv[G], rv[G], pv[G], qv[G];
  load_seg<T, VEC, G>(x, s, xv);
  load_seg<T, VEC, G>(r, s, rv);
  load_seg<T, VEC, G>(p, s, pv);
  load_seg<T, VEC, G>(q, s, qv);
  C tc[G];
  double td[G];
  int bad = 0;
#pragma unroll
  for (int i = 0; i < G; ++i) {
    xv[i] = st_t<T, C>(Ar<C>::add(ld_c<T, C>(xv[i]), Ar<C>::mul(a, ld_c<T, C>(pv[i]))));
    rv[i] = st_t<T, C>(Ar<C>::add(ld_c<T, C>(rv[i]), Ar<C>::mul(na, ld_c<T, C>(qv[i]))));
    const C rc = ld_c<T, C>(rv[i]);
    tc[i] = Ar<C>::mul(rc, rc);
    const double d = to_dbl(rv[i]);
    td[i] = d * d;
    if (VEC > 1 || i < s.len) bad |= (finite_t(rv[i]) ? 0 : 1) | (finite_t(xv[i]) ? 0 : 2);
  }
  store_seg<T, VEC, G>(x, s, xv);
  store_seg<T, VEC, G>(r, s, rv);
  or_flags(&st->cg_flags, bad);
  C sc = seg_sum<C, G>(tc, s.len);
  double sd = seg_sum<double, G>(td, s.len);
  C rsn;
  double ss;
  if (grid_finish(sc, sd, g, rd, rsn, ss)) {
    const int it = st->cg_it;
    const double rn = to_dbl(rsn);
    const int flags = *(volatile int*)&st->cg_flags;
    if (!isfinite(rn) || (flags & 1)) {
      cg_finish(st, INNER_OVERFLOW, it + 1);
    } else {
      st->cg_beta = to_dbl(div_c<C>(rsn, from_dbl<C>(st->cg_rs)));
      st->cg_rs = rn;
      st->cg_it = it + 1;
      if (it + 1 >= st->cg_max) {
        cg_finish(st, (flags & 2) ? INNER_OVERFLOW : INNER_STAGNATED, st->cg_max);
      } else if (sqrt(ss) <= st->cg_target) {
        cg_finish(st, INNER_CONVERGED, it + 1);
      }
    }
  }
}

// p = r + beta p (inner_solver.cpp:76).
template <class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_cg_pupd(const T* __restrict__ r, T* __restrict__ p, Geo g,
                                                 DevState* st) {
  if (*(volatile int*)&st->cg_done) return;
  GADI_SEG();
  const C b = from_dbl<C>(st->cg_beta);
  T rv[G], pv[G];
  load_seg<T, VEC, G>(r, s, rv);
  load_seg<T, VEC, G>(p, s, pv);
#pragma unroll
  for (int i = 0; i < G; ++i) pv[i] = st_t<T, C>(Ar<C>::add(ld_c<T, C>(rv[i]), Ar<C>::mul(b, ld_c<T, C>(pv[i]))));
  store_seg<T, VEC, G>(p, s, pv);
}

// ================================================================ GMRES
// r = rhs - S x in the inner arithmetic (inner_solver.cpp:97 / :182, the
// two-stage residual kernels.cpp:56-69), max|r|, ||r||_2, finiteness.
template <class Op, class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_gm_resid(Op op, const T* __restrict__ x, const T* __restrict__ rhs,
                                                  T* __restrict__ r, Geo g, Red rd, DevState* st) {
  GADI_SEG();
  T bv[G];
  load_seg<T, VEC, G>(rhs, s, bv);
  C acc[G];
#pragma unroll
  for (int i = 0; i < G; ++i) acc[i] = ld_c<T, C>(bv[i]);
  fold_seg<VEC, G>(op, x, s, acc, ResidF<C, T>());
  T rv[G];
  double td[G], m = 0.0;
  int bad = 0;
#pragma unroll
  for (int i = 0; i < G; ++i) {
    rv[i] = st_t<T, C>(acc[i]);
    const double d = to_dbl(rv[i]);
    td[i] = d * d;
    if (VEC > 1 || i < s.len) {
      bad |= finite_t(rv[i]) ? 0 : 1;
      m = fmax(m, fabs(d));
    }
  }
  store_seg<T, VEC, G>(r, s, rv);
  block_max_abs(&st->maxbits, m);
  or_flags(&st->flags, bad);
  double sd = seg_sum<double, G>(td, s.len);
  C dc;
  double ss;
  if (grid_finish(Ar<C>::zero(), sd, g, rd, dc, ss)) st->red_d = ss;
}

// norm2 in the inner format (kernels.cpp:71-82): m = max|w| (from maxbits),
// q = w/m, sum of q*q pairwise, m * sqrt(sum); written to *dst.
template <class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_norm2(const T* __restrict__ w, double* dst, Geo g, Red rd,
                                               DevState* st) {
  GADI_SEG();
  const double m = __longlong_as_double((long long)*(volatile unsigned long long*)&st->maxbits);
  const C mc = from_dbl<C>(m);
  T wv[G];
  load_seg<T, VEC, G>(w, s, wv);
  C tc[G];
#pragma unroll
  for (int i = 0; i < G; ++i) {
    const C q = div_c<C>(ld_c<T, C>(wv[i]), mc);
    tc[i] = Ar<C>::mul(q, q);
  }
  C sc = seg_sum<C, G>(tc, s.len);
  C sum;
  double dummy;
  if (grid_finish(sc, 0.0, g, rd, sum, dummy)) {
    if (m == 0.0 || !isfinite(m)) {
      *dst = m;
    } else {
      const C sq = Ar<C>::from_d(__dsqrt_rn(Ar<C>::to_d(sum)));
      *dst = to_dbl(Ar<C>::mul(mc, sq));
    }
  }
}

// dst = round(a * src) with a in binary64 (scale, kernels.cpp:166-171).
template <class T, int VEC>
__global__ void __launch_bounds__(256) k_scale(const T* __restrict__ src, T* __restrict__ dst, double a, Geo g) {
  GADI_SEG();
  T v[G];
  load_seg<T, VEC, G>(src, s, v);
#pragma unroll
  for (int i = 0; i < G; ++i) v[i] = from_dbl<T>(__dmul_rn(a, to_dbl(v[i])));
  store_seg<T, VEC, G>(dst, s, v);
}

// w = S v_j and h_0j = dot(w, v_0) (inner_solver.cpp:120-122).
template <class Op, class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_gm_matvec(Op op, const T* __restrict__ vj, const T* __restrict__ v0,
                                                   T* __restrict__ w, Geo g, Red rd, DevState* st) {
  GADI_SEG();
  C acc[G];
#pragma unroll
  for (int i = 0; i < G; ++i) acc[i] = Ar<C>::zero();
  fold_seg<VEC, G>(op, vj, s, acc, MatvecF<C, T>());
  T wv[G], v0v[G];
#pragma unroll
  for (int i = 0; i < G; ++i) wv[i] = st_t<T, C>(acc[i]);
  store_seg<T, VEC, G>(w, s, wv);
  load_seg<T, VEC, G>(v0, s, v0v);
  C tc[G];
#pragma unroll
  for (int i = 0; i < G; ++i) tc[i] = Ar<C>::mul(ld_c<T, C>(wv[i]), ld_c<T, C>(v0v[i]));
  C sc = seg_sum<C, G>(tc, s.len);
  C h;
  double dummy;
  if (grid_finish(sc, 0.0, g, rd, h, dummy)) st->hcol[0] = to_dbl(h);
}

// Modified Gram-Schmidt step i (inner_solver.cpp:121-125): w -= h_i v_i, then
// either h_{i+1} = dot(w, v_{i+1}) (i < j) or max|w| for the norm (i == j).
template <class T, class C, int VEC, bool LAST>
__global__ void __launch_bounds__(256) k_gm_mgs(T* __restrict__ w, const T* __restrict__ vi,
                                                const T* __restrict__ vnext, int i, Geo g, Red rd,
                                                DevState* st) {
  GADI_SEG();
  const C nh = Ar<C>::neg(from_dbl<C>(st->hcol[i]));
  T wv[G], vv[G];
  load_seg<T, VEC, G>(w, s, wv);
  load_seg<T, VEC, G>(vi, s, vv);
#pragma unroll
  for (int k = 0; k < G; ++k) wv[k] = st_t<T, C>(Ar<C>::add(ld_c<T, C>(wv[k]), Ar<C>::mul(nh, ld_c<T, C>(vv[k]))));
  store_seg<T, VEC, G>(w, s, wv);
  if constexpr (LAST) {
    double m = 0.0;
#pragma unroll
    for (int k = 0; k < G; ++k)
      if (VEC > 1 || k < s.len) m = fmax(m, fabs(to_dbl(wv[k])));
    block_max_abs(&st->maxbits, m);
  } else {
    load_seg<T, VEC, G>(vnext, s, vv);
    C tc[G];
#pragma unroll
    for (int k = 0; k < G; ++k) tc[k] = Ar<C>::mul(ld_c<T, C>(wv[k]), ld_c<T, C>(vv[k]));
    C sc = seg_sum<C, G>(tc, s.len);
    C h;
    double dummy;
    if (grid_finish(sc, 0.0, g, rd, h, dummy)) st->hcol[i + 1] = to_dbl(h);
  }
}

// x += y_0 v_0; x += y_1 v_1; ... (inner_solver.cpp:174), one pass, the
// sequence of rounded axpys kept per element.
template <class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_gm_update(T* __restrict__ x, const T* __restrict__ V, int64_t ldv,
                                                   int j, Geo g, DevState* st) {
  GADI_SEG();
  T xv[G], vv[G];
  load_seg<T, VEC, G>(x, s, xv);
  C xc[G];
#pragma unroll
  for (int k = 0; k < G; ++k) xc[k] = ld_c<T, C>(xv[k]);
  for (int i = 0; i < j; ++i) {
    const C y = from_dbl<C>(st->ycoef[i]);
    load_seg<T, VEC, G>(V + (int64_t)i * ldv, s, vv);
#pragma unroll
    for (int k = 0; k < G; ++k) xc[k] = ld_c<T, C>(st_t<T, C>(Ar<C>::add(xc[k], Ar<C>::mul(y, ld_c<T, C>(vv[k])))));
  }
  int bad = 0;
#pragma unroll
  for (int k = 0; k < G; ++k) {
    xv[k] = st_t<T, C>(xc[k]);
    if (VEC > 1 || k < s.len) bad |= finite_t(xv[k]) ? 0 : 1;
  }
  store_seg<T, VEC, G>(x, s, xv);
  or_flags(&st->flags, bad);
}

// ============================================================ outer loop
// s = b - A x in u_f (residual_uf, solver.cpp:190-192); max|s|, ||s||_2 and
// the scaling exponent e = ilogb(max|s|) (solver.cpp:48-53). s may be null
// (norm only: true_residual_norm, solver.cpp:194-197).
template <class Op, int PF, int VEC>
__global__ void __launch_bounds__(256) k_resid_A(Op op, const double* __restrict__ x, const double* __restrict__ b,
                                                 double* __restrict__ sv, int scaling, Geo g, Red rd,
                                                 DevState* st) {
  GADI_SEG();
  double acc[G];
  load_seg<double, VEC, G>(b, s, acc);
  fold_seg<VEC, G>(op, x, s, acc, ResidAF<PF>());
  double td[G], m = 0.0;
#pragma unroll
  for (int i = 0; i < G; ++i) {
    td[i] = acc[i] * acc[i];
    if (VEC > 1 || i < s.len) m = (acc[i] == acc[i]) ? fmax(m, fabs(acc[i])) : m;
  }
  if (sv) store_seg<double, VEC, G>(sv, s, acc);
  block_max_abs(&st->maxbits, m);
  double sd = seg_sum<double, G>(td, s.len);
  double dummy, ss;
  if (grid_finish(0.0, sd, g, rd, dummy, ss)) {
    __threadfence();
    const double mx = __longlong_as_double((long long)*(volatile unsigned long long*)&st->maxbits);
    st->res_ss = ss;
    st->res_max = mx;
    st->res_e = (scaling && mx != 0.0 && isfinite(mx)) ? ilogb(mx) : 0;
  }
}

// rhat = round_{u_r}(s * 2^-e) (solver.cpp:86-92) and ||rhat||_2.
template <class T, int VEC>
__global__ void __launch_bounds__(256) k_scale_round(const double* __restrict__ sv, T* __restrict__ rhat, Geo g,
                                                     Red rd, DevState* st) {
  GADI_SEG();
  const int e = st->res_e;
  double v[G], td[G];
  load_seg<double, VEC, G>(sv, s, v);
  T o[G];
#pragma unroll
  for (int i = 0; i < G; ++i) {
    o[i] = from_dbl<T>(e != 0 ? scalbn(v[i], -e) : v[i]);
    const double d = to_dbl(o[i]);
    td[i] = d * d;
  }
  store_seg<T, VEC, G>(rhat, s, o);
  double sd = seg_sum<double, G>(td, s.len);
  double dummy, ss;
  if (grid_finish(0.0, sd, g, rd, dummy, ss)) st->rhat_ss = ss;
}

// x = round_u(x + round_u(2^e y)) (solver.cpp:163-166 with axpy kernels.cpp:147-164).
template <class T, int PU, int VEC>
__global__ void __launch_bounds__(256) k_update(double* __restrict__ x, const T* __restrict__ y, Geo g,
                                                DevState* st) {
  GADI_SEG();
  const int e = st->res_e;
  double xv[G];
  T yv[G];
  load_seg<double, VEC, G>(x, s, xv);
  load_seg<T, VEC, G>(y, s, yv);
  int bad = 0;
#pragma unroll
  for (int i = 0; i < G; ++i) {
    double yd = to_dbl(yv[i]);
    if (e != 0) yd = scalbn(yd, e);
    xv[i] = round_p<PU>(__dadd_rn(xv[i], round_p<PU>(__dmul_rn(1.0, yd))));
    if (VEC > 1 || i < s.len) bad |= isfinite(xv[i]) ? 0 : 1;
  }
  store_seg<double, VEC, G>(x, s, xv);
  or_flags(&st->xbad, bad);
}

// ------------------------------------------------------------ elementwise
template <class TI, class TO, int PR>
__global__ void k_convert(const TI* __restrict__ in, TO* __restrict__ out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = from_dbl<TO>(round_p<PR>(to_dbl(in[i])));
}

__global__ void k_fill(double* __restrict__ x, double v, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform01(uint64_t seed, uint64_t i, double lo, double hi) {
  const double u = __dmul_rn((double)(splitmix64(seed, i) >> 11), 0x1p-53);
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
}
__global__ void k_uniform(double* __restrict__ x, uint64_t seed, double lo, double hi, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = uniform01(seed, (uint64_t)i, lo, hi);
}

// y = Op x with the given fold, one element per thread (tests / rhs).
template <class Op, class X, class Acc, class Y, class F>
__global__ void k_apply(Op op, const X* __restrict__ x, Y* __restrict__ y, int64_t n, F f) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  Acc a[1];
  a[0] = Ar<Acc>::zero();
  op.template fold<1>(x, e, a, f);
  y[e] = st_t<Y, Acc>(a[0]);
}

// dot / norm2 over binary64-carried values in precision C (test entry points).
template <class C>
__global__ void __launch_bounds__(256) k_dot_d(const double* __restrict__ x, const double* __restrict__ y, Geo g,
                                               Red rd, double* out) {
  constexpr int VEC = 1;
  GADI_SEG();
  C tc[G];
#pragma unroll
  for (int i = 0; i < G; ++i)
    tc[i] = i < s.len ? Ar<C>::mul(Ar<C>::from_d(x[s.lo + i]), Ar<C>::from_d(y[s.lo + i])) : Ar<C>::zero();
  C sc = seg_sum<C, G>(tc, s.len);
  C t;
  double dummy;
  if (grid_finish(sc, 0.0, g, rd, t, dummy)) *out = to_dbl(t);
}

}  // namespace gadi
