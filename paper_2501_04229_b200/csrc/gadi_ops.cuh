// gadi_ops.cuh — the operators A, H = alpha I + M, S = alpha I + N on the device.
//
// A fold visits a row's stored entries in ascending column order, exactly as
// the reference's per-row loops (kernels.cpp:41-54 matvec, :56-69 residual)
// visit the CSR it builds; the caller's functor f(acc, coef, x) supplies the
// per-entry rounding (matvec: acc + coef*x; residual: acc - coef*x).
//
// The operand is read through a "source" so that an elementwise producer can
// be fused into the operator pass: PlainSrc reads a vector; PUpdSrc forms
// p = r + beta p on the fly (CG, inner_solver.cpp:76, fused into the next
// SpMV); ScaleSrc forms v = w / h (GMRES basis, inner_solver.cpp:134, fused
// into the next Arnoldi matvec); ZeroSrc is the x = 0 start vector.
#pragma once

#include "gadi_common.cuh"

namespace gadi {

template <class T>
struct PlainSrc {
  const T* __restrict__ p;
  template <int VEC>
  __device__ __forceinline__ void vec(int64_t e0, T (&v)[VEC]) const {
    ld_vec<T, VEC>(p, e0, v);
  }
  __device__ __forceinline__ T at(int64_t e) const { return p[e]; }
};

// The operand window [lo, lo + len) of a banded sparse operator staged in
// shared memory: gathers x[col] hit shared memory (a few bank-conflict
// wavefronts per warp instruction) instead of scattered L1 sectors.
template <class T>
struct SmemSrc {
  const T* w;  // window in shared memory
  int64_t lo;  // global index of w[0] (a multiple of the segment width)
  template <int VEC>
  __device__ __forceinline__ void vec(int64_t e0, T (&v)[VEC]) const {
    const T* p = w + (e0 - lo);
    if constexpr (VEC * sizeof(T) == 16) {
      const uint4 u = *reinterpret_cast<const uint4*>(p);
      const T* t = reinterpret_cast<const T*>(&u);
#pragma unroll
      for (int i = 0; i < VEC; ++i) v[i] = t[i];
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) v[i] = p[i];
    }
  }
  __device__ __forceinline__ T at(int64_t e) const { return w[e - lo]; }
};

template <class T>
struct ZeroSrc {  // the x = 0 start vector (+0 everywhere), no memory traffic
  template <int VEC>
  __device__ __forceinline__ void vec(int64_t, T (&v)[VEC]) const {
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = from_dbl<T>(0.0);
  }
  __device__ __forceinline__ T at(int64_t) const { return from_dbl<T>(0.0); }
};

template <class T, class C>
struct PUpdSrc {  // p_new = first ? r : round(r + beta * p)
  const T* __restrict__ r;
  const T* __restrict__ p;
  C beta;
  int first;
  __device__ __forceinline__ T f(T rv, T pv) const {
    if (first) return rv;
    return st_t<T, C>(Ar<C>::add(ld_c<T, C>(rv), Ar<C>::mul(beta, ld_c<T, C>(pv))));
  }
  template <int VEC>
  __device__ __forceinline__ void vec(int64_t e0, T (&v)[VEC]) const {
    T rv[VEC], pv[VEC];
    ld_vec<T, VEC>(r, e0, rv);
    if (!first) ld_vec<T, VEC>(p, e0, pv);
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = first ? rv[i] : f(rv[i], pv[i]);
  }
  __device__ __forceinline__ T at(int64_t e) const { return first ? r[e] : f(r[e], p[e]); }
};

// round(a * x): the reference's scale (kernels.cpp:166-171) multiplies in
// binary64 and rounds once to the storage format. F32 (the GADI_ACCUM_FP32
// extension mode: binary16 storage, binary32 arithmetic) rounds a to binary32,
// multiplies in binary32 and rounds to binary16 -- no binary64 conversions on
// the Arnoldi passes; the oracle's `fused` mode restates it.
template <class T, bool F32>
__device__ __forceinline__ T scale_rn(double a, T x) {
  if constexpr (F32) {
    static_assert(std::is_same<T, __half>::value, "F32 scaling is the binary16-storage mode");
    return __float2half_rn(__fmul_rn((float)a, __half2float(x)));
  } else {
    return from_dbl<T>(__dmul_rn(a, to_dbl(x)));
  }
}

template <class T, bool F32 = false>
struct ScaleSrc {  // v = round(inv * w) (scale_rn)
  const T* __restrict__ w;
  double inv;
  __device__ __forceinline__ T f(T x) const { return scale_rn<T, F32>(inv, x); }
  template <int VEC>
  __device__ __forceinline__ void vec(int64_t e0, T (&v)[VEC]) const {
    ld_vec<T, VEC>(w, e0, v);
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = f(v[i]);
  }
  __device__ __forceinline__ T at(int64_t e) const { return f(w[e]); }
};

// Sign/finiteness summary of one stored coefficient, for the residual from
// x = 0: bit 0 = the sign bit is set (coef * +0 = -0), bit 1 = not finite
// (coef * 0 = NaN). See zero_resid (gadi_kernels.cuh).
template <class V>
__device__ __forceinline__ int zflag(V c) {
  const double d = to_dbl(c);
  return (signbit(d) ? 1 : 0) | (isfinite(d) ? 0 : 2);
}

// 3D convection-diffusion 7-point operator, matrix free (problems.cpp:8-43):
// row i*n^2 + j*n + k; c[] = {i-1, j-1, k-1, centre, k+1, j+1, i+1}, the
// stored-column order. Boundary neighbours are absent (not zero-valued), as
// in the reference CSR.
template <class V>
struct Stencil7 {
  using value_type = V;
  int64_t n, nn, N;
  V c[7];
  int lg;  // log2(n) when n is a power of two (always on the aligned path), else -1
  uint8_t zc[7];  // zflag of each coefficient (set by the engine; see zflags)
  int64_t i_off;  // first plane of a z-slab (sharded solves): local row e is global row e + i_off*n^2

  // Fold for the VEC consecutive elements e0..e0+VEC-1 of one grid row
  // (aligned path: e0 % VEC == 0 and n % VEC == 0; VEC == 1 is any element).
  // `cc` returns the operand at the VEC centre points.
  template <int VEC, class Src, class X, class Acc, class F>
  __device__ __forceinline__ void fold(const Src& x, int64_t e0, Acc (&acc)[VEC], F f, X (&cc)[VEC]) const {
    int64_t k0, j, i;
    if (lg >= 0) {  // shifts, not 64-bit division, on the hot path
      k0 = e0 & (n - 1);
      j = (e0 >> lg) & (n - 1);
      i = (e0 >> (2 * lg)) + i_off;
    } else {
      k0 = e0 % n;
      const int64_t r = e0 / n;
      j = r % n;
      i = r / n + i_off;
    }
    X nb[VEC];
    x.template vec<VEC>(e0, cc);
    if (i > 0) {
      x.template vec<VEC>(e0 - nn, nb);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = f(acc[v], c[0], nb[v]);
    }
    if (j > 0) {
      x.template vec<VEC>(e0 - n, nb);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = f(acc[v], c[1], nb[v]);
    }
    {
      const bool has0 = k0 > 0;
      X km0 = has0 ? x.at(e0 - 1) : cc[0];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        if (v > 0) acc[v] = f(acc[v], c[2], cc[v - 1]);
        else if (has0) acc[v] = f(acc[v], c[2], km0);
      }
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = f(acc[v], c[3], cc[v]);
    {
      const bool hasL = k0 + VEC < n;
      X kpL = hasL ? x.at(e0 + VEC) : cc[0];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        if (v < VEC - 1) acc[v] = f(acc[v], c[4], cc[v + 1]);
        else if (hasL) acc[v] = f(acc[v], c[4], kpL);
      }
    }
    if (j + 1 < n) {
      x.template vec<VEC>(e0 + n, nb);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = f(acc[v], c[5], nb[v]);
    }
    if (i + 1 < n) {
      x.template vec<VEC>(e0 + nn, nb);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = f(acc[v], c[6], nb[v]);
    }
  }

  // OR of zflag over the row's stored coefficients (the ones fold visits).
  __device__ __forceinline__ int zflags(int64_t e) const {
    int64_t k, j, i;
    if (lg >= 0) {
      k = e & (n - 1);
      j = (e >> lg) & (n - 1);
      i = (e >> (2 * lg)) + i_off;
    } else {
      k = e % n;
      const int64_t r = e / n;
      j = r % n;
      i = r / n + i_off;
    }
    int f = zc[3];
    if (i > 0) f |= zc[0];
    if (j > 0) f |= zc[1];
    if (k > 0) f |= zc[2];
    if (k + 1 < n) f |= zc[4];
    if (j + 1 < n) f |= zc[5];
    if (i + 1 < n) f |= zc[6];
    return f;
  }
  // the same for the VEC points e0.. of one grid row (aligned path)
  template <int VEC>
  __device__ __forceinline__ void zflags_vec(int64_t e0, int (&f)[VEC]) const {
    int64_t k0, j, i;
    if (lg >= 0) {
      k0 = e0 & (n - 1);
      j = (e0 >> lg) & (n - 1);
      i = (e0 >> (2 * lg)) + i_off;
    } else {
      k0 = e0 % n;
      const int64_t r = e0 / n;
      j = r % n;
      i = r / n + i_off;
    }
    int b = zc[3];
    if (i > 0) b |= zc[0];
    if (j > 0) b |= zc[1];
    if (j + 1 < n) b |= zc[5];
    if (i + 1 < n) b |= zc[6];
    const int mid = b | zc[2] | zc[4];
#pragma unroll
    for (int v = 0; v < VEC; ++v) f[v] = mid;
    f[0] = b | (k0 > 0 ? zc[2] : 0) | (VEC > 1 || k0 + 1 < n ? zc[4] : 0);
    if (VEC > 1) f[VEC - 1] = b | zc[2] | (k0 + VEC < n ? zc[4] : 0);
  }
};

// General sparse operator in CSR with int64 row pointers and int32 column
// indices (the reference's int64 layout, sparse.hpp:17-65, narrowed because
// N < 2^31). H and S share one pattern (the union pattern of A and A^T,
// sparse.cpp:166-178) and differ only in values.
template <class V>
struct Csr {
  using value_type = V;
  int64_t N;
  const int64_t* __restrict__ rp;
  const int32_t* __restrict__ ci;
  const V* __restrict__ val;

  template <int VEC, class Src, class X, class Acc, class F>
  __device__ __forceinline__ void fold(const Src& x, int64_t e0, Acc (&acc)[VEC], F f, X (&cc)[VEC]) const {
    x.template vec<VEC>(e0, cc);
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      const int64_t row = e0 + v;
      const int64_t b = rp[row], e = rp[row + 1];
      Acc a = acc[v];
      for (int64_t k = b; k < e; ++k) a = f(a, val[k], x.at(ci[k]));
      acc[v] = a;
    }
  }
};

}  // namespace gadi
