// gadi_ops.cuh — the operators A, H = alpha I + M, S = alpha I + N on the device.
//
// A fold visits a row's stored entries in ascending column order, exactly as
// the reference's per-row loops (kernels.cpp:41-54 matvec, :56-69 residual)
// visit the CSR it builds; the caller's functor f(acc, coef, x) supplies the
// per-entry rounding (matvec: acc + coef*x; residual: acc - coef*x).
#pragma once

#include "gadi_common.cuh"

namespace gadi {

// 3D convection-diffusion 7-point operator, matrix free (problems.cpp:8-43):
// row i*n^2 + j*n + k; c[] = {i-1, j-1, k-1, centre, k+1, j+1, i+1}, the
// stored-column order. Boundary neighbours are absent (not zero-valued), as
// in the reference CSR.
template <class V>
struct Stencil7 {
  int64_t n, nn, N;
  V c[7];

  // Fold for the VEC consecutive elements e0..e0+VEC-1 of one grid row
  // (aligned path: e0 % VEC == 0 and n % VEC == 0; VEC == 1 is any element).
  template <int VEC, class X, class Acc, class F>
  __device__ __forceinline__ void fold(const X* __restrict__ x, int64_t e0, Acc (&acc)[VEC], F f) const {
    const int64_t k0 = e0 % n;
    const int64_t r = e0 / n;
    const int64_t j = r % n;
    const int64_t i = r / n;
    X cc[VEC], nb[VEC];
    ld_vec<X, VEC>(x, e0, cc);
    if (i > 0) {
      ld_vec<X, VEC>(x, e0 - nn, nb);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = f(acc[v], c[0], nb[v]);
    }
    if (j > 0) {
      ld_vec<X, VEC>(x, e0 - n, nb);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = f(acc[v], c[1], nb[v]);
    }
    {
      const bool has0 = k0 > 0;
      X km0 = has0 ? x[e0 - 1] : cc[0];
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
      X kpL = hasL ? x[e0 + VEC] : cc[0];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        if (v < VEC - 1) acc[v] = f(acc[v], c[4], cc[v + 1]);
        else if (hasL) acc[v] = f(acc[v], c[4], kpL);
      }
    }
    if (j + 1 < n) {
      ld_vec<X, VEC>(x, e0 + n, nb);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = f(acc[v], c[5], nb[v]);
    }
    if (i + 1 < n) {
      ld_vec<X, VEC>(x, e0 + nn, nb);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = f(acc[v], c[6], nb[v]);
    }
  }
};

// General sparse operator in CSR with int64 row pointers and int32 column
// indices (the reference's int64 layout, sparse.hpp:17-65, narrowed because
// N < 2^31). H and S share one pattern (the union pattern of A and A^T,
// sparse.cpp:166-178) and differ only in values.
template <class V>
struct Csr {
  int64_t N;
  const int64_t* __restrict__ rp;
  const int32_t* __restrict__ ci;
  const V* __restrict__ val;

  template <int VEC, class X, class Acc, class F>
  __device__ __forceinline__ void fold(const X* __restrict__ x, int64_t e0, Acc (&acc)[VEC], F f) const {
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      const int64_t row = e0 + v;
      const int64_t b = rp[row], e = rp[row + 1];
      Acc a = acc[v];
      for (int64_t k = b; k < e; ++k) a = f(a, val[k], x[ci[k]]);
      acc[v] = a;
    }
  }
};

}  // namespace gadi
