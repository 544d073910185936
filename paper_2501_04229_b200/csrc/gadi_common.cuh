// gadi_common.cuh — precision traits and deterministic pairwise reductions.
//
// Arithmetic model (reference: precision.hpp:54-102, kernels.cpp:26-54):
// every scalar op is rounded once to its format. On the device this is the
// native IEEE op with round-to-nearest and NO contraction (__fadd_rn,
// __hmul_rn, ... ; the library is also built with -fmad=false), so a binary32
// or binary16 kernel reproduces the reference's emulated arithmetic bit for
// bit. Conversions binary64 -> binary16 use cvt.rn.f16.f64 (one rounding,
// as round_to_half does; a double->float->half path would double round).
//
// Pairwise sums (kernels.cpp:33-39) are reproduced exactly: the halving tree
// over N terms is cut at a depth D whose 2^D nodes ("segments") each hold
// VEC contiguous terms (N = VEC * 2^D, the aligned path) or 2..4 terms (any
// N, the general path); one thread owns one segment, and above depth D the
// tree is a perfect binary tree that a warp butterfly, a shared-memory tree
// and a last-block pass over per-block partials evaluate in exactly that
// shape. IEEE addition commutes, so only the tree shape matters. The result
// is bitwise equal to the reference's recursion and independent of timing.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

namespace gadi {

// ---------------------------------------------------------------- formats
enum Prec : int { P_HALF = 0, P_SINGLE = 1, P_DOUBLE = 2 };

template <class C>
struct Ar;

template <>
struct Ar<double> {
  static constexpr int prec = P_DOUBLE;
  __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static double sub(double a, double b) { return __dsub_rn(a, b); }
  __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ __forceinline__ static double from_d(double x) { return x; }
  __device__ __forceinline__ static double to_d(double x) { return x; }
  __device__ __forceinline__ static double neg(double x) { return -x; }
  __device__ __forceinline__ static double zero() { return 0.0; }
};

template <>
struct Ar<float> {
  static constexpr int prec = P_SINGLE;
  __device__ __forceinline__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ __forceinline__ static float sub(float a, float b) { return __fsub_rn(a, b); }
  __device__ __forceinline__ static float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ __forceinline__ static float from_d(double x) { return __double2float_rn(x); }
  __device__ __forceinline__ static double to_d(float x) { return (double)x; }
  __device__ __forceinline__ static float neg(float x) { return -x; }
  __device__ __forceinline__ static float zero() { return 0.0f; }
};

template <>
struct Ar<__half> {
  static constexpr int prec = P_HALF;
  __device__ __forceinline__ static __half add(__half a, __half b) { return __hadd_rn(a, b); }
  __device__ __forceinline__ static __half sub(__half a, __half b) { return __hsub_rn(a, b); }
  __device__ __forceinline__ static __half mul(__half a, __half b) { return __hmul_rn(a, b); }
  __device__ __forceinline__ static __half from_d(double x) { return __double2half(x); }
  __device__ __forceinline__ static double to_d(__half x) { return (double)__half2float(x); }
  __device__ __forceinline__ static __half neg(__half x) { return __hneg(x); }
  __device__ __forceinline__ static __half zero() { return __ushort_as_half((unsigned short)0); }
};

// round_to(x, P) on binary64-carried values (precision.hpp:81-87).
template <int P>
__device__ __forceinline__ double round_p(double x) {
  if constexpr (P == P_DOUBLE) return x;
  else if constexpr (P == P_SINGLE) return (double)__double2float_rn(x);
  else return (double)__half2float(__double2half(x));
}

// Correctly rounded division / sqrt in C: computed in binary64, rounded once
// (rounded_binop, precision.cpp:91-97; 53 >= 2p+2 makes it exact).
// For binary32 the native correctly rounded division is the same value; for
// binary16 a binary32 quotient rounded once to binary16 is too (24 >= 2*11+2).
template <class C>
__device__ __forceinline__ C div_c(C a, C b) {
  if constexpr (std::is_same<C, float>::value) return __fdiv_rn(a, b);
  else if constexpr (std::is_same<C, __half>::value)
    return __float2half_rn(__fdiv_rn(__half2float(a), __half2float(b)));
  else return __ddiv_rn(a, b);
}

// x * 2^e exactly as ldexp/scalbn (solver.cpp:89,165): a multiply by the exact
// power of two is the same correctly rounded value while 2^e is a normal double.
__device__ __forceinline__ double pow2d(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }
__device__ __forceinline__ double ldexp_fast(double x, int e, double p2) {
  return (e >= -1000 && e <= 1000) ? __dmul_rn(x, p2) : scalbn(x, e);
}

// Storage <-> compute conversions (exact widening; one RN narrowing).
template <class T, class C>
__device__ __forceinline__ C ld_c(T v) {
  if constexpr (std::is_same<T, C>::value) return v;
  else if constexpr (std::is_same<T, __half>::value && std::is_same<C, float>::value) return __half2float(v);
  else return Ar<C>::from_d((double)v);
}
template <class T, class C>
__device__ __forceinline__ T st_t(C v) {
  if constexpr (std::is_same<T, C>::value) return v;
  else if constexpr (std::is_same<T, __half>::value && std::is_same<C, float>::value) return __float2half_rn(v);
  else return (T)Ar<C>::to_d(v);
}
template <class T>
__device__ __forceinline__ double to_dbl(T v) {
  if constexpr (std::is_same<T, __half>::value) return (double)__half2float(v);
  else return (double)v;
}
template <class T>
__device__ __forceinline__ T from_dbl(double v) {
  if constexpr (std::is_same<T, __half>::value) return __double2half(v);
  else if constexpr (std::is_same<T, float>::value) return __double2float_rn(v);
  else return v;
}
template <class T>
__device__ __forceinline__ bool finite_t(T v) {
  return isfinite(to_dbl(v));
}

// ------------------------------------------------------------ vector I/O
// VEC contiguous elements starting at an index that is a multiple of VEC;
// VEC * sizeof(T) == 16 on the aligned path (one 128-bit access).
template <class T, int VEC>
__device__ __forceinline__ void ld_vec(const T* __restrict__ p, int64_t e0, T (&v)[VEC]) {
  if constexpr (VEC * sizeof(T) > 16 && VEC * sizeof(T) % 16 == 0) {  // several 128-bit accesses
    constexpr int per = 16 / sizeof(T);
#pragma unroll
    for (int b = 0; b < VEC / per; ++b) {
      uint4 u = __ldg(reinterpret_cast<const uint4*>(p + e0) + b);
      const T* t = reinterpret_cast<const T*>(&u);
#pragma unroll
      for (int i = 0; i < per; ++i) v[b * per + i] = t[i];
    }
  } else if constexpr (VEC * sizeof(T) == 16) {
    uint4 u = __ldg(reinterpret_cast<const uint4*>(p + e0));
    const T* t = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = t[i];
  } else if constexpr (VEC * sizeof(T) == 8) {
    uint2 u = __ldg(reinterpret_cast<const uint2*>(p + e0));
    const T* t = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = t[i];
  } else if constexpr (VEC * sizeof(T) == 4) {
    unsigned u = __ldg(reinterpret_cast<const unsigned*>(p + e0));
    const T* t = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = t[i];
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = p[e0 + i];
  }
}
template <class T, int VEC>
__device__ __forceinline__ void st_vec(T* __restrict__ p, int64_t e0, const T (&v)[VEC]) {
  if constexpr (VEC * sizeof(T) > 16 && VEC * sizeof(T) % 16 == 0) {
    constexpr int per = 16 / sizeof(T);
#pragma unroll
    for (int b = 0; b < VEC / per; ++b) {
      uint4 u;
      T* t = reinterpret_cast<T*>(&u);
#pragma unroll
      for (int i = 0; i < per; ++i) t[i] = v[b * per + i];
      reinterpret_cast<uint4*>(p + e0)[b] = u;
    }
  } else if constexpr (VEC * sizeof(T) == 16) {
    uint4 u;
    T* t = reinterpret_cast<T*>(&u);
#pragma unroll
    for (int i = 0; i < VEC; ++i) t[i] = v[i];
    *reinterpret_cast<uint4*>(p + e0) = u;
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) p[e0 + i] = v[i];
  }
}

// -------------------------------------------------------------- segments
// Layout of N terms into 2^D segments. Aligned: N = VEC * 2^D, segment t =
// [t*VEC, t*VEC+VEC). General (VEC == 1 template): D = max(0, floor(log2 N)-1),
// segment t found by descending the halving tree (lengths 1..4).
struct Seg {
  int64_t lo;
  int len;
};

template <int VEC>
__device__ __forceinline__ Seg seg_of(int64_t t, int64_t N, int D) {
  if constexpr (VEC > 1) {
    return Seg{t * VEC, VEC};
  } else {
    int64_t lo = 0, len = N;
    for (int l = D - 1; l >= 0; --l) {
      const int64_t h = len / 2;
      if ((t >> l) & 1) {
        lo += h;
        len -= h;
      } else {
        len = h;
      }
    }
    return Seg{lo, (int)len};
  }
}

// Pairwise sum of one segment's terms (halving recursion, kernels.cpp:33-39).
// GMAX = max segment length in registers: VEC on the aligned path, 4 otherwise.
template <class C, int GMAX>
__device__ __forceinline__ C seg_sum(const C (&t)[GMAX], int len) {
  using A = Ar<C>;
  if constexpr (GMAX == 1) {
    return t[0];
  } else if constexpr (GMAX == 4) {
    // general path: len in 1..4
    if (len == 1) return t[0];
    if (len == 2) return A::add(t[0], t[1]);
    if (len == 3) return A::add(t[0], A::add(t[1], t[2]));
    return A::add(A::add(t[0], t[1]), A::add(t[2], t[3]));
  } else {
    // aligned: power-of-two GMAX, perfect tree over adjacent pairs
    C w[GMAX];
#pragma unroll
    for (int i = 0; i < GMAX; ++i) w[i] = t[i];
#pragma unroll
    for (int s = 1; s < GMAX; s <<= 1)
#pragma unroll
      for (int i = 0; i < GMAX; i += 2 * s) w[i] = A::add(w[i], w[i + s]);
    return w[0];
  }
}

// ------------------------------------------------------ warp/block trees
template <class C>
__device__ __forceinline__ C shfl_xor_c(C v, int o, unsigned mask) {
  return __shfl_xor_sync(mask, v, o);
}
template <>
__device__ __forceinline__ __half shfl_xor_c<__half>(__half v, int o, unsigned mask) {
  unsigned short u = __half_as_ushort(v);
  u = (unsigned short)__shfl_xor_sync(mask, (unsigned)u, o);
  return __ushort_as_half(u);
}

// Perfect pairwise tree over `width` consecutive lanes (width power of 2 <= 32);
// every participating lane ends with the total.
template <class C>
__device__ __forceinline__ C warp_tree(C v, int width) {
  if (width >= 32) {  // the usual case: five unconditional levels (one uniform branch, not five)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) v = Ar<C>::add(v, shfl_xor_c(v, o, 0xffffffffu));
    return v;
  }
  const unsigned mask = (1u << width) - 1u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
    if (o < width) v = Ar<C>::add(v, shfl_xor_c(v, o, mask));
  return v;
}

// Perfect pairwise tree over the first `count` threads of the block (count a
// power of 2, <= blockDim.x <= 1024). Result valid in thread 0. All threads
// of the block must call it. `sm` must hold 32 C values.
template <class C>
__device__ __forceinline__ C block_tree(C v, int count, C* sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (count <= 32) {
    if (tid < count) v = warp_tree(v, count);
    return v;
  }
  v = warp_tree(v, 32);
  const int nw = count >> 5;
  __syncthreads();
  if (lane == 0 && warp < nw) sm[warp] = v;
  __syncthreads();
  if (warp == 0) {
    C w = lane < nw ? sm[lane] : Ar<C>::zero();
    if (lane < nw) w = warp_tree(w, nw);
    v = w;
  }
  return v;
}

// Exact pairwise sum of L (power of 2) contiguous values. The loads go out
// in batches of up to 16 (all in flight at once: the values are L2-resident
// partials, and a load-add-load chain would cost one L2 latency per value);
// each batch is a perfect subtree, and a binary-counter stack merges the
// batch sums as equal-size subtrees close, so the shape is the pairwise tree.
template <class C, class Load>
__device__ __forceinline__ C run_pairwise(int64_t L, Load load) {
  constexpr int B = 16;
  if (L < B) {
    C v[B];
#pragma unroll
    for (int k = 0; k < B; ++k)
      if (k < L) v[k] = load(k);
#pragma unroll
    for (int st = 1; st < B; st <<= 1)
#pragma unroll
      for (int k = 0; k + st < B; k += 2 * st)
        if (k + st < L) v[k] = Ar<C>::add(v[k], v[k + st]);
    return v[0];
  }
  C stk[40];
  int sp = 0;
  for (int64_t j = 0; j < L; j += B) {
    C v[B];
#pragma unroll
    for (int k = 0; k < B; ++k) v[k] = load(j + k);
#pragma unroll
    for (int st = 1; st < B; st <<= 1)
#pragma unroll
      for (int k = 0; k + st < B; k += 2 * st) v[k] = Ar<C>::add(v[k], v[k + st]);
    stk[sp++] = v[0];
    for (int64_t q = j / B + 1; (q & 1) == 0; q >>= 1) {
      stk[sp - 2] = Ar<C>::add(stk[sp - 2], stk[sp - 1]);
      --sp;
    }
  }
  return stk[0];
}

// Max of |v| for non-negative doubles through their bit patterns (order
// preserving); NaN never enters (std::max(m, NaN) keeps m, kernels.cpp:196).
__device__ __forceinline__ void atomic_max_abs(unsigned long long* dst, double a) {
  if (!(a == a)) return;
  atomicMax(dst, (unsigned long long)__double_as_longlong(fabs(a)));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace gadi
