// gadi_st25.cuh — 2.5D plane-marching 7-point stencil kernels with TMA staging.
//
// One CTA owns a tile of TJ grid rows (j0 .. j0+TJ-1, all n points of each
// row) over IL consecutive planes i (ib .. ib+IL-1) and marches along i, the
// slowest index (row = i*n^2 + j*n + k, problems.cpp:14). The raw inputs of
// each plane (TJ+2 rows including the j-halo: one contiguous range of
// global memory) arrive by one 1-D bulk TMA copy per input
// (cp.async.bulk ... mbarrier::complete_tx) into an S-stage shared-memory
// ring, so each input element is read from HBM once and the copies run
// ahead of the math. The operand of the operator (p = r + beta p for CG,
// v = w / h for an Arnoldi step, x as is for residuals) is formed ONCE per
// point into a 3-plane shared-memory ring (planes i-1, i, i+1), and the fold
// reads all seven neighbours from there in the reference's stored-column
// order (problems.cpp:28-34, kernels.cpp:47-52 / 63-66), so the arithmetic is
// bit-identical to the generic kernels.
//
// Reductions: a CTA's chunk of one plane (TJ rows = TJ*n contiguous
// entries) is one perfect pairwise subtree (lanes -> warps -> CTA); its sum
// goes to partials[plane * (n/TJ) + tile], which are contiguous aligned
// blocks in global order, and the last CTA folds them pairwise. The result
// is the reference's pairwise sum bit for bit (see gadi_common.cuh).
#pragma once

#include "gadi_kernels.cuh"

namespace gadi {

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <class T, int VEC>
__device__ __forceinline__ void lds16(const T* p, T (&v)[VEC]) {
  static_assert(VEC * sizeof(T) == 16, "16-byte chunks");
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const T* t = reinterpret_cast<const T*>(&u);
#pragma unroll
  for (int i = 0; i < VEC; ++i) v[i] = t[i];
}
template <class T, int VEC>
__device__ __forceinline__ void sts16(T* p, const T (&v)[VEC]) {
  uint4 u;
  T* t = reinterpret_cast<T*>(&u);
#pragma unroll
  for (int i = 0; i < VEC; ++i) t[i] = v[i];
  *reinterpret_cast<uint4*>(p) = u;
}

// VEC values of R from / to shared memory in 16-byte pieces.
template <class R, int VEC>
__device__ __forceinline__ void lds_vec(const R* p, R (&v)[VEC]) {
  constexpr int per = 16 / sizeof(R);
  static_assert(VEC % per == 0, "whole 16-byte pieces");
#pragma unroll
  for (int b = 0; b < VEC / per; ++b) {
    const uint4 u = *reinterpret_cast<const uint4*>(p + b * per);
    const R* t = reinterpret_cast<const R*>(&u);
#pragma unroll
    for (int i = 0; i < per; ++i) v[b * per + i] = t[i];
  }
}
template <class R, int VEC>
__device__ __forceinline__ void sts_vec(R* p, const R (&v)[VEC]) {
  constexpr int per = 16 / sizeof(R);
#pragma unroll
  for (int b = 0; b < VEC / per; ++b) {
    uint4 u;
    R* t = reinterpret_cast<R*>(&u);
#pragma unroll
    for (int i = 0; i < per; ++i) t[i] = v[b * per + i];
    *reinterpret_cast<uint4*>(p + b * per) = u;
  }
}

// acc[v] = f(acc[v], coef, x[v]) for all v, except v = 0 / v = VEC-1 when the
// neighbour is absent (skip0 / skipL). binary32 matvec / residual folds pair
// the products (FMUL2: one RN rounding per lane, the same values as scalar
// __fmul_rn) and keep the adds scalar (see MatvecF::PACKED).
template <class F, class A, class X, int VEC>
__device__ __forceinline__ void fold_vec(const F& f, A (&acc)[VEC], A coef, const X (&x)[VEC], bool skip0,
                                         bool skipL) {
  const A a0 = acc[0], aL = acc[VEC - 1];
  if constexpr (std::is_same<A, float>::value && (VEC % 2 == 0) && F::PACKED) {
    const float2 c2 = make_float2(coef, coef);
#pragma unroll
    for (int v = 0; v < VEC; v += 2) {
      const float2 pr = __fmul2_rn(c2, make_float2(ld_c<X, float>(x[v]), ld_c<X, float>(x[v + 1])));
      acc[v] = F::NEG ? __fsub_rn(acc[v], pr.x) : __fadd_rn(acc[v], pr.x);
      acc[v + 1] = F::NEG ? __fsub_rn(acc[v + 1], pr.y) : __fadd_rn(acc[v + 1], pr.y);
    }
  } else {
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = f(acc[v], coef, x[v]);
  }
  if (skip0) acc[0] = a0;
  if (skipL) acc[VEC - 1] = aL;
}

// out[v] = a * x[v] rounded in C; binary32 pairs the products (FMUL2).
template <class C, class X, int VEC>
__device__ __forceinline__ void mul_vec(C a, const X (&x)[VEC], C (&out)[VEC]) {
  if constexpr (std::is_same<C, float>::value && VEC % 2 == 0) {
    const float2 a2 = make_float2(a, a);
#pragma unroll
    for (int v = 0; v < VEC; v += 2) {
      const float2 pr = __fmul2_rn(a2, make_float2(ld_c<X, float>(x[v]), ld_c<X, float>(x[v + 1])));
      out[v] = pr.x;
      out[v + 1] = pr.y;
    }
  } else {
#pragma unroll
    for (int v = 0; v < VEC; ++v) out[v] = Ar<C>::mul(a, ld_c<X, C>(x[v]));
  }
}

// ---------------------------------------------- binary16 lanes, packed
// The binary16-storage / binary32-arithmetic operator passes keep 8 values
// per 16-byte chunk as 4 packed 32-bit registers and never unpack them:
// FHFMA / FHADD (sm_100) read either half of a register directly. Every
// product on these paths multiplies two binary16 values, exact in binary32,
// so a fused op rounds exactly once where the reference rounds the sum (see
// fhfma in gadi_kernels.cuh): the bits are the reference's.
// a.half(S) + c in binary32, one rounding (FHADD)
template <int S>
__device__ __forceinline__ float fhadd(uint32_t a, float c) {
  float d;
  if constexpr (S == 0)
    asm("{.reg .f16 al, ah; mov.b32 {al, ah}, %1; add.rn.f32.f16 %0, al, %2;}" : "=f"(d) : "r"(a), "f"(c));
  else
    asm("{.reg .f16 al, ah; mov.b32 {al, ah}, %1; add.rn.f32.f16 %0, ah, %2;}" : "=f"(d) : "r"(a), "f"(c));
  return d;
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {  // two RN roundings (F2FP)
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t u4_at(const uint4& u, int k) {
  return k == 0 ? u.x : k == 1 ? u.y : k == 2 ? u.z : u.w;
}
__device__ __forceinline__ uint4 lds_u4(const void* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ void sts_u4(void* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

// acc[e] += c * x[e + SH] over one chunk, c in the low half of `c`;
// SH = -1 / +1 take the k-1 / k+1 neighbours: x[-1] = edge (its low half),
// x[8] = edge. A missing edge neighbour passes the coefficient's neutral
// operand (nh_of), whose product is -0: acc + -0 == acc for every acc.
template <int SH>
__device__ __forceinline__ void fold8h(float (&a)[8], uint32_t c, const uint4& x, uint32_t edge) {
  const uint32_t r[4] = {x.x, x.y, x.z, x.w};
  if constexpr (SH == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[2 * k] = fhf<0, 0>(c, r[k], a[2 * k]);
      a[2 * k + 1] = fhf<0, 1>(c, r[k], a[2 * k + 1]);
    }
  } else if constexpr (SH < 0) {
    a[0] = fhf<0, 0>(c, edge, a[0]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[2 * k + 1] = fhf<0, 0>(c, r[k], a[2 * k + 1]);
      if (k < 3) a[2 * k + 2] = fhf<0, 1>(c, r[k], a[2 * k + 2]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[2 * k] = fhf<0, 1>(c, r[k], a[2 * k]);
      if (k < 3) a[2 * k + 1] = fhf<0, 0>(c, r[k + 1], a[2 * k + 1]);
    }
    a[7] = fhf<0, 0>(c, edge, a[7]);
  }
}
// the operand whose product with coefficient c is -0 (sign(c) XOR sign(-0))
__device__ __forceinline__ uint32_t nh_of(uint32_t c) { return (c & 0x8000u) ^ 0x8000u; }
// pairwise sum of the 8 exact products a[e] * b[e] (kernels.cpp:33-39): each
// first-level node RN(a0 b0 + a1 b1) is one FHFMA onto the exact product
// a1 b1 (an FHFMA onto -0, which returns it unchanged)
__device__ __forceinline__ float dot8h(const uint4& a, const uint4& b) {
  const uint32_t x[4] = {a.x, a.y, a.z, a.w}, y[4] = {b.x, b.y, b.z, b.w};
  float s[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) s[k] = fhf<0, 0>(x[k], y[k], fhf<1, 1>(x[k], y[k], -0.0f));
  return __fadd_rn(__fadd_rn(s[0], s[1]), __fadd_rn(s[2], s[3]));
}

struct St25Geo {
  int n, lg;      // points per direction (power of two), log2 n
  int TJ, lgTJ;   // rows per tile
  int IL;         // planes per CTA
  int TR, lgTR;   // 16-byte chunks per row
  int CPT;        // chunks per thread per plane (power of two)
  int njt;        // tiles per plane = n / TJ
  int i0, i1;     // the planes this device owns (a z-slab of a sharded solve; 0, n on one device)
  int nblk;       // CTAs = njt * (i1 - i0) / IL
  int threads;
  int stages;
  int64_t nn;
  size_t smem;    // dynamic shared memory bytes
};

constexpr int ST25_CPT_MAX = 4;
constexpr int ST25_IL_MAX = 32;  // planes per CTA (make_st25)
constexpr int ST25_MAXW = 16;    // warps per CTA

// The pairwise trees of CPT per-lane values v[rr] over the 32 lanes (lane
// levels xor 1, 2, ..., 16, as warp_tree), then over rr ((v0+v1)+(v2+v3)),
// with the total in lane 0. The first log2(CPT) lane levels run as a
// reduce-scatter (each lane keeps half of the trees and receives its
// partner's half), so the CPT trees cost 2*CPT-2+5-log2(CPT) shuffles instead
// of 5*CPT. Same pairs at every level, so bitwise equal to CPT warp_trees.
template <int CPT, class C>
__device__ __forceinline__ C warp_tree_cpt(C (&v)[CPT]) {
  const int lane = threadIdx.x & 31;
  C w[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) w[k] = v[k];
  int o = 1;
#pragma unroll
  for (int m = CPT; m > 1; m >>= 1, o <<= 1) {  // keep trees [0,m/2) (bit clear) or [m/2,m) (bit set)
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < m / 2; ++k) {
      const C send = hi ? w[k] : w[k + m / 2];
      const C keep = hi ? w[k + m / 2] : w[k];
      w[k] = Ar<C>::add(keep, shfl_xor_c(send, o, 0xffffffffu));
    }
  }
  // this lane holds tree rr = sum_b bit_b(lane) * CPT / 2^(b+1) over levels 1..o
  C t = w[0];
#pragma unroll
  for (int oo = o; oo < 32; oo <<= 1) t = Ar<C>::add(t, shfl_xor_c(t, oo, 0xffffffffu));
  // tree over rr: its lowest level pairs rr differing in the last split bit
#pragma unroll
  for (int oo = o >> 1; oo >= 1; oo >>= 1) t = Ar<C>::add(t, shfl_xor_c(t, oo, 0xffffffffu));
  return t;
}

// After a tile's plane loop: each plane's warp partials -> one pairwise
// subtree per (plane, tile) -> partials[plane * njt + tile].
template <class P, class PL>
__device__ __forceinline__ void st25_partials(const St25Geo& g, const Red& rd, const PL* plb, int nw, int ib,
                                              int jt, const PL* plb1 = nullptr) {
  if (!plb1) plb1 = plb;  // one reduced quantity: R1 shares the buffer
  using R0 = typename P::R0;
  if (P::HAS_R0 || P::HAS_R1) {
    __syncthreads();
    for (int t = threadIdx.x; t < g.IL; t += blockDim.x) {
      R0 v0[ST25_MAXW];
      double v1[ST25_MAXW];
#pragma unroll
      for (int k = 0; k < ST25_MAXW; ++k)
        if (k < nw) {
          if (P::HAS_R0) v0[k] = from_dbl<R0>(plb[t * nw + k]);
          if (P::HAS_R1) v1[k] = plb1[t * nw + k];
        }
#pragma unroll
      for (int s2 = 1; s2 < ST25_MAXW; s2 <<= 1)
#pragma unroll
        for (int k = 0; k + s2 < ST25_MAXW; k += 2 * s2)
          if (k + s2 < nw) {
            if (P::HAS_R0) v0[k] = Ar<R0>::add(v0[k], v0[k + s2]);
            if (P::HAS_R1) v1[k] = __dadd_rn(v1[k], v1[k + s2]);
          }
      const int64_t slot = (int64_t)(ib - g.i0 + t) * g.njt + jt;
      if (P::HAS_R0) rd.part0[slot] = to_dbl(v0[0]);
      if (P::HAS_R1) rd.part1[slot] = v1[0];
    }
  }
}

// After all of a CTA's tiles: max / flags, then the grid ticket over the
// `nctas` CTAs; the last CTA folds the partials.
template <class P>
__device__ __forceinline__ void st25_ticket(const P& pol, const St25Geo& g, const Red& rd, DevState* st,
                                            double mloc, int flag, unsigned nctas) {
  using R0 = typename P::R0;
  __shared__ __align__(8) unsigned char redb0[32 * sizeof(double)];
  __shared__ double redb1[32];
  __shared__ int s_last;
  R0* red0 = reinterpret_cast<R0*>(redb0);
  const int tid = threadIdx.x;
  // the partials were written by threads t < IL <= 32 (st25_partials), all in warp 0 with the ticket thread
  if ((P::HAS_R0 || P::HAS_R1) && tid < ST25_IL_MAX) __threadfence();
  if (P::HAS_MAX) block_max_abs(&st->maxbits, mloc);
  if (P::HAS_FLAG) or_flags(pol.flag_dst(st), flag);
  // every warp's max / flag atomics precede this CTA's ticket (the last CTA reads them)
  if (P::HAS_MAX || P::HAS_FLAG) __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned t = atomicAdd(rd.ticket, 1u);
    s_last = (t == nctas - 1u);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int64_t P_ = (int64_t)(g.i1 - g.i0) * g.njt;  // partials (power of two)
  const int B = blockDim.x;
  R0 t0 = Ar<R0>::zero();
  double t1 = 0.0;
  int cnt;
  if (P_ <= B) {
    if (P::HAS_R0) t0 = tid < P_ ? from_dbl<R0>(__ldcg(rd.part0 + tid)) : Ar<R0>::zero();
    if (P::HAS_R1) t1 = tid < P_ ? __ldcg(rd.part1 + tid) : 0.0;
    cnt = (int)P_;
  } else {
    const int64_t Lr = P_ / B;
    const double* p0 = rd.part0 + (int64_t)tid * Lr;
    const double* p1 = rd.part1 + (int64_t)tid * Lr;
    if (P::HAS_R0) t0 = run_pairwise<R0>(Lr, [&](int64_t j) { return from_dbl<R0>(__ldcg(p0 + j)); });
    if (P::HAS_R1) t1 = run_pairwise<double>(Lr, [&](int64_t j) { return __ldcg(p1 + j); });
    cnt = B;
  }
  if (P::HAS_R0) t0 = block_tree(t0, cnt, red0);
  if (P::HAS_R1) t1 = block_tree(t1, cnt, redb1);
  if (tid == 0) {
    *rd.ticket = 0u;
    __threadfence();
    finish_red(pol, st, t0, t1);
  }
}

template <class P, class PL>
__device__ __forceinline__ void st25_finish(const P& pol, const St25Geo& g, const Red& rd, DevState* st,
                                            const PL* plb, int nw, int ib, int jt, double mloc, int flag,
                                            const PL* plb1 = nullptr) {
  st25_partials<P>(g, rd, plb, nw, ib, jt, plb1);
  st25_ticket(pol, g, rd, st, mloc, flag, (unsigned)g.nblk);
}

// ------------------------------------------------------------ the kernel
template <class P, int CPT>
__global__ void __launch_bounds__(512) k_st25(const P pol_in, St25Geo g, Red rd, DevState* st) {
  using T = typename P::T;
  using Acc = typename P::Acc;
  using R0 = typename P::R0;
  using RT = typename P::RT;  // operand ring element: C when widening binary16 is free, else T
  static_assert(!P::IDENT || std::is_same<RT, T>::value, "identity operands are folded from the stages");
  constexpr int VEC = 16 / sizeof(T);
  // packed binary16 path (fold8h / dot8h): binary16 operands, binary32
  // arithmetic, exact products
  constexpr bool FASTH = P::FASTH;
  if (pol_in.skip(st)) return;
  P pol = pol_in;
  pol.prepare(st);  // device-resident scalars (e.g. CG beta) the host never sees
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  const int S = g.stages;
  const int nin = pol.nin();
  const int n = g.n;
  const int pe = (g.TJ + 2) * n;  // elements of one staged plane (rows j0-1 .. j0+TJ)
  T* raw = reinterpret_cast<T*>(smem + 128);
  RT* opr = reinterpret_cast<RT*>(raw + (size_t)S * P::NIN * pe);
  // per-(plane, warp) partial sums, folded over the warps once after the
  // plane loop (no block barrier per plane for the reductions)
  __shared__ double plb[ST25_IL_MAX * ST25_MAXW];  // R0 values are held exactly in binary64
  // a second reduced quantity (R0 and R1 both) gets its own buffer
  __shared__ double plb1[(P::HAS_R0 && P::HAS_R1) ? ST25_IL_MAX * ST25_MAXW : 1];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int jt = blockIdx.x % g.njt, ic = blockIdx.x / g.njt;
  const int j0 = jt << g.lgTJ, ib = g.i0 + ic * g.IL, ie = ib + g.IL;
  const int rlo = max(j0 - 1, 0), rhi = min(j0 + g.TJ, n - 1);
  const uint32_t bytes_in = (uint32_t)((rhi - rlo + 1) * n * sizeof(T));
  const int soff = (rlo - (j0 - 1)) * n;
  const int qlo = max(ib - 1, 0), qhi = min(ie, n - 1);

  auto issue = [&](int q) {  // one thread
    const int s = (q - qlo) % S;
    mbar_expect_tx(&bar[s], (uint32_t)nin * bytes_in);
    for (int k = 0; k < nin; ++k)
      bulk_g2s(raw + ((size_t)s * P::NIN + k) * pe + soff, pol.in(k) + (int64_t)q * g.nn + (int64_t)rlo * n,
               bytes_in, &bar[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int q = qlo; q <= qhi && q < qlo + S; ++q) issue(q);

  // operand of plane q (all staged rows) into ring slot q % 4: building
  // plane i+1 overwrites plane i-3, last read by the fold of plane i-2, which
  // precedes the barrier after building plane i; one barrier per plane.
  auto build = [&](int q) {
    const int s = (q - qlo) % S;
    mbar_wait(&bar[s], (uint32_t)(((q - qlo) / S) & 1));
    const T* rs = raw + (size_t)s * P::NIN * pe;
    RT* o = opr + (size_t)(q & 3) * pe;
    const int nch = (rhi - rlo + 1) << g.lgTR;
    for (int c = tid; c < nch; c += blockDim.x) {
      const int idx = soff + c * VEC;
      if constexpr (FASTH) {
        sts_u4(o + idx, pol.make_h(rs, pe, idx));
      } else {
        RT v[VEC];
        pol.make(rs, pe, idx, v);
        sts_vec<RT, VEC>(o + idx, v);
      }
    }
  };

  // IDENT policies (the operand is input 0 as stored: residuals) fold
  // straight from the staged planes, and no operand ring is built.
  auto stage_of = [&](int q) { return raw + (size_t)((q - qlo) % S) * P::NIN * pe; };
  auto wait_q = [&](int q) { mbar_wait(&bar[(q - qlo) % S], (uint32_t)(((q - qlo) / S) & 1)); };
  // IDENT: each thread keeps its own chunks of planes i-1 and i+1 in
  // registers, so only plane i must stay staged while it is folded: stage
  // i is refilled right after its fold, and S-2 planes stay in flight.
  RT xprv[CPT][VEC], xnxt[CPT][VEC];
  auto own_sidx = [&](int rr) {
    const int c = ((warp * CPT + rr) << 5) + lane;
    return ((c >> g.lgTR) + 1) * n + (c & (g.TR - 1)) * VEC;
  };
  if constexpr (P::IDENT) {
    if (ib - 1 >= 0) {
      wait_q(ib - 1);
      const RT* sp = stage_of(ib - 1);
#pragma unroll
      for (int rr = 0; rr < CPT; ++rr) lds_vec<RT, VEC>(sp + own_sidx(rr), xprv[rr]);
    }
    wait_q(ib);
    __syncthreads();  // stage ib-1 is consumed
    if (tid == 0 && ib - 1 >= qlo && ib - 1 + S <= qhi) {
      fence_proxy_async();
      issue(ib - 1 + S);
    }
  } else {
    if (ib - 1 >= 0) build(ib - 1);
    build(ib);
    __syncthreads();
    if (tid == 0) {
      fence_proxy_async();
      if (ib - 1 >= 0 && ib - 1 + S <= qhi) issue(ib - 1 + S);
      if (ib + S <= qhi) issue(ib + S);
    }
  }

  double mloc = 0.0;
  int flag = 0;
  // identity-operand policies start each point from a global vector (b, rhs):
  // those loads are issued one plane ahead so their latency hides behind a
  // plane of folding
  auto chunk_e0 = [&](int ii, int rr) -> int64_t {
    const int c = ((warp * CPT + rr) << 5) + lane;
    return (int64_t)ii * g.nn + (int64_t)(j0 + (c >> g.lgTR)) * n + (c & (g.TR - 1)) * VEC;
  };
  Acc nxt[CPT][VEC];
  if constexpr (P::IDENT) {
#pragma unroll
    for (int rr = 0; rr < CPT; ++rr) pol.init(chunk_e0(ib, rr), nxt[rr]);
  }
  for (int i = ib; i < ie; ++i) {
    Acc cur[CPT][VEC];
    if constexpr (P::IDENT) {
#pragma unroll
      for (int rr = 0; rr < CPT; ++rr)
#pragma unroll
        for (int v = 0; v < VEC; ++v) cur[rr][v] = nxt[rr][v];
      if (i + 1 < ie) {
#pragma unroll
        for (int rr = 0; rr < CPT; ++rr) pol.init(chunk_e0(i + 1, rr), nxt[rr]);
      }
    }
    const RT *om, *oc, *op;
    if constexpr (P::IDENT) {
      if (i + 1 <= n - 1) {
        wait_q(i + 1);
        const RT* sp = stage_of(i + 1);
#pragma unroll
        for (int rr = 0; rr < CPT; ++rr) lds_vec<RT, VEC>(sp + own_sidx(rr), xnxt[rr]);
      }
      om = i > 0 ? stage_of(i) : nullptr;  // non-null marks presence; the values are xprv / xnxt
      oc = stage_of(i);
      op = i < n - 1 ? stage_of(i) : nullptr;
    } else {
      if (i + 1 <= n - 1) build(i + 1);
      __syncthreads();
      if (tid == 0 && i + 1 <= n - 1 && i + 1 + S <= qhi) {
        fence_proxy_async();
        issue(i + 1 + S);
      }
      om = i > 0 ? opr + (size_t)((i - 1) & 3) * pe : nullptr;
      oc = opr + (size_t)(i & 3) * pe;
      op = i < n - 1 ? opr + (size_t)((i + 1) & 3) * pe : nullptr;
    }
    R0 a0[CPT];
    double a1[CPT];
#pragma unroll
    for (int rr = 0; rr < CPT; ++rr) {
      {
        const int c = ((warp * CPT + rr) << 5) + lane;  // chunk of the tile, row major
        const int jl = c >> g.lgTR, k0 = (c & (g.TR - 1)) * VEC;
        const int j = j0 + jl;
        const int sidx = (jl + 1) * n + k0;
        const int64_t e0 = (int64_t)i * g.nn + (int64_t)j * n + k0;
        if constexpr (FASTH) {
          float acc[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) acc[v] = 0.0f;  // matvec folds start from +0 (kernels.cpp:46)
          const uint32_t* ch = pol.ch;  // coefficients, binary16 in the low halves
          const unsigned short* ocu = reinterpret_cast<const unsigned short*>(oc);
          const uint4 ccu = lds_u4(oc + sidx);
          // the seven neighbours in stored-column order; absent i / j
          // neighbours are skipped, absent k neighbours fold the neutral -0 product
          if (om) fold8h<0>(acc, ch[0], lds_u4(om + sidx), 0u);
          if (j > 0) fold8h<0>(acc, ch[1], lds_u4(oc + sidx - n), 0u);
          fold8h<-1>(acc, ch[2], ccu, k0 > 0 ? (uint32_t)ocu[sidx - 1] : nh_of(ch[2]));
          fold8h<0>(acc, ch[3], ccu, 0u);
          fold8h<1>(acc, ch[4], ccu, k0 + VEC < n ? (uint32_t)ocu[sidx + VEC] : nh_of(ch[4]));
          if (j < n - 1) fold8h<0>(acc, ch[5], lds_u4(oc + sidx + n), 0u);
          if (op) fold8h<0>(acc, ch[6], lds_u4(op + sidx), 0u);
          a0[rr] = pol.epi_h(e0, acc, ccu);
          continue;
        }
        Acc acc[VEC];
        if constexpr (P::IDENT) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) acc[v] = cur[rr][v];
        } else {
          pol.init(e0, acc);
        }
        const auto& c7 = pol.c7;
        const auto f = pol.fold();
        RT cc[VEC], nb[VEC];
        lds_vec<RT, VEC>(oc + sidx, cc);
        // the seven neighbours in stored-column order; an absent neighbour is
        // skipped, never folded as a zero (fold_vec restores acc there)
        if (om) {
          if constexpr (P::IDENT) fold_vec(f, acc, c7[0], xprv[rr], false, false);
          else {
            lds_vec<RT, VEC>(om + sidx, nb);
            fold_vec(f, acc, c7[0], nb, false, false);
          }
        }
        if (j > 0) {
          lds_vec<RT, VEC>(oc + sidx - n, nb);
          fold_vec(f, acc, c7[1], nb, false, false);
        }
        nb[0] = k0 > 0 ? oc[sidx - 1] : cc[0];
#pragma unroll
        for (int v = 1; v < VEC; ++v) nb[v] = cc[v - 1];
        fold_vec(f, acc, c7[2], nb, k0 == 0, false);
        fold_vec(f, acc, c7[3], cc, false, false);
        {
          const bool hasL = k0 + VEC < n;
#pragma unroll
          for (int v = 0; v < VEC - 1; ++v) nb[v] = cc[v + 1];
          nb[VEC - 1] = hasL ? oc[sidx + VEC] : cc[0];
          fold_vec(f, acc, c7[4], nb, false, !hasL);
        }
        if (j < n - 1) {
          lds_vec<RT, VEC>(oc + sidx + n, nb);
          fold_vec(f, acc, c7[5], nb, false, false);
        }
        if (op) {
          if constexpr (P::IDENT) fold_vec(f, acc, c7[6], xnxt[rr], false, false);
          else {
            lds_vec<RT, VEC>(op + sidx, nb);
            fold_vec(f, acc, c7[6], nb, false, false);
          }
        }
        if constexpr (P::IDENT) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) xprv[rr][v] = cc[v];
        }
        R0 c0 = Ar<R0>::zero();
        double d0 = 0.0;
        pol.epi(e0, acc, cc, c0, d0, mloc, flag);
        if (P::HAS_R0) a0[rr] = c0;
        if (P::HAS_R1) a1[rr] = d0;
      }
    }
    // pairwise tree over each 32-chunk block's lanes, then over this warp's
    // CPT contiguous blocks (total in lane 0), then over warps
    if (P::HAS_R0) a0[0] = warp_tree_cpt<CPT>(a0);
    if (P::HAS_R1) a1[0] = warp_tree_cpt<CPT>(a1);
    if (lane == 0) {
      if (P::HAS_R0) plb[(i - ib) * nw + warp] = to_dbl(a0[0]);
      if (P::HAS_R1) ((P::HAS_R0 && P::HAS_R1) ? plb1 : plb)[(i - ib) * nw + warp] = a1[0];
    }
    if constexpr (P::IDENT) {
      __syncthreads();  // plane i is no longer read (plane i+1 folds it from xprv): refill its stage
      if (tid == 0 && i + S <= qhi) {
        fence_proxy_async();
        issue(i + S);
      }
    }
  }
  st25_finish(pol, g, rd, st, plb, nw, ib, jt, mloc, flag, (P::HAS_R0 && P::HAS_R1) ? plb1 : plb);
}

// ------------------------------------------------ binary16 operator passes
// k_st25h: the FASTH operator passes (binary16 storage, binary32 arithmetic:
// CG p-update + SpMV, Arnoldi matvec) with the operand of each thread's own
// chunks kept in registers for planes i-1, i, i+1 (rotated by unrolling the
// plane loop by three). Only plane i's operand lives in shared memory (a
// 3-slot ring; the j +- 1 rows and the k edges of the fold read it), so a
// chunk's fold costs two 16-byte and two 2-byte shared loads. Ring rows are
// padded by 8 entries that hold the neutral k-edge operands, and off-grid
// halo rows hold the neutral j-edge operands: an absent neighbour folds a
// product of -0, which leaves every accumulator unchanged (the reference
// skips it), so the fold has no per-lane branches. The i-edges are
// warp-uniform branches. The j-halo rows of each plane are built by all
// warps evenly. Same arithmetic, same stored-column order, same reduction
// tree as k_st25. Requires finite binary16 coefficients (the host checks).
__device__ __forceinline__ uint4 splat4(uint32_t h16) {
  const uint32_t w = (h16 & 0xffffu) | (h16 << 16);
  return make_uint4(w, w, w, w);
}
// ring plane size in entries: TJ+2 rows of n entries, each after an 8-entry
// lead pad, plus one trailing pad
__host__ __device__ inline int st25h_plane(int TJ, int n) { return (TJ + 2) * (n + 8) + 8; }

// pairwise sums over the 32 lanes of CPT per-lane values at once (each a
// perfect butterfly subtree, the shape of warp_tree), then over the CPT
// contiguous 32-chunk blocks; the result is valid in lane 0
template <int CPT>
__device__ __forceinline__ float warp_tree_multi(float (&v)[CPT], int lane) {
  if constexpr (CPT == 2) {
    const bool odd = lane & 1;
    float s = odd ? v[1] : v[0];
    const float o = __shfl_xor_sync(0xffffffffu, odd ? v[0] : v[1], 1);
    s = __fadd_rn(s, o);  // even lanes: v[0] pairs, odd lanes: v[1] pairs
#pragma unroll
    for (int m = 2; m < 32; m <<= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, m));
    const float b = __shfl_sync(0xffffffffu, s, 1);
    return __fadd_rn(s, b);
  } else {
#pragma unroll
    for (int rr = 0; rr < CPT; ++rr) v[rr] = warp_tree(v[rr], 32);
#pragma unroll
    for (int s2 = 1; s2 < CPT; s2 <<= 1)
#pragma unroll
      for (int rr = 0; rr + s2 < CPT; rr += 2 * s2) v[rr] = __fadd_rn(v[rr], v[rr + s2]);
    return v[0];
  }
}

template <class P, int CPT, int MINB>
__global__ void __launch_bounds__(MINB == 2 ? 512 : 256, MINB == 2 ? 1 : MINB)
    k_st25h(const P pol_in, St25Geo g, Red rd, DevState* st) {
  using T = typename P::T;
  static_assert(P::FASTH && std::is_same<T, __half>::value, "binary16 storage only");
  constexpr int VEC = 8;
  if (pol_in.skip(st)) return;
  P pol = pol_in;
  pol.prepare(st);
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  const int S = g.stages;
  const int nin = pol.nin();
  const int n = g.n, rs = n + 8;
  const int pe = (g.TJ + 2) * n;
  const int pr = st25h_plane(g.TJ, n);
  T* raw = reinterpret_cast<T*>(smem + 128);
  T* ring = raw + (size_t)S * P::NIN * pe;  // 3 operand planes of pr entries
  __shared__ float plb[ST25_IL_MAX * ST25_MAXW];  // binary32 partials (R0 = float)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;

  // Persistent CTAs: tiles blockIdx.x, +gridDim.x, ... The TMA stream runs
  // across tile boundaries (thread 0 issues the planes of all of this CTA's
  // tiles in consumption order), so the pipeline never drains.
  int iss_t = blockIdx.x, iss_q = 0, iss_qhi = -1, iss_s = 0;
  uint32_t iss_bytes = 0;
  int64_t iss_src = 0;
  T* iss_dst = raw;
  auto iss_tile = [&]() {  // geometry of tile iss_t (thread 0)
    const int jt = iss_t % g.njt, ic = iss_t / g.njt;
    const int j0 = jt << g.lgTJ, ib = g.i0 + ic * g.IL;
    const int rlo = max(j0 - 1, 0), rhi = min(j0 + g.TJ, n - 1);
    iss_q = max(ib - 1, 0);
    iss_qhi = min(ib + g.IL, n - 1);
    iss_bytes = (uint32_t)((rhi - rlo + 1) * n * sizeof(T));
    iss_src = (int64_t)rlo * n;
    iss_dst = raw + (rlo - (j0 - 1)) * n;
  };
  auto issue_next = [&]() {
    if (iss_t >= g.nblk) return;
    mbar_expect_tx(&bar[iss_s], (uint32_t)nin * iss_bytes);
    for (int k = 0; k < nin; ++k)
      bulk_g2s(iss_dst + ((size_t)iss_s * P::NIN + k) * pe, pol.in(k) + (int64_t)iss_q * g.nn + iss_src, iss_bytes,
               &bar[iss_s]);
    iss_s = iss_s + 1 == S ? 0 : iss_s + 1;
    if (++iss_q > iss_qhi) {
      iss_t += gridDim.x;
      if (iss_t < g.nblk) iss_tile();
    }
  };
  const uint32_t* ch = pol.ch;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  {  // the k-edge pads of every ring row hold the neutral operands
    const unsigned short ne2 = (unsigned short)nh_of(ch[2]), ne4 = (unsigned short)nh_of(ch[4]);
    unsigned short* ru = reinterpret_cast<unsigned short*>(ring);
    for (int t = tid; t < 3 * (g.TJ + 3); t += blockDim.x) {
      const int sl = t / (g.TJ + 3), r = t % (g.TJ + 3);
      ru[sl * pr + r * rs + 0] = ne4;  // after the end of row r-1
      ru[sl * pr + r * rs + 7] = ne2;  // before the start of row r
    }
  }
  __syncthreads();
  if (tid == 0) {
    iss_tile();
    for (int s = 0; s < S; ++s) issue_next();
  }
  int cs = 0;
  uint32_t cph = 0;  // consumption: stage, parity
  auto consume = [&]() -> const T* {
    mbar_wait(&bar[cs], cph);
    const T* r = raw + (size_t)cs * P::NIN * pe;
    if (++cs == S) {
      cs = 0;
      cph ^= 1u;
    }
    return r;
  };
  // own chunks: fixed positions within every tile
  int sidx[CPT], ridx[CPT], ebase[CPT];
#pragma unroll
  for (int rr = 0; rr < CPT; ++rr) {
    const int c = ((warp * CPT + rr) << 5) + lane;
    const int jl = c >> g.lgTR, k0 = (c & (g.TR - 1)) * VEC;
    sidx[rr] = (jl + 1) * n + k0;
    ridx[rr] = (jl + 1) * rs + 8 + k0;
    ebase[rr] = jl * n + k0;
  }
  const int nhalo = 2 * g.TR, hpw = (nhalo + nw - 1) / nw;  // halo chunks spread evenly over the warps
  const uint4 n1 = splat4(nh_of(ch[1])), n5 = splat4(nh_of(ch[5]));

  for (int tile = blockIdx.x; tile < g.nblk; tile += gridDim.x) {
    const int jt = tile % g.njt, ic = tile / g.njt;
    const int j0 = jt << g.lgTJ, ib = g.i0 + ic * g.IL, ie = ib + g.IL;
    const bool hrow0 = j0 > 0, hrow1 = j0 + g.TJ < n;
    // off-grid halo rows hold the neutral j-edge operands (the previous
    // tile's folds are complete: st25_partials ends with a barrier)
    for (int t = tid; t < 3 * g.TR; t += blockDim.x) {
      const int sl = t / g.TR, k0 = (t % g.TR) * VEC;
      if (!hrow0) sts_u4(ring + sl * pr + 8 + k0, n1);
      if (!hrow1) sts_u4(ring + sl * pr + (g.TJ + 1) * rs + 8 + k0, n5);
    }
    int64_t e0[CPT];
#pragma unroll
    for (int rr = 0; rr < CPT; ++rr) e0[rr] = (int64_t)ib * g.nn + (int64_t)j0 * n + ebase[rr];

    // the operand of plane q: own chunks -> registers (and the ring slot),
    // halo chunks -> the ring slot
    auto build = [&](const T* rsg, T* slot, uint4 (&xo)[CPT], bool to_ring) {
#pragma unroll
      for (int rr = 0; rr < CPT; ++rr) {
        xo[rr] = pol.make_h(rsg, pe, sidx[rr]);
        if (to_ring) sts_u4(slot + ridx[rr], xo[rr]);
      }
      if (to_ring)
        for (int x = lane; x < hpw; x += 32) {
          const int hc = warp * hpw + x;
          if (hc < nhalo) {
            const bool top = hc < g.TR;
            if (top ? hrow0 : hrow1) {
              const int k0 = (hc & (g.TR - 1)) * VEC;
              const int row = top ? 0 : g.TJ + 1;
              sts_u4(slot + row * rs + 8 + k0, pol.make_h(rsg, pe, row * n + k0));
            }
          }
        }
    };

    uint4 xa[CPT], xb[CPT], xq[CPT];
    if (ib - 1 >= 0) build(consume(), nullptr, xa, false);
    build(consume(), ring, xb, true);
    __syncthreads();  // stages of planes ib-1, ib consumed; plane ib in the ring
    if (tid == 0) {
      fence_proxy_async();
      issue_next();
      if (ib - 1 >= 0) issue_next();
    }

    // one plane: build plane i+1 into xp (ring slot sp), fold plane i from
    // xm / xc / xp and ring slot sc
    auto plane = [&](int i, const uint4 (&xm)[CPT], const uint4 (&xc)[CPT], uint4 (&xp)[CPT], int sc, int sp) {
      uint4 pf[CPT];  // per-point global operands of the epilogue (Arnoldi: v_0), a build + barrier ahead
#pragma unroll
      for (int rr = 0; rr < CPT; ++rr) pf[rr] = pol.pref(e0[rr]);
      const bool hasp = i + 1 <= n - 1, hasm = i > 0;
      if (hasp) build(consume(), ring + (size_t)sp * pr, xp, true);
      // plane i+1 is in the ring and its stage consumed. Slot (i+2)%3, written
      // next, was last read by the fold of plane i-1, before this barrier.
      __syncthreads();
      if (tid == 0 && hasp) {
        fence_proxy_async();
        issue_next();
      }
      const T* oc = ring + (size_t)sc * pr;
      const unsigned short* ocu = reinterpret_cast<const unsigned short*>(oc);
      float a0[CPT];
#pragma unroll
      for (int rr = 0; rr < CPT; ++rr) {
        float acc[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[v] = 0.0f;  // matvec folds start from +0 (kernels.cpp:46)
        const int ri = ridx[rr];
        const uint4 vjm = lds_u4(oc + ri - rs), vjp = lds_u4(oc + ri + rs);
        const uint32_t em = ocu[ri - 1], ep = ocu[ri + VEC];
        // stored-column order (problems.cpp:28-34): i-1, j-1, k-1, centre, k+1, j+1, i+1
        if (hasm) fold8h<0>(acc, ch[0], xm[rr], 0u);
        fold8h<0>(acc, ch[1], vjm, 0u);
        fold8h<-1>(acc, ch[2], xc[rr], em);
        fold8h<0>(acc, ch[3], xc[rr], 0u);
        fold8h<1>(acc, ch[4], xc[rr], ep);
        fold8h<0>(acc, ch[5], vjp, 0u);
        if (hasp) fold8h<0>(acc, ch[6], xp[rr], 0u);
        a0[rr] = pol.epi_h(e0[rr], acc, xc[rr], pf[rr]);
        e0[rr] += g.nn;
      }
      const float t = warp_tree_multi<CPT>(a0, lane);
      if (lane == 0) plb[(i - ib) * nw + warp] = t;
    };
    int i = ib;
    for (; i + 3 <= ie; i += 3) {  // ring slots: plane ib in 0, ib+1 in 1, ...
      plane(i, xa, xb, xq, 0, 1);
      plane(i + 1, xb, xq, xa, 1, 2);
      plane(i + 2, xq, xa, xb, 2, 0);
    }
    if (i < ie) plane(i, xa, xb, xq, 0, 1);
    if (i + 1 < ie) plane(i + 1, xb, xq, xa, 1, 2);
    st25_partials<P>(g, rd, plb, nw, ib, jt);
    __syncthreads();  // plb and the ring are free for the next tile
  }
  st25_ticket(pol, g, rd, st, 0.0, 0, gridDim.x);
}

// ------------------------------------------------------------ policies
#define ST25_VEC (16 / (int)sizeof(T))

// Element type of the operand ring. Widening binary16 operands to binary32
// in the ring (exact, one conversion per point instead of per use) was
// measured slower on B200 (r01: CG SpMV 356 -> 438 us): the doubled ring
// forces a 2-stage TMA ring to keep two CTAs per SM. The ring stays in the
// storage type.
template <class T, class C>
struct RingOf {
  using type = T;
};

// CG: p = r + beta p (first: p = r), q = H p, pap = dot(p, q)  (= k_cg_spmvp)
template <class TS, class C>
struct PolSpmvp {
  using T = TS;
  using Acc = C;
  using R0 = C;
  using RT = typename RingOf<T, C>::type;
  static constexpr int NIN = 2;
  static constexpr bool HAS_R0 = true, HAS_R1 = false, HAS_MAX = false, HAS_FLAG = false, IDENT = false;
  static constexpr bool FASTH = std::is_same<T, __half>::value && std::is_same<C, float>::value;
  C c7[7];
  const T* r;
  const T* p_in;
  T* p_out;
  T* q;
  C beta;
  int first;
  uint32_t ch[7];  // FASTH: c7 as binary16 (exact: the coefficients are u_r values)
  __device__ bool skip(DevState* st) const { return *(volatile int*)&st->cg_done; }
  __device__ void prepare(DevState* st) {
    beta = from_dbl<C>(st->cg_beta);
    if constexpr (FASTH)
      for (int k = 0; k < 7; ++k) ch[k] = __half_as_ushort(__float2half_rn(c7[k]));
  }
  // FASTH: p = r + beta p as FMUL2 products + FHADD sums, one F2FP per pair
  __device__ uint4 make_h(const T* rs, int pe, int idx) const {
    const uint4 rv = lds_u4(rs + idx);
    if (first) return rv;
    const uint4 pv = lds_u4(rs + pe + idx);
    const float2 b2 = make_float2(beta, beta);
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t pk = u4_at(pv, k), rk = u4_at(rv, k);
      const float2 bp = __fmul2_rn(b2, __half22float2(*reinterpret_cast<const __half2*>(&pk)));
      o[k] = pack_h2(fhadd<0>(rk, bp.x), fhadd<1>(rk, bp.y));
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
  }
  __device__ uint4 pref(int64_t) const { return make_uint4(0, 0, 0, 0); }
  __device__ C epi_h(int64_t e0, const float (&acc)[8], const uint4& pc, const uint4& = uint4()) const {
    const uint4 qv = make_uint4(pack_h2(acc[0], acc[1]), pack_h2(acc[2], acc[3]), pack_h2(acc[4], acc[5]),
                                pack_h2(acc[6], acc[7]));
    *reinterpret_cast<uint4*>(q + e0) = qv;
    *reinterpret_cast<uint4*>(p_out + e0) = pc;
    return dot8h(pc, qv);
  }
  __device__ int nin() const { return first ? 1 : 2; }
  __device__ const T* in(int k) const { return k == 0 ? r : p_in; }
  __device__ void make(const T* rs, int pe, int idx, RT (&v)[ST25_VEC]) const {
    T rv[ST25_VEC];
    lds16<T, ST25_VEC>(rs + idx, rv);
    if (first) {
#pragma unroll
      for (int e = 0; e < ST25_VEC; ++e) v[e] = ld_c<T, RT>(rv[e]);
    } else {
      T pv[ST25_VEC];
      lds16<T, ST25_VEC>(rs + pe + idx, pv);
      C bp[ST25_VEC];
      mul_vec<C, T, ST25_VEC>(beta, pv, bp);
#pragma unroll
      for (int e = 0; e < ST25_VEC; ++e) v[e] = ld_c<T, RT>(st_t<T, C>(Ar<C>::add(ld_c<T, C>(rv[e]), bp[e])));
    }
  }
  __device__ MatvecF<C, RT> fold() const { return MatvecF<C, RT>(); }
  __device__ void init(int64_t, C (&acc)[ST25_VEC]) const {
#pragma unroll
    for (int e = 0; e < ST25_VEC; ++e) acc[e] = Ar<C>::zero();
  }
  __device__ void epi(int64_t e0, const C (&acc)[ST25_VEC], const RT (&cc)[ST25_VEC], C& c, double&, double&,
                      int&) const {
    T qv[ST25_VEC], pv[ST25_VEC];
    C tc[ST25_VEC];
#pragma unroll
    for (int e = 0; e < ST25_VEC; ++e) {
      qv[e] = st_t<T, C>(acc[e]);
      pv[e] = st_t<T, RT>(cc[e]);  // exact: cc holds a T value
      tc[e] = Ar<C>::mul(ld_c<RT, C>(cc[e]), ld_c<T, C>(qv[e]));
    }
    st_vec<T, ST25_VEC>(q, e0, qv);
    st_vec<T, ST25_VEC>(p_out, e0, pv);
    c = seg_sum<C, ST25_VEC>(tc, ST25_VEC);
  }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ void finish(C pap, double t1, DevState* st) const { EpiCgPap{}.finish(pap, t1, st); }
};

// Arnoldi step: v_j = round(inv * w_prev) (stored), w = S v_j, h_0j = dot(w, v_0)  (= k_gm_matvec)
template <class TS, class C>
struct PolGmMatvec {
  using T = TS;
  using Acc = C;
  using R0 = C;
  using RT = typename RingOf<T, C>::type;
  static constexpr int NIN = 1;
  static constexpr bool HAS_R0 = true, HAS_R1 = false, HAS_MAX = false, HAS_FLAG = false, IDENT = false;
  static constexpr bool FASTH = std::is_same<T, __half>::value && std::is_same<C, float>::value;
  C c7[7];
  const T* wprev;
  double inv;
  T* vj;
  const T* v0;
  T* w;
  uint32_t ch[7];
  int inv_dev;  // 1: inv is st->gm_inv, formed by the previous step's epilogue (no host sync in between)
  __device__ bool skip(DevState*) const { return false; }
  __device__ void prepare(DevState* st) {
    if (inv_dev) inv = *(volatile double*)&st->gm_inv;
    if constexpr (FASTH)
      for (int k = 0; k < 7; ++k) ch[k] = __half_as_ushort(__float2half_rn(c7[k]));
  }
  // FASTH (= the accum FP32 mode): v = round_h(round_f32(inv) * w), the product in
  // binary32 (scale_rn<T, true>), two lanes per FMUL2 / F2FP
  __device__ uint4 make_h(const T* rs, int, int idx) const {
    const uint4 wv = lds_u4(rs + idx);
    const float invf = (float)inv;
    const float2 i2 = make_float2(invf, invf);
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t wk = u4_at(wv, k);
      const float2 pr = __fmul2_rn(i2, __half22float2(*reinterpret_cast<const __half2*>(&wk)));
      o[k] = pack_h2(pr.x, pr.y);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
  }
  __device__ uint4 pref(int64_t e0) const {  // v_0 (unless v_j is v_0)
    return vj == v0 ? make_uint4(0, 0, 0, 0) : __ldg(reinterpret_cast<const uint4*>(v0 + e0));
  }
  __device__ C epi_h(int64_t e0, const float (&acc)[8], const uint4& vc, const uint4& v0p) const {
    const uint4 wq = make_uint4(pack_h2(acc[0], acc[1]), pack_h2(acc[2], acc[3]), pack_h2(acc[4], acc[5]),
                                pack_h2(acc[6], acc[7]));
    *reinterpret_cast<uint4*>(vj + e0) = vc;
    *reinterpret_cast<uint4*>(w + e0) = wq;
    return dot8h(wq, vj == v0 ? vc : v0p);
  }
  __device__ C epi_h(int64_t e0, const float (&acc)[8], const uint4& vc) const {
    return epi_h(e0, acc, vc, pref(e0));
  }
  __device__ int nin() const { return 1; }
  __device__ const T* in(int) const { return wprev; }
  __device__ void make(const T* rs, int, int idx, RT (&v)[ST25_VEC]) const {
    T wv[ST25_VEC];
    lds16<T, ST25_VEC>(rs + idx, wv);
#pragma unroll
    for (int e = 0; e < ST25_VEC; ++e) v[e] = ld_c<T, RT>(scale_rn<T, FASTH>(inv, wv[e]));
  }
  __device__ MatvecF<C, RT> fold() const { return MatvecF<C, RT>(); }
  __device__ void init(int64_t, C (&acc)[ST25_VEC]) const {
#pragma unroll
    for (int e = 0; e < ST25_VEC; ++e) acc[e] = Ar<C>::zero();
  }
  __device__ void epi(int64_t e0, const C (&acc)[ST25_VEC], const RT (&cc)[ST25_VEC], C& c, double&, double&,
                      int&) const {
    T wv[ST25_VEC], vv[ST25_VEC];
    C v0c[ST25_VEC], tc[ST25_VEC];
#pragma unroll
    for (int e = 0; e < ST25_VEC; ++e) vv[e] = st_t<T, RT>(cc[e]);
    st_vec<T, ST25_VEC>(vj, e0, vv);
    if (vj == v0) {
#pragma unroll
      for (int e = 0; e < ST25_VEC; ++e) v0c[e] = ld_c<RT, C>(cc[e]);
    } else {
      T v0v[ST25_VEC];
      ld_vec<T, ST25_VEC>(v0, e0, v0v);
#pragma unroll
      for (int e = 0; e < ST25_VEC; ++e) v0c[e] = ld_c<T, C>(v0v[e]);
    }
#pragma unroll
    for (int e = 0; e < ST25_VEC; ++e) {
      wv[e] = st_t<T, C>(acc[e]);
      tc[e] = Ar<C>::mul(ld_c<T, C>(wv[e]), v0c[e]);
    }
    st_vec<T, ST25_VEC>(w, e0, wv);
    c = seg_sum<C, ST25_VEC>(tc, ST25_VEC);
  }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ void finish(C h, double t1, DevState* st) const { EpiHcol{0}.finish(h, t1, st); }
};

// GMRES restart residual r = rhs - S x (x != 0), max|r|, ||r||, finiteness (= k_gm_resid)
template <class TS, class C>
struct PolGmResid {
  using T = TS;
  using Acc = C;
  using R0 = C;
  using RT = TS;
  static constexpr int NIN = 1;
  static constexpr bool HAS_R0 = false, HAS_R1 = true, HAS_MAX = true, HAS_FLAG = true, IDENT = true;
  static constexpr bool FASTH = false;
  C c7[7];
  const T* x;
  const T* rhs;
  T* r;
  __device__ bool skip(DevState*) const { return false; }
  __device__ void prepare(DevState*) {}
  __device__ int nin() const { return 1; }
  __device__ const T* in(int) const { return x; }
  __device__ void make(const T* rs, int, int idx, T (&v)[ST25_VEC]) const { lds16<T, ST25_VEC>(rs + idx, v); }
  __device__ ResidF<C, T> fold() const { return ResidF<C, T>(); }
  __device__ void init(int64_t e0, C (&acc)[ST25_VEC]) const {
    T bv[ST25_VEC];
    ld_vec<T, ST25_VEC>(rhs, e0, bv);
#pragma unroll
    for (int e = 0; e < ST25_VEC; ++e) acc[e] = ld_c<T, C>(bv[e]);
  }
  __device__ void epi(int64_t e0, const C (&acc)[ST25_VEC], const T (&)[ST25_VEC], C&, double& d, double& m,
                      int& flag) const {
    T rv[ST25_VEC];
    double td[ST25_VEC];
#pragma unroll
    for (int e = 0; e < ST25_VEC; ++e) {
      rv[e] = st_t<T, C>(acc[e]);
      const double dv = to_dbl(rv[e]);
      td[e] = __dmul_rn(dv, dv);
      flag |= finite_t(rv[e]) ? 0 : 1;
      m = (dv == dv) ? fmax(m, fabs(dv)) : m;
    }
    st_vec<T, ST25_VEC>(r, e0, rv);
    d = seg_sum<double, ST25_VEC>(td, ST25_VEC);
  }
  __device__ int* flag_dst(DevState* st) const { return &st->flags; }
  __device__ void finish(C t0, double ss, DevState* st) const { EpiRedD{}.finish(t0, ss, st); }
};

// Outer residual s = b - A x in u_f (binary64 carried), max|s|, ||s||, e (= k_resid_A)
template <int PF>
struct PolResidA {
  using T = double;
  using Acc = double;
  using R0 = double;
  using RT = double;
  static constexpr int NIN = 1;
  static constexpr bool HAS_R0 = false, HAS_R1 = true, HAS_MAX = true, HAS_FLAG = false, IDENT = true;
  static constexpr bool FASTH = false;
  double c7[7];
  const double* x;
  const double* b;
  double* s;
  int scaling;
  double nsc;  // 2^-ns: the squares are those of s 2^-ns (1.0: unscaled)
  __device__ bool skip(DevState*) const { return false; }
  __device__ void prepare(DevState*) {}
  __device__ int nin() const { return 1; }
  __device__ const double* in(int) const { return x; }
  __device__ void make(const double* rs, int, int idx, double (&v)[2]) const { lds16<double, 2>(rs + idx, v); }
  __device__ ResidAF<PF> fold() const { return ResidAF<PF>(); }
  __device__ void init(int64_t e0, double (&acc)[2]) const { ld_vec<double, 2>(b, e0, acc); }
  __device__ void epi(int64_t e0, const double (&acc)[2], const double (&)[2], double&, double& d, double& m,
                      int&) const {
    double td[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const double av = nsc != 1.0 ? __dmul_rn(acc[e], nsc) : acc[e];
      td[e] = __dmul_rn(av, av);
      m = (acc[e] == acc[e]) ? fmax(m, fabs(acc[e])) : m;
    }
    if (s) st_vec<double, 2>(s, e0, acc);
    d = seg_sum<double, 2>(td, 2);
  }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ void finish(double t0, double ss, DevState* st) const { EpiResidA{scaling}.finish(t0, ss, st); }
};

// Speculative outer residual (u_f = binary64): s = b - A x as PolResidA, and in
// the same pass rhat = round_{u_r}(s 2^-ep) (solver.cpp:86-92) with the
// exponent ep of the previous outer step, plus ||rhat||^2 as a second
// reduced quantity (R0). s itself is not stored. The host accepts the pass
// when the exponent the epilogue derives from max|s| equals ep; otherwise it
// reruns PolResidA + k_scale_round (same values, same trees).
template <class TR>
struct PolResidSpec {
  using T = double;
  using Acc = double;
  using R0 = double;
  using RT = double;
  static constexpr int NIN = 1;
  static constexpr bool HAS_R0 = true, HAS_R1 = true, HAS_MAX = true, HAS_FLAG = false, IDENT = true;
  static constexpr bool FASTH = false;
  double c7[7];
  const double* x;
  const double* b;
  TR* rhat;
  int ep;
  double p2;  // 2^-ep
  int scaling;
  double nsc, nsc_r;  // 2^-ns for the squares of s, and for those of rhat (1.0: unscaled)
  __device__ bool skip(DevState*) const { return false; }
  __device__ void prepare(DevState*) {}
  __device__ int nin() const { return 1; }
  __device__ const double* in(int) const { return x; }
  __device__ void make(const double* rs, int, int idx, double (&v)[2]) const { lds16<double, 2>(rs + idx, v); }
  __device__ ResidAF<P_DOUBLE> fold() const { return ResidAF<P_DOUBLE>(); }
  __device__ void init(int64_t e0, double (&acc)[2]) const { ld_vec<double, 2>(b, e0, acc); }
  __device__ void epi(int64_t e0, const double (&acc)[2], const double (&)[2], double& c, double& d, double& m,
                      int&) const {
    double td[2], tc[2];
    TR o[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const double av = nsc != 1.0 ? __dmul_rn(acc[e], nsc) : acc[e];
      td[e] = __dmul_rn(av, av);
      m = (acc[e] == acc[e]) ? fmax(m, fabs(acc[e])) : m;
      o[e] = from_dbl<TR>(ep != 0 ? ldexp_fast(acc[e], -ep, p2) : acc[e]);
      double dv = to_dbl(o[e]);
      if (nsc_r != 1.0) dv = __dmul_rn(dv, nsc_r);
      tc[e] = __dmul_rn(dv, dv);
    }
    st_vec<TR, 2>(rhat, e0, o);
    c = seg_sum<double, 2>(tc, 2);
    d = seg_sum<double, 2>(td, 2);
  }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ void finish(double t0, double ss, DevState* st) const { EpiResidSpec{scaling}.finish(t0, ss, st); }
};

#undef ST25_VEC

}  // namespace gadi
