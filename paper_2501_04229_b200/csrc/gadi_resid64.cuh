// gadi_resid64.cuh — lean versions of two streaming passes of the C3 outer step.
//
// k_resid64: the binary64 outer residual s = b - A x of the 7-point stencil
// (residual_uf with u_f = double, solver.cpp:190-192, kernels.cpp:56-69) with
// the policies of gadi_st25.cuh (PolResidA<P_DOUBLE>: s, max|s|, ||s||^2;
// PolResidSpec: the speculative pass that also rounds rhat and reduces
// ||rhat||^2). Same arithmetic per point (one DMUL and one DADD per stored
// neighbour in stored-column order, absent neighbours skipped) and the same
// perfect pairwise tree over the global index as k_st25, so the results are
// the bits of k_st25 / k_resid_A. What differs is the schedule:
//   * the plane loop is unrolled by three, so the thread's own points of
//     planes i-1, i, i+1 and the prefetched b rotate by renaming (no moves);
//   * absent k neighbours fold the coefficient's neutral operand (the product
//     is +0 and acc - (+0) == acc for every acc), so the fold has no selects;
//     absent i / j neighbours are warp-uniform branches;
//   * stages are released per warp through `empty` mbarriers (no block-wide
//     barrier in the plane loop): the bulk copies run S-2 planes ahead and
//     only the issuing thread ever waits for the slowest warp;
//   * the CPT chunk sums of both reduced quantities go through ONE
//     reduce-scatter multi-tree per plane (same pairs at every level).
// Requires finite coefficients and n >= 64 (a warp's 32 chunks lie in one grid
// row); the host falls back to k_st25 otherwise.
//
// k_gm_resid0p: k_gm_resid0 (gadi_kernels.cuh) for the stencil operators with
// the 16-byte chunks kept packed: HMUL2 scaling, one bit test per word for the
// -0 entries the zero-start sign rules touch, squares as FHFMA onto -0.
#pragma once

#include "gadi_st25.cuh"

namespace gadi {

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Pairwise trees over the 32 lanes of the CPT per-lane values of two
// quantities at once (warp_tree_cpt for each, sharing the shuffle levels):
// level xor 1 splits the two quantities, levels xor 2.. split the CPT trees,
// the remaining levels are plain butterflies, then the tree over rr. On
// return lanes with bit 0 clear hold the total of a[], lanes with bit 0 set
// the total of b[]. Same pairs at every level as warp_tree_cpt.
template <int CPT>
__device__ __forceinline__ double warp_tree2_cpt(const double (&a)[CPT], const double (&b)[CPT]) {
  const int lane = threadIdx.x & 31;
  double w[CPT];
  {
    const bool hi = (lane & 1) != 0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const double send = hi ? a[k] : b[k];
      const double keep = hi ? b[k] : a[k];
      w[k] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 1));
    }
  }
  int o = 2;
#pragma unroll
  for (int m = CPT; m > 1; m >>= 1, o <<= 1) {
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < m / 2; ++k) {
      const double send = hi ? w[k] : w[k + m / 2];
      const double keep = hi ? w[k + m / 2] : w[k];
      w[k] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, o));
    }
  }
  double t = w[0];
#pragma unroll
  for (int oo = o; oo < 32; oo <<= 1) t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, oo));
#pragma unroll
  for (int oo = o >> 1; oo >= 2; oo >>= 1) t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, oo));
  return t;
}

// s != nullptr / rhat: what a policy stores per point
template <class P>
struct R64Out;
template <int PF>
struct R64Out<PolResidA<PF>> {
  using O = double;
  static __device__ __forceinline__ O* ptr(const PolResidA<PF>& p) { return p.s; }
};
template <class TR>
struct R64Out<PolResidSpec<TR>> {
  using O = TR;
  static __device__ __forceinline__ O* ptr(const PolResidSpec<TR>& p) { return p.rhat; }
};

// two consecutive entries as one store (p is aligned to the pair)
template <class O>
__device__ __forceinline__ void st2(O* p, O a, O b) {
  if constexpr (sizeof(O) == 2) {
    *reinterpret_cast<uint32_t*>(p) = (uint32_t)*reinterpret_cast<const unsigned short*>(&a) |
                                      ((uint32_t)*reinterpret_cast<const unsigned short*>(&b) << 16);
  } else if constexpr (sizeof(O) == 4) {
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&a);
    u.y = *reinterpret_cast<const uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = u;
  } else {
    *reinterpret_cast<double2*>(p) = make_double2((double)a, (double)b);
  }
}

template <class P, int CPT, int THREADS, int MINB, int R64_S /* staged planes, a power of two */>
__global__ void __launch_bounds__(THREADS, MINB) k_resid64(const P pol, St25Geo g, Red rd, DevState* st) {
  static_assert(P::IDENT && std::is_same<typename P::T, double>::value, "binary64 identity-operand policies");
  static_assert(P::HAS_R1 && P::HAS_MAX && !P::HAS_FLAG, "residual policies");
  constexpr bool TWO = P::HAS_R0;  // PolResidSpec: ||rhat||^2 as a second reduced quantity
  using O = typename R64Out<P>::O;
  constexpr int S = R64_S;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 8;
  double* raw = reinterpret_cast<double*>(smem + 128);
  __shared__ double plb[ST25_IL_MAX * ST25_MAXW];
  __shared__ double plb1[TWO ? ST25_IL_MAX * ST25_MAXW : 1];

  const int n = g.n;
  const int pe = (g.TJ + 2) * n;
  const int ps = pe + 2;  // stage stride: the rows, then the neutral k-edge operands
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = THREADS / 32;
  const int jt = blockIdx.x % g.njt, ic = blockIdx.x / g.njt;
  const int j0 = jt << g.lgTJ, ib = g.i0 + ic * g.IL, ie = ib + g.IL;
  const int rlo = max(j0 - 1, 0), rhi = min(j0 + g.TJ, n - 1);
  const uint32_t bytes_in = (uint32_t)((rhi - rlo + 1) * n * sizeof(double));
  const int soff = (rlo - (j0 - 1)) * n;
  const int qlo = max(ib - 1, 0), qhi = min(ie, n - 1);

  const double c0 = pol.c7[0], c1 = pol.c7[1], c2 = pol.c7[2], c3 = pol.c7[3], c4 = pol.c7[4], c5 = pol.c7[5],
               c6 = pol.c7[6];
  // An absent neighbour folds the operand whose product with the coefficient
  // is +0: acc - (+0) == acc for every acc (the reference skips the entry).
  // Off-grid halo rows and the two pad entries of every stage hold them.
  for (int s = 0; s < S; ++s) {
    double* sb = raw + (size_t)s * ps;
    if (j0 == 0)
      for (int k = tid; k < n; k += THREADS) sb[k] = copysign(0.0, c1);
    if (j0 + g.TJ == n)
      for (int k = tid; k < n; k += THREADS) sb[(g.TJ + 1) * n + k] = copysign(0.0, c5);
    if (tid == 0) {
      sb[pe] = copysign(0.0, c2);
      sb[pe + 1] = copysign(0.0, c4);
    }
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nw);
    }
    mbar_fence_init();
  }
  __syncthreads();

  // thread 0: plane q into stage (q - qlo) % S, once every warp has released
  // the plane that used the stage before
  int iss_q = qlo;
  auto issue = [&]() {
    const int p = iss_q - qlo, s = p & (S - 1);
    if (p >= S) mbar_wait(&empty[s], (uint32_t)((p / S - 1) & 1));
    fence_proxy_async();
    mbar_expect_tx(&full[s], bytes_in);
    bulk_g2s(raw + (size_t)s * ps + soff, pol.x + (int64_t)iss_q * g.nn + (int64_t)rlo * n, bytes_in, &full[s]);
    ++iss_q;
  };
  if (tid == 0)
    while (iss_q <= qhi && iss_q < qlo + S) issue();

  auto stage_of = [&](int q) { return raw + (size_t)((q - qlo) & (S - 1)) * ps; };
  auto wait_full = [&](int q) { mbar_wait(&full[(q - qlo) & (S - 1)], (uint32_t)(((q - qlo) / S) & 1)); };
  auto release = [&](int q) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[(q - qlo) & (S - 1)]);
  };

  // this thread's chunks: chunk c = ((warp*CPT + rr) << 5) + lane of the tile,
  // row major; the tile's rows are whole grid rows, so chunk c sits 2c
  // entries into the tile both in global memory and in a staged plane
  const int cb = (warp * CPT) << 5 | lane;
  const int own = n + 2 * cb;  // offset of chunk rr = 0 in a staged plane (+ 64 rr)
  int offl[CPT], offr[CPT];    // the k-1 / k+1 operands of the chunk's end points
#pragma unroll
  for (int rr = 0; rr < CPT; ++rr) {
    const int k0 = ((cb + 32 * rr) & (g.TR - 1)) * 2;
    offl[rr] = k0 == 0 ? pe : own + 64 * rr - 1;
    offr[rr] = k0 + 2 == n ? pe + 1 : own + 64 * rr + 2;
  }
  const int64_t tb = (int64_t)j0 * n + 2 * cb;  // j*n + k0 of chunk rr = 0
  const double* bp = pol.b + (int64_t)ib * g.nn + tb;
  O* op = R64Out<P>::ptr(pol);
  if (op) op += (int64_t)ib * g.nn + tb;
  const double nsc = pol.nsc;

  double xa[CPT][2], xb[CPT][2], xc_[CPT][2];
  double ba[CPT][2], bb[CPT][2], bc[CPT][2];
  // prologue: own points of planes ib-1 and ib, b of plane ib
  if (ib - 1 >= 0) {
    wait_full(ib - 1);
    const double* sp = stage_of(ib - 1) + own;
#pragma unroll
    for (int rr = 0; rr < CPT; ++rr) lds16<double, 2>(sp + 64 * rr, xa[rr]);
    release(ib - 1);
  } else {
#pragma unroll
    for (int rr = 0; rr < CPT; ++rr) xa[rr][0] = xa[rr][1] = copysign(0.0, c0);
  }
  {
    wait_full(ib);
    const double* sp = stage_of(ib) + own;
#pragma unroll
    for (int rr = 0; rr < CPT; ++rr) {
      lds16<double, 2>(sp + 64 * rr, xb[rr]);
      ld_vec<double, 2>(bp, 64 * rr, ba[rr]);
    }
    bp += g.nn;
  }

  double mloc = 0.0;
  auto step = [&](int i, double (&xm)[CPT][2], double (&xc)[CPT][2], double (&xn)[CPT][2], double (&bcur)[CPT][2],
                  double (&bnxt)[CPT][2]) {
    // thread 0: refill the stages of the planes folded before plane i
    if (tid == 0)
      while (iss_q <= qhi && iss_q - S < i) issue();
    {  // b of plane i+1, one plane ahead (the last plane reloads its own: no predicated loads)
      const double* bq = i + 1 < ie ? bp : bp - g.nn;
#pragma unroll
      for (int rr = 0; rr < CPT; ++rr) ld_vec<double, 2>(bq, 64 * rr, bnxt[rr]);
      bp += g.nn;
    }
    const double* sc = stage_of(i);
    double a0[CPT], a1[CPT];
#pragma unroll
    for (int rr = 0; rr < CPT; ++rr) {
      double acc0 = bcur[rr][0], acc1 = bcur[rr][1];
      const double* pc = sc + own + 64 * rr;
      double jm[2], jp[2];
      lds16<double, 2>(pc - n, jm);
      lds16<double, 2>(pc + n, jp);
      const double xl = sc[offl[rr]], xr = sc[offr[rr]];
      acc0 = __dsub_rn(acc0, __dmul_rn(c0, xm[rr][0]));
      acc1 = __dsub_rn(acc1, __dmul_rn(c0, xm[rr][1]));
      acc0 = __dsub_rn(acc0, __dmul_rn(c1, jm[0]));
      acc1 = __dsub_rn(acc1, __dmul_rn(c1, jm[1]));
      acc0 = __dsub_rn(acc0, __dmul_rn(c2, xl));
      acc1 = __dsub_rn(acc1, __dmul_rn(c2, xc[rr][0]));
      acc0 = __dsub_rn(acc0, __dmul_rn(c3, xc[rr][0]));
      acc1 = __dsub_rn(acc1, __dmul_rn(c3, xc[rr][1]));
      acc0 = __dsub_rn(acc0, __dmul_rn(c4, xc[rr][1]));
      acc1 = __dsub_rn(acc1, __dmul_rn(c4, xr));
      acc0 = __dsub_rn(acc0, __dmul_rn(c5, jp[0]));
      acc1 = __dsub_rn(acc1, __dmul_rn(c5, jp[1]));
      bcur[rr][0] = acc0;
      bcur[rr][1] = acc1;
    }
    release(i);  // plane i's stage is read no more (its own points live in xc)
    // the thread's own points of plane i+1: the last operand, and next plane's centre
    if (i < n - 1) {
      wait_full(i + 1);
      const double* sp = stage_of(i + 1) + own;
#pragma unroll
      for (int rr = 0; rr < CPT; ++rr) lds16<double, 2>(sp + 64 * rr, xn[rr]);
    } else {
#pragma unroll
      for (int rr = 0; rr < CPT; ++rr) xn[rr][0] = xn[rr][1] = copysign(0.0, c6);
    }
#pragma unroll
    for (int rr = 0; rr < CPT; ++rr) {
      const double acc0 = __dsub_rn(bcur[rr][0], __dmul_rn(c6, xn[rr][0]));
      const double acc1 = __dsub_rn(bcur[rr][1], __dmul_rn(c6, xn[rr][1]));
      // max|s| over the non-NaN entries (a NaN compares false and is skipped)
      const double f0 = fabs(acc0), f1 = fabs(acc1);
      mloc = f0 > mloc ? f0 : mloc;
      mloc = f1 > mloc ? f1 : mloc;
      // squares of s 2^-ns (nsc = 1: exact, the unscaled squares)
      const double v0 = __dmul_rn(acc0, nsc), v1 = __dmul_rn(acc1, nsc);
      a1[rr] = __dadd_rn(__dmul_rn(v0, v0), __dmul_rn(v1, v1));
      if constexpr (TWO) {
        // rhat = round(s 2^-ep) (solver.cpp:86-92) and its squares (scaled by 2^-ns_r)
        const double p2 = pol.p2;
        O o[2];
        if (pol.ep >= -1000 && pol.ep <= 1000) {  // p2 = 2^-ep is a normal double (1.0 for ep = 0)
          o[0] = from_dbl<O>(__dmul_rn(acc0, p2));
          o[1] = from_dbl<O>(__dmul_rn(acc1, p2));
        } else {
          o[0] = from_dbl<O>(scalbn(acc0, -pol.ep));
          o[1] = from_dbl<O>(scalbn(acc1, -pol.ep));
        }
        const double w0 = __dmul_rn(to_dbl(o[0]), pol.nsc_r), w1 = __dmul_rn(to_dbl(o[1]), pol.nsc_r);
        a0[rr] = __dadd_rn(__dmul_rn(w0, w0), __dmul_rn(w1, w1));
        st2(op + 64 * rr, o[0], o[1]);
      } else {
        a0[rr] = 0.0;
        if (op) st2(op + 64 * rr, acc0, acc1);
      }
    }
    if (op) op += g.nn;
    if constexpr (TWO) {
      const double t = warp_tree2_cpt<CPT>(a0, a1);
      if (lane == 0) plb[(i - ib) * nw + warp] = t;
      if (lane == 1) plb1[(i - ib) * nw + warp] = t;
    } else {
      const double t = warp_tree_cpt<CPT>(a1);
      if (lane == 0) plb[(i - ib) * nw + warp] = t;
    }
  };
  for (int i = ib; i < ie; i += 3) {
    step(i, xa, xb, xc_, ba, bb);
    if (i + 1 < ie) step(i + 1, xb, xc_, xa, bb, bc);
    if (i + 2 < ie) step(i + 2, xc_, xa, xb, bc, ba);
  }
  st25_finish(pol, g, rd, st, plb, nw, ib, jt, mloc, 0, TWO ? plb1 : plb);
}

// ------------------------------------------------ packed zero-start residual

template <class Op>
__global__ void __launch_bounds__(256) k_gm_resid0p(Op op, const __half* __restrict__ src, __half* __restrict__ r,
                                                    Geo g, Red rd, DevState* st, int scale, uint32_t p2bits) {
  using C = float;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int nf = 0;
#pragma unroll
  for (int i = 0; i < 7; ++i) nf |= op.zc[i];
  nf &= 2;  // a non-finite coefficient: every row takes the general rule
  const __half2 p2 = *reinterpret_cast<const __half2*>(&p2bits);
  uint4 v[RMAX];
#pragma unroll
  for (int q = 0; q < RMAX; ++q)
    if (q < g.R) {
      const int64_t t = (((int64_t)blockIdx.x * g.W + warp) * g.R + q) * g.L + lane;
      v[q] = __ldg(reinterpret_cast<const uint4*>(src) + t);
    }
  C a0[RMAX];
  double a1[RMAX];
  int bad = 0;
#pragma unroll
  for (int q = 0; q < RMAX; ++q) {
    if (q < g.R) {
      const int64_t t = (((int64_t)blockIdx.x * g.W + warp) * g.R + q) * g.L + lane;
      uint32_t w[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
      if (scale) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const __half2 pr = __hmul2(*reinterpret_cast<const __half2*>(&w[k]), p2);
          w[k] = *reinterpret_cast<const uint32_t*>(&pr);
        }
      }
      uint32_t sp = (uint32_t)nf;
#pragma unroll
      for (int k = 0; k < 4; ++k) sp |= any_half_eq(w[k], 0x80008000u);
      if (sp) {  // rare: a -0 entry (or a non-finite coefficient): the zero-start sign rules
        int fl[8];
        op.template zflags_vec<8>(t * 8, fl);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          __half2 h = *reinterpret_cast<const __half2*>(&w[k]);
          const __half lo = st_t<__half, C>(zero_resid(__half2float(__low2half(h)), fl[2 * k]));
          const __half hi = st_t<__half, C>(zero_resid(__half2float(__high2half(h)), fl[2 * k + 1]));
          h = __halves2half2(lo, hi);
          w[k] = *reinterpret_cast<const uint32_t*>(&h);
        }
      }
      C tc[8];
      double td[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        tc[2 * k] = fhf<0, 0>(w[k], w[k], -0.0f);  // exact squares
        tc[2 * k + 1] = fhf<1, 1>(w[k], w[k], -0.0f);
        td[2 * k] = (double)tc[2 * k];
        td[2 * k + 1] = (double)tc[2 * k + 1];
      }
      reinterpret_cast<uint4*>(r)[t] = make_uint4(w[0], w[1], w[2], w[3]);
      const C c = seg_sum<C, 8>(tc, 8);
      const double d = seg_sum<double, 8>(td, 8);
      bad |= isfinite(c) ? 0 : 1;
      a0[q] = warp_tree(c, g.L);
      a1[q] = warp_tree(d, g.L);
    }
  }
#pragma unroll
  for (int s2 = 1; s2 < RMAX; s2 <<= 1)
#pragma unroll
    for (int q = 0; q + s2 < RMAX; q += 2 * s2)
      if (q + s2 < g.R) {
        a0[q] = __fadd_rn(a0[q], a0[q + s2]);
        a1[q] = __dadd_rn(a1[q], a1[q + s2]);
      }
  or_flags(&st->flags, bad);
  C dc;
  double ss;
  if (grid_finish(a0[0], a1[0], g, rd, dc, ss)) finish_red(EpiResidF{}, st, dc, ss);
}

}  // namespace gadi
