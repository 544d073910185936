// gadi_kernels.cuh — the device kernels of the GADI-IR hot path.
//
// Work decomposition. The N vector entries are cut into 2^D reduction
// segments (gadi_common.cuh). A lane owns R segments that are 32 apart, so a
// warp's loads at each step are one contiguous 512-byte run (VEC*sizeof(T)
// == 16 bytes per lane); the warp folds its R x 32 contiguous segments into
// one pairwise partial (butterfly per step, then a tree over the R steps), a
// block folds its W warps, and the last block to finish folds the block
// partials. Every level is a perfect binary tree over contiguous ranges, so
// the result is the reference's pairwise sum (kernels.cpp:33-39) bit for bit.
//
// Every kernel that produces a dot product or norm folds it into the pass
// that writes the vector (SpMV + p.Ap with p = r + beta p formed on the fly;
// both CG axpys + r.r + ||r||_2; GMRES MGS axpy + the next Arnoldi dot), and
// the last block evaluates the scalar recurrences (alpha, beta, stop tests)
// on the device: the host never waits inside a CG solve.
//
// Template parameters: Op (Stencil7 / Csr), T (storage: __half, float,
// double), C (arithmetic: T, or float for binary16 storage with binary32
// accumulation), VEC (elements per segment on the aligned path; 1 = general).
#pragma once

#include "gadi_common.cuh"
#include "gadi_ops.cuh"

namespace gadi {

constexpr int RMAX = 8;  // segments per lane (unrolled)
#define GADI_MAX_RANKS 64

struct Geo {
  int64_t N;
  int D;     // 2^D segments
  int L;     // lanes per warp chunk (32, or 2^D when smaller)
  int W;     // warps per block
  int R;     // segments per lane
  int nblk;  // blocks; nblk * W * R * L == 2^D
  int64_t gh = 0;  // ghost entries on each side of the operand (a sharded CSR row block)
  __host__ __device__ int threads() const { return L * W; }
};

constexpr int GM_SPEC_MAX = 8;  // Arnoldi steps queued per host sync

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
  int cg_xvalid;
  unsigned long long maxbits;
  // speculative Arnoldi windows (fused mode): 1 / h(j+1, j) (or 1 / beta) for the next step's
  // basis scaling, formed on the device
  double gm_inv;
  // outer loop
  double res_ss, res_max, rhat_ss;
  int res_e, xbad;
  int* hdone;  // mapped host flag raised when a CG solve finishes
  // sharded solves (gadi_dist.cuh): this rank's subtree sums + flag/max
  // words, parked by a reduction's last block; all ranks' copies, gathered
  // Both are double-buffered by collective parity (dist_par, toggled by
  // k_dist_finish): a peer may still be pulling record c while this rank's
  // next reduction writes record c+1.
  int dist, dist_par;
  // ---- the head above is what read_state copies; the arrays below only on request
  // GMRES Arnoldi column, h(0..j+1, j), and the columns of the steps of a speculative window
  double hcol[72];
  double hhist[GM_SPEC_MAX][72];
  double ycoef[72];
  double dist_loc[2][4];
  double dist_all[2][4 * GADI_MAX_RANKS];
};

enum : int { INNER_CONVERGED = 0, INNER_STAGNATED = 1, INNER_OVERFLOW = 2 };

// host_it: the host loop iteration whose kernels decided (-1: the init pass).
// The mapped flag carries host_it + 2, so a sharded solve's ranks can all stop
// queueing at the same iteration (Engine::cg).
__device__ __forceinline__ void cg_finish(DevState* st, int status, int iters, int host_it) {
  st->cg_done = 1;
  st->cg_status = status;
  st->cg_iters = iters;
  if (st->hdone) {
    *(volatile int*)st->hdone = host_it + 2;
    __threadfence_system();
  }
}

// ------------------------------------------------------------ epilogues
// A reduction's scalar epilogue (the recurrences / stop tests that follow a
// dot or norm in the reference) is an object with finish(t0, t1, st) and
// flag_dst(st). On one device the last block applies it directly. In a
// sharded solve (st->dist) the last block parks the rank's subtree sums and
// its flag / max words in st->dist_loc; the host all-gathers them and
// k_dist_finish folds the ranks' values in rank order -- the slabs are
// aligned power-of-two blocks of the pairwise tree, so this is the
// single-device value bit for bit -- and applies the same epilogue.
template <class Epi, class C0>
__device__ __forceinline__ void finish_red(const Epi& epi, DevState* st, C0 t0, double t1) {
  if (st->dist) {
    int* f = epi.flag_dst(st);
    double* rec = st->dist_loc[st->dist_par];
    rec[0] = to_dbl(t0);
    rec[1] = t1;
    rec[2] = f ? (double)*(volatile int*)f : 0.0;
    rec[3] = __longlong_as_double((long long)*(volatile unsigned long long*)&st->maxbits);
  } else {
    epi.finish(t0, t1, st);
  }
}

// the flag / max words alone (kernels without a grid reduction)
static __global__ void k_dist_pack(DevState* st, int* flags) {
  double* rec = st->dist_loc[st->dist_par];
  rec[0] = 0.0;
  rec[1] = 0.0;
  rec[2] = flags ? (double)*flags : 0.0;
  rec[3] = __longlong_as_double((long long)st->maxbits);
}

template <class Epi, class C0>
__global__ void k_dist_finish(const Epi epi, DevState* st, int world, int half) {
  C0 v0[GADI_MAX_RANKS];
  double v1[GADI_MAX_RANKS];
  int fl = 0;
  unsigned long long mb = 0;
  const double* all = st->dist_all[half];
  for (int r = 0; r < world; ++r) {
    v0[r] = from_dbl<C0>(all[4 * r]);
    v1[r] = all[4 * r + 1];
    fl |= (int)all[4 * r + 2];
    const unsigned long long b = (unsigned long long)__double_as_longlong(all[4 * r + 3]);
    mb = b > mb ? b : mb;
  }
  for (int s = 1; s < world; s <<= 1)  // world is a power of two
    for (int k = 0; k + s < world; k += 2 * s) {
      v0[k] = Ar<C0>::add(v0[k], v0[k + s]);
      v1[k] = __dadd_rn(v1[k], v1[k + s]);
    }
  st->dist_par = half ^ 1;
  if (epi.skip(st)) return;  // the kernel returned early (CG done): nothing was reduced
  if (int* f = epi.flag_dst(st)) *f = fl;
  st->maxbits = mb;
  epi.finish(v0[0], v1[0], st);
}

struct EpiNone {  // flags / max only
  int* flags = nullptr;
  template <class C0>
  __device__ void finish(C0, double, DevState*) const {}
  __device__ int* flag_dst(DevState*) const { return flags; }
  __device__ bool skip(DevState*) const { return false; }
};

// ------------------------------------------------------------ segment loop
// Runs body(seg, c, d) on this lane's R segments and returns the warp's
// pairwise totals of c (in C0) and d (in binary64), valid in every lane.
template <int VEC, bool R0, bool R1, class C0, class Body>
__device__ __forceinline__ void seg_run(const Geo& g, Body&& body, C0& w0, double& w1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  C0 a0[RMAX];
  double a1[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    if (r < g.R) {
      const int64_t t = (((int64_t)blockIdx.x * g.W + warp) * g.R + r) * g.L + lane;
      const Seg s = seg_of<VEC>(t, g.N, g.D);
      C0 c = Ar<C0>::zero();
      double d = 0.0;
      body(s, c, d);
      if (R0) a0[r] = warp_tree(c, g.L);
      if (R1) a1[r] = warp_tree(d, g.L);
    }
  }
#pragma unroll
  for (int st = 1; st < RMAX; st <<= 1)
#pragma unroll
    for (int r = 0; r + st < RMAX; r += 2 * st)
      if (r + st < g.R) {
        if (R0) a0[r] = Ar<C0>::add(a0[r], a0[r + st]);
        if (R1) a1[r] = __dadd_rn(a1[r], a1[r + st]);
      }
  w0 = R0 ? a0[0] : Ar<C0>::zero();
  w1 = R1 ? a1[0] : 0.0;
}

// seg_run over one input stream whose R segment loads are all issued before
// any of them is consumed (memory-level parallelism for single-stream
// reductions); body(seg, v, c, d) gets the segment's G values.
template <int VEC, bool R0, bool R1, int G, class T, class C0, class Body>
__device__ __forceinline__ void seg_run_ld(const Geo& g, const T* __restrict__ p, Body&& body, C0& w0, double& w1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T v[RMAX][G];
#pragma unroll
  for (int r = 0; r < RMAX; ++r)
    if (r < g.R) {
      const int64_t t = (((int64_t)blockIdx.x * g.W + warp) * g.R + r) * g.L + lane;
      if constexpr (VEC > 1) {
        ld_vec<T, VEC>(p, t * VEC, v[r]);
      } else {
        const Seg s = seg_of<VEC>(t, g.N, g.D);
#pragma unroll
        for (int i = 0; i < G; ++i) v[r][i] = i < s.len ? p[s.lo + i] : from_dbl<T>(0.0);
      }
    }
  C0 a0[RMAX];
  double a1[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    if (r < g.R) {
      const int64_t t = (((int64_t)blockIdx.x * g.W + warp) * g.R + r) * g.L + lane;
      C0 c = Ar<C0>::zero();
      double d = 0.0;
      body(seg_of<VEC>(t, g.N, g.D), v[r], c, d);
      if (R0) a0[r] = warp_tree(c, g.L);
      if (R1) a1[r] = warp_tree(d, g.L);
    }
  }
#pragma unroll
  for (int st = 1; st < RMAX; st <<= 1)
#pragma unroll
    for (int r = 0; r + st < RMAX; r += 2 * st)
      if (r + st < g.R) {
        if (R0) a0[r] = Ar<C0>::add(a0[r], a0[r + st]);
        if (R1) a1[r] = __dadd_rn(a1[r], a1[r + st]);
      }
  w0 = R0 ? a0[0] : Ar<C0>::zero();
  w1 = R1 ? a1[0] : 0.0;
}

// Elementwise loop over this lane's segments (no reduction).
template <int VEC, class Body>
__device__ __forceinline__ void seg_each(const Geo& g, Body&& body) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < RMAX; ++r)
    if (r < g.R) {
      const int64_t t = (((int64_t)blockIdx.x * g.W + warp) * g.R + r) * g.L + lane;
      body(seg_of<VEC>(t, g.N, g.D));
    }
}

// Fold the warp totals over the block and the grid. Returns true in exactly
// one thread (thread 0 of the last block), which then holds the grid totals.
// Every thread of every block must call it.
template <class C0>
__device__ __forceinline__ bool grid_finish(C0 w0, double w1, const Geo& g, const Red& r, C0& t0, double& t1) {
  __shared__ __align__(8) unsigned char smb0[32 * sizeof(double)];
  __shared__ double sm1[32];
  __shared__ int last;
  C0* sm0 = reinterpret_cast<C0*>(smb0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (g.W > 1) {
    if (lane == 0) {
      sm0[warp] = w0;
      sm1[warp] = w1;
    }
    __syncthreads();
    if (warp == 0) {
      C0 v0 = lane < g.W ? sm0[lane] : Ar<C0>::zero();
      double v1 = lane < g.W ? sm1[lane] : 0.0;
      if (lane < g.W) {
        v0 = warp_tree(v0, g.W);
        v1 = warp_tree(v1, g.W);
      }
      w0 = v0;
      w1 = v1;
    }
  }
  if (tid == 0) {
    r.part0[blockIdx.x] = to_dbl(w0);
    r.part1[blockIdx.x] = w1;
    __threadfence();
    const unsigned t = atomicAdd(r.ticket, 1u);
    last = (t == (unsigned)g.nblk - 1u);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  const int P = g.nblk, B = blockDim.x;
  C0 a0;
  double a1;
  int cnt;
  if (P <= B) {
    a0 = tid < P ? from_dbl<C0>(__ldcg(r.part0 + tid)) : Ar<C0>::zero();
    a1 = tid < P ? __ldcg(r.part1 + tid) : 0.0;
    cnt = P;
  } else {
    const int64_t Lr = P / B;
    const double* p0 = r.part0 + (int64_t)tid * Lr;
    const double* p1 = r.part1 + (int64_t)tid * Lr;
    a0 = run_pairwise<C0>(Lr, [&](int64_t j) { return from_dbl<C0>(__ldcg(p0 + j)); });
    a1 = run_pairwise<double>(Lr, [&](int64_t j) { return __ldcg(p1 + j); });
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
// element by element. `cc` returns the operand at the segment's points.
template <int VEC, int G, class Op, class Src, class X, class Acc, class F>
__device__ __forceinline__ void fold_seg(const Op& op, const Src& x, const Seg& s, Acc (&acc)[G], F f,
                                         X (&cc)[G]) {
  if constexpr (VEC > 1) {
    op.template fold<VEC>(x, s.lo, acc, f, cc);
  } else {
#pragma unroll
    for (int i = 0; i < G; ++i) {
      if (i < s.len) {
        Acc a1[1] = {acc[i]};
        X c1[1];
        op.template fold<1>(x, s.lo + i, a1, f, c1);
        acc[i] = a1[0];
        cc[i] = c1[0];
      } else {
        cc[i] = from_dbl<X>(0.0);
      }
    }
  }
}

// Rows a block covers on the aligned path (seg_run's contiguous W*R*L segments).
template <int VEC>
__device__ __forceinline__ int64_t block_rows(const Geo& g) {
  return (int64_t)g.W * g.R * g.L * VEC;
}

// Stage x[block rows +- band] in dynamic shared memory (banded sparse operators).
template <class T, int VEC>
__device__ __forceinline__ SmemSrc<T> stage_window(const T* __restrict__ x, const Geo& g, int64_t band) {
  extern __shared__ __align__(16) unsigned char gadi_wsm[];
  T* w = reinterpret_cast<T*>(gadi_wsm);
  const int64_t BR = block_rows<VEC>(g), r0 = (int64_t)blockIdx.x * BR;
  int64_t lo = r0 - band;  // ghosts (g.gh, a multiple of 8) are part of the operand
  lo = lo < -g.gh ? -g.gh : (lo & ~(int64_t)(VEC - 1));
  int64_t hi = r0 + BR + band;
  hi = hi > g.N + g.gh ? g.N + g.gh : hi;
  const int64_t len = hi - lo;
  for (int64_t i = (int64_t)threadIdx.x * VEC; i < len; i += (int64_t)blockDim.x * VEC) {
    if (VEC * sizeof(T) == 16 && i + VEC <= len) {
      *reinterpret_cast<uint4*>(w + i) = __ldg(reinterpret_cast<const uint4*>(x + lo + i));
    } else {
      for (int k = 0; k < VEC && i + k < len; ++k) w[i + k] = x[lo + i + k];
    }
  }
  __syncthreads();
  return SmemSrc<T>{w, lo};
}

// acc + a * b for binary16 a, b in binary32 arithmetic, one instruction
// (FHFMA, sm_100): the product of two binary16 values is exact in binary32
// (11 + 11 <= 24 significand bits, exponents in range), so the single
// rounding of the fused op IS the reference's round(acc + round(a * b)) --
// the same bits as __fadd_rn(acc, __fmul_rn(a, b)), signed zeros included.
__device__ __forceinline__ float fhfma(__half a, __half b, float c) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(__half_as_ushort(a)), "h"(__half_as_ushort(b)), "f"(c));
  return d;
}

template <int SA, int SB>  // SA / SB: which half (0 low, 1 high) of a / b
__device__ __forceinline__ float fhf(uint32_t a, uint32_t b, float c) {
  float d;
  if constexpr (SA == 0 && SB == 0)
    asm("{.reg .f16 al, ah, bl, bh; mov.b32 {al, ah}, %1; mov.b32 {bl, bh}, %2; fma.rn.f32.f16 %0, al, bl, %3;}"
        : "=f"(d) : "r"(a), "r"(b), "f"(c));
  else if constexpr (SA == 0 && SB == 1)
    asm("{.reg .f16 al, ah, bl, bh; mov.b32 {al, ah}, %1; mov.b32 {bl, bh}, %2; fma.rn.f32.f16 %0, al, bh, %3;}"
        : "=f"(d) : "r"(a), "r"(b), "f"(c));
  else if constexpr (SA == 1 && SB == 0)
    asm("{.reg .f16 al, ah, bl, bh; mov.b32 {al, ah}, %1; mov.b32 {bl, bh}, %2; fma.rn.f32.f16 %0, ah, bl, %3;}"
        : "=f"(d) : "r"(a), "r"(b), "f"(c));
  else
    asm("{.reg .f16 al, ah, bl, bh; mov.b32 {al, ah}, %1; mov.b32 {bl, bh}, %2; fma.rn.f32.f16 %0, ah, bh, %3;}"
        : "=f"(d) : "r"(a), "r"(b), "f"(c));
  return d;
}
// nonzero iff one of the two binary16 halves of w equals the pattern's half (pat2 = pat | pat << 16)
__device__ __forceinline__ uint32_t any_half_eq(uint32_t w, uint32_t pat2) {
  const uint32_t t = w ^ pat2;
  return (t - 0x00010001u) & ~t & 0x80008000u;
}
template <class C, class T>
struct MatvecF {  // acc + coef * x (kernels.cpp:47-52)
  // PACKED: binary32 folds may pair the products (FMUL2, fold_vec in
  // gadi_st25.cuh) but keep the adds scalar: ptxas (CUDA 12.9) contracts
  // mul.rn.f32x2 + add.rn.f32x2 into one FFMA2 (a single rounding) despite
  // .rn and -fmad=false, which would break the reference's two-rounding fold;
  // FMUL2 + scalar FADD is never contracted (checked in the SASS).
  // EXACT_H: binary16 operands in binary32 arithmetic. The coefficients are
  // u_r = binary16 values too (rounded_copy, inner_solver.cpp:41-45), so each
  // product is exact and the fold is one FHFMA per entry (see fhfma).
  static constexpr bool EXACT_H = std::is_same<C, float>::value && std::is_same<T, __half>::value;
  static constexpr bool PACKED = std::is_same<C, float>::value && !EXACT_H, NEG = false;
  __device__ __forceinline__ C operator()(C a, C coef, T xv) const {
    if constexpr (EXACT_H) return fhfma(__float2half_rn(coef), xv, a);
    else return Ar<C>::add(a, Ar<C>::mul(coef, ld_c<T, C>(xv)));
  }
};
template <class C, class T>
struct ResidF {  // acc - coef * x (kernels.cpp:63-66)
  // EXACT_H: acc - c x = round(acc + (-c) x), -c exact (see MatvecF)
  static constexpr bool EXACT_H = std::is_same<C, float>::value && std::is_same<T, __half>::value;
  static constexpr bool PACKED = std::is_same<C, float>::value && !EXACT_H, NEG = true;
  __device__ __forceinline__ C operator()(C a, C coef, T xv) const {
    if constexpr (EXACT_H) return fhfma(__float2half_rn(-coef), xv, a);
    else return Ar<C>::sub(a, Ar<C>::mul(coef, ld_c<T, C>(xv)));
  }
};
template <int P>
struct ResidAF {  // binary64-carried residual rounded to u_f per op
  static constexpr bool PACKED = false, NEG = false;
  __device__ __forceinline__ double operator()(double a, double coef, double xv) const {
    return round_p<P>(__dsub_rn(a, round_p<P>(__dmul_rn(coef, xv))));
  }
};
struct MatvecAF {  // b = A x in binary64 (problems.cpp:44)
  static constexpr bool PACKED = false, NEG = false;
  __device__ __forceinline__ double operator()(double a, double coef, double xv) const {
    return __dadd_rn(a, __dmul_rn(coef, xv));
  }
};

#define GADI_G constexpr int G = VEC > 1 ? VEC : 4
#define GADI_LIVE(i) (VEC > 1 || (i) < s.len)

// ================================================================== CG
struct EpiCgInit {  // inner_solver.cpp:51-57
  int max_inner;
  double target;
  int known;  // 1: ||r||^2 (binary64) is st->rhat_ss, reduced by the outer pass that produced r = rhat
  template <class C>
  __device__ void finish(C rs, double ss, DevState* st) const {
    st->red_d = ss;  // the sum this pass reduced (GADI_CHECK_SS compares it with rhat_ss)
    if (known) ss = st->rhat_ss;
    st->cg_rs = to_dbl(rs);
    st->cg_it = 0;
    st->cg_flags = 0;
    st->cg_xvalid = 0;
    st->cg_max = max_inner;
    st->cg_target = target;
    st->cg_done = 0;
    if (max_inner <= 0) cg_finish(st, INNER_STAGNATED, 0, -1);
    else if (sqrt(ss) <= target) cg_finish(st, INNER_CONVERGED, 0, -1);
  }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ bool skip(DevState* st) const { return (void)st, false; }
};
struct EpiCgPap {  // alpha = rs / pap, or `break` (inner_solver.cpp:62-65)
  template <class C>
  __device__ void finish(C pap, double, DevState* st) const {
    const double pd = to_dbl(pap);
    st->cg_pap = pd;
    if (pd == 0.0 || !isfinite(pd)) {
      // `break` -> Stagnated / Overflow with iters = max (:64, :79-81)
      cg_finish(st, (st->cg_flags & 2) ? INNER_OVERFLOW : INNER_STAGNATED, st->cg_max, st->cg_it);
    } else {
      st->cg_a = to_dbl(div_c<C>(from_dbl<C>(st->cg_rs), pap));
    }
  }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ bool skip(DevState* st) const { return *(volatile int*)&st->cg_done != 0; }
};
struct EpiCgUpdate {  // beta, the overflow / max-iteration / residual stop tests (inner_solver.cpp:66-77)
  template <class C>
  __device__ void finish(C rsn, double ss, DevState* st) const {
    const int it = st->cg_it;
    const double rn = to_dbl(rsn);
    const int flags = *(volatile int*)&st->cg_flags;
    st->cg_xvalid = 1;
    if (!isfinite(rn) || (flags & 1)) {
      cg_finish(st, INNER_OVERFLOW, it + 1, it);
    } else {
      st->cg_beta = to_dbl(div_c<C>(rsn, from_dbl<C>(st->cg_rs)));
      st->cg_rs = rn;
      st->cg_it = it + 1;
      if (it + 1 >= st->cg_max) cg_finish(st, (flags & 2) ? INNER_OVERFLOW : INNER_STAGNATED, st->cg_max, it);
      else if (sqrt(ss) <= st->cg_target) cg_finish(st, INNER_CONVERGED, it + 1, it);
    }
  }
  __device__ int* flag_dst(DevState* st) const { return &st->cg_flags; }
  __device__ bool skip(DevState* st) const { return *(volatile int*)&st->cg_done != 0; }
};
struct EpiRedD {  // ||r||_2 of a GMRES restart residual (+ flags, max)
  template <class C>
  __device__ void finish(C, double ss, DevState* st) const { st->red_d = ss; }
  __device__ int* flag_dst(DevState* st) const { return &st->flags; }
  __device__ bool skip(DevState* st) const { return (void)st, false; }
};
struct EpiHcol {  // an Arnoldi coefficient h(i, j)
  int i;
  template <class C>
  __device__ void finish(C h, double, DevState* st) const { st->hcol[i] = to_dbl(h); }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ bool skip(DevState* st) const { return (void)st, false; }
};

// r = rhs (in place), rs = dot(r, r) and the initial stop test
// (inner_solver.cpp:51-57). x and p are produced by the first iteration.
// DBL = false: the binary64 ||r||^2 of the stop test is already known (r is the rhat an outer
// residual pass just produced and reduced over the same tree: st->rhat_ss), so only the
// inner-format dot is reduced -- no binary64 conversions, adds or second tree.
template <class T, class C, int VEC, bool DBL = true>
__global__ void __launch_bounds__(256) k_cg_init(const T* __restrict__ r, int max_inner, double target, Geo g,
                                                 Red rd, DevState* st) {
  GADI_G;
  C w0;
  double w1;
  seg_run_ld<VEC, true, DBL, G>(g, r, [&](const Seg& s, const T (&v)[G], C& c, double& d) {
    C tc[G];
    double td[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      if constexpr (MatvecF<C, T>::EXACT_H) {  // the square of a binary16 value is exact in binary32
        tc[i] = fhfma(v[i], v[i], -0.0f);
        if (DBL) td[i] = (double)tc[i];
      } else {
        const C cv = ld_c<T, C>(v[i]);
        tc[i] = Ar<C>::mul(cv, cv);
        if (DBL) {
          const double dv = to_dbl(v[i]);
          td[i] = __dmul_rn(dv, dv);
        }
      }
    }
    c = seg_sum<C, G>(tc, s.len);
    if (DBL) d = seg_sum<double, G>(td, s.len);
  }, w0, w1);
  C rs;
  double ss;
  if (grid_finish(w0, w1, g, rd, rs, ss)) finish_red(EpiCgInit{max_inner, target, DBL ? 0 : 1}, st, rs, ss);
}

// p_out = r + beta p_in (or r on the first iteration; inner_solver.cpp:53,76),
// q = H p_out, pap = dot(p_out, q); then alpha = rs / pap or `break`
// (inner_solver.cpp:62-65).
// FUSE = false (sparse operators, where a gathered operand would be re-formed
// per nonzero): p_in already holds the updated p (k_cg_pupd) and is only read.
template <class Op, class T, class C, int VEC, bool FUSE = true>
__global__ void __launch_bounds__(256) k_cg_spmvp(Op op, const T* __restrict__ r, const T* __restrict__ p_in,
                                                  T* __restrict__ p_out, T* __restrict__ q, int first, Geo g,
                                                  Red rd, DevState* st, int64_t wband = 0) {
  if (*(volatile int*)&st->cg_done) return;
  GADI_G;
  C w0;
  double w1;
  auto body = [&](const Seg& s, C& c, const auto& src) {
    C acc[G];
    T pv[G], qv[G];
#pragma unroll
    for (int i = 0; i < G; ++i) acc[i] = Ar<C>::zero();
    fold_seg<VEC, G>(op, src, s, acc, MatvecF<C, T>(), pv);
    C tc[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      qv[i] = st_t<T, C>(acc[i]);
      tc[i] = Ar<C>::mul(ld_c<T, C>(pv[i]), ld_c<T, C>(qv[i]));
    }
    store_seg<T, VEC, G>(q, s, qv);
    if (FUSE) store_seg<T, VEC, G>(p_out, s, pv);
    c = seg_sum<C, G>(tc, s.len);
  };
  if constexpr (FUSE) {
    const PUpdSrc<T, C> src{r, p_in, from_dbl<C>(st->cg_beta), first};
    seg_run<VEC, true, false>(g, [&](const Seg& s, C& c, double&) { body(s, c, src); }, w0, w1);
  } else if (VEC > 1 && wband > 0) {
    const SmemSrc<T> src = stage_window<T, VEC>(p_in, g, wband);
    seg_run<VEC, true, false>(g, [&](const Seg& s, C& c, double&) { body(s, c, src); }, w0, w1);
  } else {
    const PlainSrc<T> src{p_in};
    seg_run<VEC, true, false>(g, [&](const Seg& s, C& c, double&) { body(s, c, src); }, w0, w1);
  }
  C pap;
  double dummy;
  if (grid_finish(w0, w1, g, rd, pap, dummy)) finish_red(EpiCgPap{}, st, pap, dummy);
}

// p_out = r + beta p_in, or r on the first iteration (inner_solver.cpp:53,76);
// the separate pass used with sparse operators.
template <class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_cg_pupd(const T* __restrict__ r, const T* __restrict__ p_in,
                                                 T* __restrict__ p_out, int first, Geo g, DevState* st) {
  if (*(volatile int*)&st->cg_done) return;
  GADI_G;
  const PUpdSrc<T, C> src{r, p_in, from_dbl<C>(st->cg_beta), first};
  seg_each<VEC>(g, [&](const Seg& s) {
    T v[G];
    if constexpr (VEC > 1) {
      src.template vec<VEC>(s.lo, v);
    } else {
#pragma unroll
      for (int i = 0; i < G; ++i) v[i] = i < s.len ? src.at(s.lo + i) : from_dbl<T>(0.0);
    }
    store_seg<T, VEC, G>(p_out, s, v);
  });
}

// x += a p (x = 0 + a p on the first iteration); r -= a q; rs' = dot(r, r);
// ||r||_2 in binary64 for the next stop test; overflow checks
// (inner_solver.cpp:66-77).
template <class T, class C, int VEC>
__global__ void __launch_bounds__(256, 4) k_cg_update(T* __restrict__ x, T* __restrict__ r, const T* __restrict__ p,
                                                   const T* __restrict__ q, int first, Geo g, Red rd,
                                                   DevState* st, int keep_r = 1) {
  // keep_r = 0: the solve ends with this iteration whatever the stop test says (it is
  // iteration max_inner), and nothing reads the residual vector afterwards: r is reduced, not stored
  if (*(volatile int*)&st->cg_done) return;
  GADI_G;
  const C a = from_dbl<C>(st->cg_a);
  const C na = Ar<C>::neg(a);
  int bad = 0;
  C w0;
  double w1;
  if constexpr (VEC == 8 && MatvecF<C, T>::EXACT_H) {
    // binary16 storage, binary32 arithmetic: the chunks stay packed (two lanes per FMUL2 / F2FP,
    // squares as FHFMA onto -0, finiteness from one bit test per word); the same operations per
    // element and the same trees as the generic body below
    const float2 a2 = make_float2(a, a), na2 = make_float2(na, na);
    seg_run<VEC, true, true>(g, [&](const Seg& s, C& c, double& d) {
      const int64_t ch = s.lo >> 3;
      uint4 xu = make_uint4(0, 0, 0, 0);
      if (!first) xu = reinterpret_cast<const uint4*>(x)[ch];
      const uint4 ru = reinterpret_cast<const uint4*>(r)[ch];
      const uint4 pu = __ldg(reinterpret_cast<const uint4*>(p) + ch);
      const uint4 qu = __ldg(reinterpret_cast<const uint4*>(q) + ch);
      const uint32_t xw[4] = {xu.x, xu.y, xu.z, xu.w}, rw[4] = {ru.x, ru.y, ru.z, ru.w};
      const uint32_t pw[4] = {pu.x, pu.y, pu.z, pu.w}, qw[4] = {qu.x, qu.y, qu.z, qu.w};
      uint32_t xo[4], ro[4], infs = 0;
      float tc[8];
      double td[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 xf = first ? make_float2(0.0f, 0.0f) : __half22float2(*reinterpret_cast<const __half2*>(&xw[k]));
        const float2 ap = __fmul2_rn(a2, __half22float2(*reinterpret_cast<const __half2*>(&pw[k])));
        const __half2 xn = __floats2half2_rn(__fadd_rn(xf.x, ap.x), __fadd_rn(xf.y, ap.y));
        xo[k] = *reinterpret_cast<const uint32_t*>(&xn);
        const float2 rf = __half22float2(*reinterpret_cast<const __half2*>(&rw[k]));
        const float2 aq = __fmul2_rn(na2, __half22float2(*reinterpret_cast<const __half2*>(&qw[k])));
        const __half2 rn = __floats2half2_rn(__fadd_rn(rf.x, aq.x), __fadd_rn(rf.y, aq.y));
        ro[k] = *reinterpret_cast<const uint32_t*>(&rn);
        tc[2 * k] = fhf<0, 0>(ro[k], ro[k], -0.0f);
        tc[2 * k + 1] = fhf<1, 1>(ro[k], ro[k], -0.0f);
        td[2 * k] = (double)tc[2 * k];
        td[2 * k + 1] = (double)tc[2 * k + 1];
        // an exponent field of all ones: r -> bit 0, x -> bit 1 of `bad`
        infs |= (any_half_eq(ro[k] & 0x7c007c00u, 0x7c007c00u) ? 1u : 0u) |
                (any_half_eq(xo[k] & 0x7c007c00u, 0x7c007c00u) ? 2u : 0u);
      }
      reinterpret_cast<uint4*>(x)[ch] = make_uint4(xo[0], xo[1], xo[2], xo[3]);
      if (keep_r) reinterpret_cast<uint4*>(r)[ch] = make_uint4(ro[0], ro[1], ro[2], ro[3]);
      bad |= (int)infs;
      c = seg_sum<C, G>(tc, G);
      d = seg_sum<double, G>(td, G);
    }, w0, w1);
  } else
  seg_run<VEC, true, true>(g, [&](const Seg& s, C& c, double& d) {
    T xv[G], rv[G], pv[G], qv[G];
    if (!first) load_seg<T, VEC, G>(x, s, xv);
    load_seg<T, VEC, G>(r, s, rv);
    load_seg<T, VEC, G>(p, s, pv);
    load_seg<T, VEC, G>(q, s, qv);
    C tc[G];
    double td[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const C x0 = first ? Ar<C>::zero() : ld_c<T, C>(xv[i]);
      xv[i] = st_t<T, C>(Ar<C>::add(x0, Ar<C>::mul(a, ld_c<T, C>(pv[i]))));
      rv[i] = st_t<T, C>(Ar<C>::add(ld_c<T, C>(rv[i]), Ar<C>::mul(na, ld_c<T, C>(qv[i]))));
      if constexpr (MatvecF<C, T>::EXACT_H) {  // exact binary16 squares; finiteness from the bits
        tc[i] = fhfma(rv[i], rv[i], -0.0f);
        td[i] = (double)tc[i];
        if (GADI_LIVE(i))
          bad |= ((__half_as_ushort(rv[i]) & 0x7c00u) == 0x7c00u ? 1 : 0) |
                 ((__half_as_ushort(xv[i]) & 0x7c00u) == 0x7c00u ? 2 : 0);
      } else {
        const C rc = ld_c<T, C>(rv[i]);
        tc[i] = Ar<C>::mul(rc, rc);
        const double dv = to_dbl(rv[i]);
        td[i] = __dmul_rn(dv, dv);
        if (GADI_LIVE(i)) bad |= (finite_t(rv[i]) ? 0 : 1) | (finite_t(xv[i]) ? 0 : 2);
      }
    }
    store_seg<T, VEC, G>(x, s, xv);
    if (keep_r) store_seg<T, VEC, G>(r, s, rv);
    c = seg_sum<C, G>(tc, s.len);
    d = seg_sum<double, G>(td, s.len);
  }, w0, w1);
  or_flags(&st->cg_flags, bad);
  C rsn;
  double ss;
  if (grid_finish(w0, w1, g, rd, rsn, ss)) finish_red(EpiCgUpdate{}, st, rsn, ss);
}

// ================================================================ GMRES
// acc - c_1*0 - c_2*0 - ... in the row's stored order, from the row's zflag
// summary alone: coef*0 is +0, -0 (sign bit set) or NaN (coef not finite);
// subtracting +-0 leaves a nonzero acc unchanged, turns -0 into +0 once any
// -0 is subtracted, and a NaN term gives the canonical NaN. Bitwise the same
// as the fold over x = 0 without reading the matrix.
template <class C>
__device__ __forceinline__ C zero_resid(C acc, int f) {
  const C z = Ar<C>::zero();
  if (f & 2) return Ar<C>::sub(acc, Ar<C>::mul(Ar<C>::from_d(INFINITY), z));
  if (f & 1) return Ar<C>::sub(acc, Ar<C>::neg(z));
  return acc;
}

// r = rhs - S x in the inner arithmetic (inner_solver.cpp:97 / :182, the
// two-stage residual kernels.cpp:56-69; x_zero: the restart from x = 0,
// folded over +0 without reading x), max|r| (for norm2), ||r||_2 (binary64),
// finiteness.
template <class Op, class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_gm_resid(Op op, const T* __restrict__ x, int x_zero,
                                                  const T* __restrict__ rhs, T* __restrict__ r, Geo g, Red rd,
                                                  DevState* st, int64_t wband = 0,
                                                  const T* __restrict__ zsrc = nullptr, double phat = 0.0) {
  GADI_G;
  constexpr bool EH = MatvecF<C, T>::EXACT_H;
  int bad = 0;
  double m = 0.0;
  unsigned mh = 0;  // EH: max |r| as binary16 magnitude bits (order preserving; NaN excluded)
  C w0;
  double w1;
  auto fin = [&](const Seg& s, double& d, const C (&acc)[G]) {
    T rv[G];
    double td[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      rv[i] = st_t<T, C>(acc[i]);
      if constexpr (EH) {  // no binary64 work but the exact square's widening
        td[i] = (double)fhfma(rv[i], rv[i], -0.0f);
        const unsigned mag = __half_as_ushort(rv[i]) & 0x7fffu;
        if (GADI_LIVE(i)) {
          bad |= mag >= 0x7c00u ? 1 : 0;
          mh = (mag <= 0x7c00u && mag > mh) ? mag : mh;
        }
      } else {
        const double dv = to_dbl(rv[i]);
        td[i] = __dmul_rn(dv, dv);
        if (GADI_LIVE(i)) {
          bad |= finite_t(rv[i]) ? 0 : 1;
          m = (dv == dv) ? fmax(m, fabs(dv)) : m;
        }
      }
    }
    store_seg<T, VEC, G>(r, s, rv);
    d = seg_sum<double, G>(td, s.len);
  };
  auto body = [&](const Seg& s, double& d, const auto& src) {
    T bv[G], xc[G];
    load_seg<T, VEC, G>(rhs, s, bv);
    C acc[G];
#pragma unroll
    for (int i = 0; i < G; ++i) acc[i] = ld_c<T, C>(bv[i]);
    fold_seg<VEC, G>(op, src, s, acc, ResidF<C, T>(), xc);
    fin(s, d, acc);
  };
  if (x_zero) {  // from x = 0: the per-row zflag summaries, the matrix is not read
    // zsrc != null: rhs = round(phat * z) is formed here (k_scale's formula;
    // solver.cpp:155, the scale of z before solve_S) instead of being read.
    // Binary16 z and phat: the product is exact in binary32 (22 significant
    // bits, exponents in range), so one binary32 multiply and one rounding to
    // binary16 equal the binary64 route.
    const float pf = (float)phat;
    bool f16 = false;
    if constexpr (std::is_same<T, __half>::value) f16 = (double)__half2float(__float2half_rn(pf)) == phat;
    seg_run_ld<VEC, false, true, G>(g, zsrc ? zsrc : rhs, [&](const Seg& s, const T (&bv0)[G], C&, double& d) {
      T bv[G];
      if (zsrc && f16) {
        if constexpr (std::is_same<T, __half>::value) {
#pragma unroll
          for (int i = 0; i < G; ++i) bv[i] = __float2half_rn(__fmul_rn(pf, __half2float(bv0[i])));
        }
      } else {
#pragma unroll
        for (int i = 0; i < G; ++i) bv[i] = zsrc ? from_dbl<T>(__dmul_rn(phat, to_dbl(bv0[i]))) : bv0[i];
      }
      C acc[G];
      if constexpr (VEC > 1) {
        int fl[VEC];
        op.template zflags_vec<VEC>(s.lo, fl);
#pragma unroll
        for (int i = 0; i < G; ++i) acc[i] = zero_resid(ld_c<T, C>(bv[i]), fl[i]);
      } else {
#pragma unroll
        for (int i = 0; i < G; ++i)
          acc[i] = GADI_LIVE(i) ? zero_resid(ld_c<T, C>(bv[i]), op.zflags(s.lo + i)) : ld_c<T, C>(bv[i]);
      }
      fin(s, d, acc);
    }, w0, w1);
  } else if (VEC > 1 && wband > 0) {
    const SmemSrc<T> src = stage_window<T, VEC>(x, g, wband);
    seg_run<VEC, false, true>(g, [&](const Seg& s, C&, double& d) { body(s, d, src); }, w0, w1);
  } else {
    const PlainSrc<T> src{x};
    seg_run<VEC, false, true>(g, [&](const Seg& s, C&, double& d) { body(s, d, src); }, w0, w1);
  }
  if constexpr (EH) m = (double)__half2float(__ushort_as_half((unsigned short)mh));
  block_max_abs(&st->maxbits, m);
  or_flags(&st->flags, bad);
  C dc;
  double ss;
  if (grid_finish(w0, w1, g, rd, dc, ss)) finish_red(EpiRedD{}, st, dc, ss);
}

// The fused mode's restart residual from x = 0 (accum = FP32: binary16 storage,
// binary32 arithmetic): r = rhs (or round(phat z), formed here) under the
// zero-start sign rules, ||r||_2 in binary64 for the stop test AND
// beta = sqrt(dot(r, r)) in binary32 (the unscaled norm of the fused Arnoldi
// step; the native modes keep the reference's max-scaled norm2 in k_norm2),
// finiteness from the segment's sum of squares (a square of a finite binary16
// is at most 4.3e9, so the sum is finite exactly when every entry is).
// Packed fast path: binary16 pairs are scaled with HMUL2 (the product of two
// binary16 values is exact in binary32, so one rounding to binary16 is the
// reference's scale), and the zero-start rules only touch -0 entries and
// non-finite coefficients -- a chunk with neither is stored as it is.
// v_0 = r / beta: the factor for a speculative first Arnoldi step (out of line, as gm_column_done)
static __device__ __noinline__ void gm_beta_done(DevState* st) { st->gm_inv = 1.0 / st->red_c; }
struct EpiResidF {
  template <class C>
  __device__ void finish(C ss32, double ss, DevState* st) const {
    st->red_d = ss;
    const double beta = to_dbl(Ar<C>::from_d(__dsqrt_rn(Ar<C>::to_d(ss32))));
    st->red_c = beta;
    gm_beta_done(st);
  }
  __device__ int* flag_dst(DevState* st) const { return &st->flags; }
  __device__ bool skip(DevState* st) const { return (void)st, false; }
};
template <class Op, int VEC>
__global__ void __launch_bounds__(256) k_gm_resid0(Op op, const __half* __restrict__ rhs, __half* __restrict__ r,
                                                   Geo g, Red rd, DevState* st, const __half* __restrict__ zsrc,
                                                   double phat) {
  using T = __half;
  using C = float;
  GADI_G;
  const float pf = (float)phat;
  const bool f16 = zsrc && (double)__half2float(__float2half_rn(pf)) == phat;
  const __half2 p2 = __float2half2_rn(pf);
  int bad = 0;
  C w0;
  double w1;
  seg_run_ld<VEC, true, true, G>(g, zsrc ? zsrc : rhs, [&](const Seg& s, const T (&bv0)[G], C& c, double& d) {
    T rv[G];
    if (f16) {
#pragma unroll
      for (int i = 0; i < G; i += 2) {
        const __half2 pr = __hmul2(__halves2half2(bv0[i], bv0[i + 1]), p2);
        rv[i] = __low2half(pr);
        rv[i + 1] = __high2half(pr);
      }
    } else {
#pragma unroll
      for (int i = 0; i < G; ++i) rv[i] = zsrc ? from_dbl<T>(__dmul_rn(phat, to_dbl(bv0[i]))) : bv0[i];
    }
    int fl[G];
    if constexpr (VEC > 1) {
      op.template zflags_vec<VEC>(s.lo, fl);
    } else {
#pragma unroll
      for (int i = 0; i < G; ++i) fl[i] = GADI_LIVE(i) ? op.zflags(s.lo + i) : 0;
    }
    int special = 0;
#pragma unroll
    for (int i = 0; i < G; ++i) special |= (fl[i] & 2) | ((__half_as_ushort(rv[i]) == 0x8000u) ? (fl[i] & 1) : 0);
    if (special) {  // rare: a -0 entry under a sign-set coefficient, or a non-finite coefficient
#pragma unroll
      for (int i = 0; i < G; ++i)
        if (GADI_LIVE(i)) rv[i] = st_t<T, C>(zero_resid(ld_c<T, C>(rv[i]), fl[i]));
    }
    C tc[G];
    double td[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const float f = GADI_LIVE(i) ? __half2float(rv[i]) : 0.0f;
      tc[i] = __fmul_rn(f, f);  // exact
      td[i] = (double)tc[i];
    }
    store_seg<T, VEC, G>(r, s, rv);
    c = seg_sum<C, G>(tc, s.len);
    d = seg_sum<double, G>(td, s.len);
    bad |= isfinite(c) ? 0 : 1;
  }, w0, w1);
  or_flags(&st->flags, bad);
  C dc;
  double ss;
  if (grid_finish(w0, w1, g, rd, dc, ss)) finish_red(EpiResidF{}, st, dc, ss);
}

// beta = sqrt(dot(w, w)) in the inner arithmetic into st->red_c (the fused mode's
// norm after a restart residual from x != 0)
struct EpiSqrtRedC {
  template <class C>
  __device__ void finish(C ss, double, DevState* st) const {
    const double beta = to_dbl(Ar<C>::from_d(__dsqrt_rn(Ar<C>::to_d(ss))));
    st->red_c = beta;
    gm_beta_done(st);
  }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ bool skip(DevState* st) const { return (void)st, false; }
};
template <class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_selfdot(const T* __restrict__ w, Geo g, Red rd, DevState* st) {
  GADI_G;
  C w0;
  double w1;
  seg_run_ld<VEC, true, false, G>(g, w, [&](const Seg& s, const T (&wv)[G], C& c, double&) {
    C tc[G];
#pragma unroll
    for (int i = 0; i < G; ++i) tc[i] = Ar<C>::mul(ld_c<T, C>(wv[i]), ld_c<T, C>(wv[i]));
    c = seg_sum<C, G>(tc, s.len);
  }, w0, w1);
  C ss;
  double dummy;
  if (grid_finish(w0, w1, g, rd, ss, dummy)) finish_red(EpiSqrtRedC{}, st, ss, dummy);
}

struct EpiNorm2 {  // m * sqrt(sum) in the inner format (kernels.cpp:79-81), m = max|w| from maxbits
  double* dst;
  template <class C>
  __device__ void finish(C sum, double, DevState* st) const {
    const double m = __longlong_as_double((long long)*(volatile unsigned long long*)&st->maxbits);
    if (m == 0.0 || !isfinite(m)) {
      *dst = m;
    } else {
      const C sq = Ar<C>::from_d(__dsqrt_rn(Ar<C>::to_d(sum)));
      *dst = to_dbl(Ar<C>::mul(from_dbl<C>(m), sq));
    }
  }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ bool skip(DevState* st) const { return (void)st, false; }
};

// norm2 in the inner format (kernels.cpp:71-82): m = max|w| (from maxbits),
// q = w/m, pairwise sum of q*q, m * sqrt(sum); written to *dst.
template <class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_norm2(const T* __restrict__ w, double* dst, Geo g, Red rd,
                                               DevState* st) {
  GADI_G;
  const double m = __longlong_as_double((long long)*(volatile unsigned long long*)&st->maxbits);
  const C mc = from_dbl<C>(m);
  // w/m for binary16/32 operands: round(w * RN64(1/m)) is the correctly
  // rounded quotient (the binary64 product is within 2^-52 of w/m, and a
  // quotient of p-bit numbers is either exact in p bits or at least 2^-2p-1
  // away from a p-bit rounding boundary, p <= 24); binary64 divides.
  const double rinv = __ddiv_rn(1.0, m);
  // binary16 operands in binary32 arithmetic: Markstein's correction of the
  // product with y = RN(1/m) (two FMAs) gives the correctly rounded quotient
  // without binary64 work; checked exhaustively against RN(w/m) over all
  // binary16 pairs 0 <= w <= m (tools/check_markstein.c).
  constexpr bool MK = std::is_same<T, __half>::value && std::is_same<C, float>::value;
  const float mf = (float)m, yf = MK ? __frcp_rn(mf) : 0.f;
  C w0;
  double w1;
  seg_run_ld<VEC, true, false, G>(g, w, [&](const Seg& s, const T (&wv)[G], C& c, double&) {
    C tc[G];
    if constexpr (MK && G % 2 == 0) {
      // the same Markstein quotient and square per lane, two lanes per
      // instruction (FMUL2 / FFMA2: one RN rounding per lane); the squares
      // feed scalar FADDs, which ptxas never contracts with an FMUL2
      const float2 y2 = make_float2(yf, yf), m2 = make_float2(-mf, -mf);
#pragma unroll
      for (int i = 0; i < G; i += 2) {
        const float2 wf = __half22float2(__halves2half2(wv[i], wv[i + 1]));
        const float2 q0 = __fmul2_rn(wf, y2);
        const float2 q = __ffma2_rn(__ffma2_rn(q0, m2, wf), y2, q0);
        const float2 sq = __fmul2_rn(q, q);
        tc[i] = sq.x;
        tc[i + 1] = sq.y;
      }
      c = seg_sum<C, G>(tc, s.len);
      return;
    }
#pragma unroll
    for (int i = 0; i < G; ++i) {
      C qv;
      if constexpr (std::is_same<C, double>::value) {
        qv = div_c<C>(ld_c<T, C>(wv[i]), mc);
      } else if constexpr (MK) {
        const float wf = __half2float(wv[i]);
        const float q0 = __fmul_rn(wf, yf);
        qv = __fmaf_rn(__fmaf_rn(-q0, mf, wf), yf, q0);
      } else {
        qv = Ar<C>::from_d(__dmul_rn(to_dbl(wv[i]), rinv));
      }
      tc[i] = Ar<C>::mul(qv, qv);
    }
    c = seg_sum<C, G>(tc, s.len);
  }, w0, w1);
  C sum;
  double dummy;
  if (grid_finish(w0, w1, g, rd, sum, dummy)) finish_red(EpiNorm2{dst}, st, sum, dummy);
}

// dst = round(a * src) with a in binary64 (scale, kernels.cpp:166-171); F32: scale_rn's binary32 variant.
template <class T, int VEC, bool F32 = false>
__global__ void __launch_bounds__(256) k_scale(const T* __restrict__ src, T* __restrict__ dst, double a, Geo g) {
  GADI_G;
  seg_each<VEC>(g, [&](const Seg& s) {
    T v[G];
    load_seg<T, VEC, G>(src, s, v);
#pragma unroll
    for (int i = 0; i < G; ++i) v[i] = scale_rn<T, F32>(a, v[i]);
    store_seg<T, VEC, G>(dst, s, v);
  });
}

// Arnoldi step j (inner_solver.cpp:120-122, 133-134): v_j = w_prev / h (the
// previous step's scale, fused here; SCALED == false: v_j as stored), then
// w = S v_j and h_0j = dot(w, v_0). wprev and w must be different buffers.
template <class Op, class T, class C, int VEC, bool SCALED>
__global__ void __launch_bounds__(256) k_gm_matvec(Op op, const T* __restrict__ wprev, double inv,
                                                   T* vj, const T* v0,
                                                   T* __restrict__ w, Geo g, Red rd, DevState* st,
                                                   int64_t wband = 0) {
  GADI_G;
  C w0;
  double w1;
  auto body = [&](const Seg& s, C& c, const auto& src) {
    C acc[G];
    T vv[G], wv[G], v0v[G];
#pragma unroll
    for (int i = 0; i < G; ++i) acc[i] = Ar<C>::zero();
    fold_seg<VEC, G>(op, src, s, acc, MatvecF<C, T>(), vv);
    if constexpr (SCALED) store_seg<T, VEC, G>(vj, s, vv);
#pragma unroll
    for (int i = 0; i < G; ++i) wv[i] = st_t<T, C>(acc[i]);
    store_seg<T, VEC, G>(w, s, wv);
    if (vj == v0) {  // step 0: v_0 is the operand just formed (never re-read)
#pragma unroll
      for (int i = 0; i < G; ++i) v0v[i] = vv[i];
    } else {
      load_seg<T, VEC, G>(v0, s, v0v);
    }
    C tc[G];
#pragma unroll
    for (int i = 0; i < G; ++i) tc[i] = Ar<C>::mul(ld_c<T, C>(wv[i]), ld_c<T, C>(v0v[i]));
    c = seg_sum<C, G>(tc, s.len);
  };
  if constexpr (SCALED) {
    const ScaleSrc<T, std::is_same<T, __half>::value && std::is_same<C, float>::value> src{wprev, inv};
    seg_run<VEC, true, false>(g, [&](const Seg& s, C& c, double&) { body(s, c, src); }, w0, w1);
  } else if (VEC > 1 && wband > 0) {
    const SmemSrc<T> src = stage_window<T, VEC>(vj, g, wband);
    seg_run<VEC, true, false>(g, [&](const Seg& s, C& c, double&) { body(s, c, src); }, w0, w1);
  } else {
    const PlainSrc<T> src{vj};
    seg_run<VEC, true, false>(g, [&](const Seg& s, C& c, double&) { body(s, c, src); }, w0, w1);
  }
  C h;
  double dummy;
  if (grid_finish(w0, w1, g, rd, h, dummy)) finish_red(EpiHcol{0}, st, h, dummy);
}

// Modified Gram-Schmidt step i (inner_solver.cpp:121-125): w -= h_i v_i, then
// either h_{i+1} = dot(w, v_{i+1}) (i < j) or max|w| for the norm (i == j).
template <class T, class C, int VEC, bool LAST>
__global__ void __launch_bounds__(256) k_gm_mgs(T* __restrict__ w, const T* __restrict__ vi,
                                                const T* __restrict__ vnext, int i, Geo g, Red rd,
                                                DevState* st) {
  GADI_G;
  const C nh = Ar<C>::neg(from_dbl<C>(st->hcol[i]));
  double m = 0.0;
  C w0;
  double w1;
  seg_run<VEC, !LAST, false>(g, [&](const Seg& s, C& c, double&) {
    T wv[G], vv[G];
    load_seg<T, VEC, G>(w, s, wv);
    load_seg<T, VEC, G>(vi, s, vv);
#pragma unroll
    for (int k = 0; k < G; ++k) wv[k] = st_t<T, C>(Ar<C>::add(ld_c<T, C>(wv[k]), Ar<C>::mul(nh, ld_c<T, C>(vv[k]))));
    store_seg<T, VEC, G>(w, s, wv);
    if constexpr (LAST) {
#pragma unroll
      for (int k = 0; k < G; ++k)
        if (GADI_LIVE(k)) {
          const double dv = to_dbl(wv[k]);
          m = (dv == dv) ? fmax(m, fabs(dv)) : m;
        }
    } else {
      load_seg<T, VEC, G>(vnext, s, vv);
      C tc[G];
#pragma unroll
      for (int k = 0; k < G; ++k) tc[k] = Ar<C>::mul(ld_c<T, C>(wv[k]), ld_c<T, C>(vv[k]));
      c = seg_sum<C, G>(tc, s.len);
    }
  }, w0, w1);
  if constexpr (LAST) {
    block_max_abs(&st->maxbits, m);
  } else {
    C h;
    double dummy;
    if (grid_finish(w0, w1, g, rd, h, dummy)) finish_red(EpiHcol{i + 1}, st, h, dummy);
  }
}

// ------------------------------------------------ fused Gram-Schmidt (accum = FP32)
// The GADI_ACCUM_FP32 extension mode (binary16 storage, binary32 arithmetic;
// not in the reference) orthogonalises an Arnoldi vector in two passes instead
// of j + 2: every h(i, j) = dot(w, v_i) from the same w (classical
// Gram-Schmidt; h(0, j) comes from the matvec pass), then ONE update pass
// w <- w - sum_i h_i v_i carried in binary32 with a single rounding to the
// storage format, fused with dot(w, w) for h(j+1, j) = sqrt(.) -- (2j + 7) N
// values moved per step instead of (4j + 7) N. The oracle restates exactly
// this (gadi_oracle.c gmres_solve, `fused`).

// J-channel versions of seg_run / grid_finish (C0 channels only): the same
// pairwise trees per channel, one pass over the data, one grid ticket.
template <int VEC, int J, class C0, class Body>
__device__ __forceinline__ void seg_run_multi(const Geo& g, Body&& body, C0 (&w)[J]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  C0 a[J][RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    if (r < g.R) {
      const int64_t t = (((int64_t)blockIdx.x * g.W + warp) * g.R + r) * g.L + lane;
      const Seg s = seg_of<VEC>(t, g.N, g.D);
      C0 c[J];
#pragma unroll
      for (int k = 0; k < J; ++k) c[k] = Ar<C0>::zero();
      body(s, c);
#pragma unroll
      for (int k = 0; k < J; ++k) a[k][r] = warp_tree(c[k], g.L);
    }
  }
#pragma unroll
  for (int st = 1; st < RMAX; st <<= 1)
#pragma unroll
    for (int r = 0; r + st < RMAX; r += 2 * st)
      if (r + st < g.R) {
#pragma unroll
        for (int k = 0; k < J; ++k) a[k][r] = Ar<C0>::add(a[k][r], a[k][r + st]);
      }
#pragma unroll
  for (int k = 0; k < J; ++k) w[k] = a[k][0];
}

// part: J arrays of `stride` block partials. True in thread 0 of the last block.
template <int J, class C0>
__device__ __forceinline__ bool grid_finish_multi(C0 (&w)[J], const Geo& g, double* part, int64_t stride,
                                                  unsigned* ticket, C0 (&tot)[J]) {
  __shared__ __align__(8) unsigned char smb[J][32 * sizeof(double)];
  __shared__ int last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (g.W > 1) {
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < J; ++k) reinterpret_cast<C0*>(smb[k])[warp] = w[k];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int k = 0; k < J; ++k) {
        C0 v = lane < g.W ? reinterpret_cast<C0*>(smb[k])[lane] : Ar<C0>::zero();
        if (lane < g.W) v = warp_tree(v, g.W);
        w[k] = v;
      }
    }
  }
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < J; ++k) part[k * stride + blockIdx.x] = to_dbl(w[k]);
    __threadfence();
    const unsigned t = atomicAdd(ticket, 1u);
    last = (t == (unsigned)g.nblk - 1u);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  const int P = g.nblk, B = blockDim.x;
#pragma unroll
  for (int k = 0; k < J; ++k) {
    const double* pk = part + k * stride;
    C0 a;
    int cnt;
    if (P <= B) {
      a = tid < P ? from_dbl<C0>(__ldcg(pk + tid)) : Ar<C0>::zero();
      cnt = P;
    } else {
      const int64_t Lr = P / B;
      const double* p0 = pk + (int64_t)tid * Lr;
      a = run_pairwise<C0>(Lr, [&](int64_t j) { return from_dbl<C0>(__ldcg(p0 + j)); });
      cnt = B;
    }
    __syncthreads();
    a = block_tree(a, cnt, reinterpret_cast<C0*>(smb[k]));
    if (tid == 0) tot[k] = a;
  }
  if (tid == 0) *ticket = 0u;
  return tid == 0;
}

// h(i0 + k, j) = dot(w, v_{i0+k}), k < J, in one pass over w and the J basis vectors.
template <class T, class C, int VEC, int J>
__global__ void __launch_bounds__(256) k_gm_dots(const T* __restrict__ w, const T* __restrict__ V, int64_t ldv, int i0,
                                                 Geo g, Red rd, double* partm, int64_t pstride, DevState* st) {
  GADI_G;
  C ws[J];
  seg_run_multi<VEC, J>(g, [&](const Seg& s, C (&c)[J]) {
    T wv[G], vv[G];
    load_seg<T, VEC, G>(w, s, wv);
#pragma unroll
    for (int k = 0; k < J; ++k) {
      load_seg<T, VEC, G>(V + (int64_t)(i0 + k) * ldv, s, vv);
      C tc[G];
#pragma unroll
      for (int e = 0; e < G; ++e) tc[e] = Ar<C>::mul(ld_c<T, C>(wv[e]), ld_c<T, C>(vv[e]));
      c[k] = seg_sum<C, G>(tc, s.len);
    }
  }, ws);
  C tot[J];
  if (grid_finish_multi<J>(ws, g, partm, pstride, rd.ticket, tot)) {
    if (J == 1) {
      finish_red(EpiHcol{i0}, st, tot[0], 0.0);  // sharded solves: one record per dot
    } else {
#pragma unroll
      for (int k = 0; k < J; ++k) st->hcol[i0 + k] = to_dbl(tot[k]);
    }
  }
}

// After column j of a speculative Arnoldi window is complete (one thread, its own launch so
// that k_gm_cgs keeps its code): the host's inv for v_{j+1} = w / h1, and the column into
// hhist[slot].
static __global__ void k_gm_column_done(DevState* st, int j, int slot) {
  const double h1 = st->hcol[j + 1];
  st->gm_inv = h1 != 0.0 ? 1.0 / h1 : 0.0;
  for (int i = 0; i <= j + 1; ++i) st->hhist[slot][i] = st->hcol[i];
}
struct EpiCgsNorm {  // h(j+1, j) = sqrt(dot(w, w)) in the inner arithmetic
  int j;
  template <class C>
  __device__ void finish(C ss, double, DevState* st) const {
    st->hcol[j + 1] = to_dbl(Ar<C>::from_d(__dsqrt_rn(Ar<C>::to_d(ss))));
  }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ bool skip(DevState* st) const { return (void)st, false; }
};

// w <- round_T(w - h_0 v_0 - ... - h_j v_j) (each op rounded to C) and dot(w, w).
template <class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_gm_cgs(T* __restrict__ w, const T* __restrict__ V, int64_t ldv, int j, Geo g,
                                                Red rd, DevState* st) {
  GADI_G;
  __shared__ C snh[72];  // -h(i, j), read by every segment
  for (int i = threadIdx.x; i <= j; i += blockDim.x) snh[i] = Ar<C>::neg(from_dbl<C>(st->hcol[i]));
  __syncthreads();
  C w0;
  double w1;
  seg_run<VEC, true, false>(g, [&](const Seg& s, C& c, double&) {
    T wv[G], vv[G];
    C acc[G];
    load_seg<T, VEC, G>(w, s, wv);
#pragma unroll
    for (int e = 0; e < G; ++e) acc[e] = ld_c<T, C>(wv[e]);
    int i = 0;
    for (; i + 4 <= j + 1; i += 4) {  // four basis vectors in flight at a time
      T v4[4][G];
#pragma unroll
      for (int u = 0; u < 4; ++u) load_seg<T, VEC, G>(V + (int64_t)(i + u) * ldv, s, v4[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const C nh = snh[i + u];
#pragma unroll
        for (int e = 0; e < G; ++e) acc[e] = Ar<C>::add(acc[e], Ar<C>::mul(nh, ld_c<T, C>(v4[u][e])));
      }
    }
    for (; i <= j; ++i) {
      const C nh = snh[i];
      load_seg<T, VEC, G>(V + (int64_t)i * ldv, s, vv);
#pragma unroll
      for (int e = 0; e < G; ++e) acc[e] = Ar<C>::add(acc[e], Ar<C>::mul(nh, ld_c<T, C>(vv[e])));
    }
    C tc[G];
#pragma unroll
    for (int e = 0; e < G; ++e) {
      wv[e] = st_t<T, C>(acc[e]);
      const C r = ld_c<T, C>(wv[e]);
      tc[e] = Ar<C>::mul(r, r);
    }
    store_seg<T, VEC, G>(w, s, wv);
    c = seg_sum<C, G>(tc, s.len);
  }, w0, w1);
  C ss;
  double dummy;
  if (grid_finish(w0, w1, g, rd, ss, dummy)) finish_red(EpiCgsNorm{j}, st, ss, dummy);
}

// k_gm_cgs for the first Arnoldi steps (NB = j + 1 <= 7 basis vectors): all of a segment's
// loads are issued together, and with NB <= 2 the next segment's loads too (double buffer),
// so at least four 16-byte loads per lane are in flight (the generic body has NB + 1: 198 us
// for 0.8 GB at j = 0). Same per-element sequence and the same reduction tree.
// STORE = false: the last step of a cycle (restart or max_inner reached) -- the updated w is
// only reduced (h(j+1, j)), nothing reads it afterwards.
template <class T, class C, int VEC, int NB, bool STORE = true>
__global__ void __launch_bounds__(256) k_gm_cgs_few(T* __restrict__ w, const T* __restrict__ V, int64_t ldv, Geo g,
                                                    Red rd, DevState* st) {
  GADI_G;
  static_assert(VEC > 1, "aligned segments");
  constexpr int j = NB - 1;
  constexpr bool PF = NB <= 2;
  C nh[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) nh[i] = Ar<C>::neg(from_dbl<C>(st->hcol[i]));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto seg_t = [&](int r) { return (((int64_t)blockIdx.x * g.W + warp) * g.R + r) * g.L + lane; };
  T wv[PF ? 2 : 1][G], vb[PF ? 2 : 1][NB][G];
  auto loads = [&](int r, int buf) {
    const int64_t e0 = seg_t(r) * VEC;
    ld_vec<T, VEC>(w, e0, wv[buf]);
#pragma unroll
    for (int u = 0; u < NB; ++u) ld_vec<T, VEC>(V + (int64_t)u * ldv, e0, vb[buf][u]);
  };
  C a0[RMAX];
  if (PF) loads(0, 0);
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    if (r < g.R) {
      const int buf = PF ? (r & 1) : 0;
      if (PF) {
        if (r + 1 < g.R) loads(r + 1, buf ^ 1);
      } else {
        loads(r, 0);
      }
      C acc[G];
#pragma unroll
      for (int e = 0; e < G; ++e) acc[e] = ld_c<T, C>(wv[buf][e]);
#pragma unroll
      for (int u = 0; u < NB; ++u)
#pragma unroll
        for (int e = 0; e < G; ++e) acc[e] = Ar<C>::add(acc[e], Ar<C>::mul(nh[u], ld_c<T, C>(vb[buf][u][e])));
      C tc[G];
      T ov[G];
#pragma unroll
      for (int e = 0; e < G; ++e) {
        ov[e] = st_t<T, C>(acc[e]);
        const C rr = ld_c<T, C>(ov[e]);
        tc[e] = Ar<C>::mul(rr, rr);
      }
      if constexpr (STORE) st_vec<T, VEC>(w, seg_t(r) * VEC, ov);
      a0[r] = warp_tree(seg_sum<C, G>(tc, G), g.L);
    }
  }
#pragma unroll
  for (int s2 = 1; s2 < RMAX; s2 <<= 1)
#pragma unroll
    for (int r = 0; r + s2 < RMAX; r += 2 * s2)
      if (r + s2 < g.R) a0[r] = Ar<C>::add(a0[r], a0[r + s2]);
  C ss;
  double dummy;
  if (grid_finish(a0[0], 0.0, g, rd, ss, dummy)) finish_red(EpiCgsNorm{j}, st, ss, dummy);
}

// x += y_0 v_0; x += y_1 v_1; ... (inner_solver.cpp:174), one pass, the
// sequence of rounded axpys kept per element; x_zero: x starts at 0.
template <class T, class C, int VEC>
__global__ void __launch_bounds__(256) k_gm_update(T* __restrict__ x, int x_zero, const T* __restrict__ V,
                                                   int64_t ldv, int j, Geo g, DevState* st) {
  GADI_G;
  int bad = 0;
  __shared__ C sy[72];  // the coefficients, read by every segment
  for (int i = threadIdx.x; i < j; i += blockDim.x) sy[i] = from_dbl<C>(st->ycoef[i]);
  __syncthreads();
  seg_each<VEC>(g, [&](const Seg& s) {
    T xv[G], vv[G];
    C xc[G];
    if (!x_zero) load_seg<T, VEC, G>(x, s, xv);
#pragma unroll
    for (int k = 0; k < G; ++k) xc[k] = x_zero ? Ar<C>::zero() : ld_c<T, C>(xv[k]);
    int i = 0;
    for (; i + 4 <= j; i += 4) {  // four basis vectors in flight at a time
      T v4[4][G];
#pragma unroll
      for (int u = 0; u < 4; ++u) load_seg<T, VEC, G>(V + (int64_t)(i + u) * ldv, s, v4[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const C y = sy[i + u];
#pragma unroll
        for (int k = 0; k < G; ++k)
          xc[k] = ld_c<T, C>(st_t<T, C>(Ar<C>::add(xc[k], Ar<C>::mul(y, ld_c<T, C>(v4[u][k])))));
      }
    }
    for (; i < j; ++i) {
      const C y = sy[i];
      load_seg<T, VEC, G>(V + (int64_t)i * ldv, s, vv);
#pragma unroll
      for (int k = 0; k < G; ++k) xc[k] = ld_c<T, C>(st_t<T, C>(Ar<C>::add(xc[k], Ar<C>::mul(y, ld_c<T, C>(vv[k])))));
    }
#pragma unroll
    for (int k = 0; k < G; ++k) {
      xv[k] = st_t<T, C>(xc[k]);
      if (GADI_LIVE(k)) bad |= finite_t(xv[k]) ? 0 : 1;
    }
    store_seg<T, VEC, G>(x, s, xv);
  });
  or_flags(&st->flags, bad);
}

// k_gm_update for a short cycle (NB = j <= 7 basis vectors): every load of a segment is issued
// before the first axpy (the generic body reads the vectors past a multiple of four one at a
// time). Same sequence of rounded axpys per element.
template <class T, class C, int VEC, int NB>
__global__ void __launch_bounds__(256) k_gm_update_few(T* __restrict__ x, int x_zero, const T* __restrict__ V,
                                                       int64_t ldv, Geo g, DevState* st) {
  GADI_G;
  static_assert(VEC > 1, "aligned segments");
  int bad = 0;
  C y[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) y[i] = from_dbl<C>(st->ycoef[i]);
  seg_each<VEC>(g, [&](const Seg& s) {
    T xv[G], vb[NB][G];
    if (!x_zero) load_seg<T, VEC, G>(x, s, xv);
#pragma unroll
    for (int u = 0; u < NB; ++u) load_seg<T, VEC, G>(V + (int64_t)u * ldv, s, vb[u]);
    C xc[G];
#pragma unroll
    for (int k = 0; k < G; ++k) xc[k] = x_zero ? Ar<C>::zero() : ld_c<T, C>(xv[k]);
#pragma unroll
    for (int u = 0; u < NB; ++u)
#pragma unroll
      for (int k = 0; k < G; ++k)
        xc[k] = ld_c<T, C>(st_t<T, C>(Ar<C>::add(xc[k], Ar<C>::mul(y[u], ld_c<T, C>(vb[u][k])))));
#pragma unroll
    for (int k = 0; k < G; ++k) {
      xv[k] = st_t<T, C>(xc[k]);
      bad |= finite_t(xv[k]) ? 0 : 1;
    }
    store_seg<T, VEC, G>(x, s, xv);
  });
  or_flags(&st->flags, bad);
}

// ============================================================ outer loop
struct EpiResidA {  // ||s||, max|s| and the scaling exponent (solver.cpp:48-53)
  int scaling;
  __device__ void finish(double, double ss, DevState* st) const {
    const double mx = __longlong_as_double((long long)*(volatile unsigned long long*)&st->maxbits);
    st->res_ss = ss;
    st->res_max = mx;
    st->res_e = (scaling && mx != 0.0 && isfinite(mx)) ? ilogb(mx) : 0;
  }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ bool skip(DevState* st) const { return (void)st, false; }
};
struct EpiResidSpec {  // EpiResidA + ||rhat||^2 of the speculative pass (PolResidSpec)
  int scaling;
  __device__ void finish(double rss, double ss, DevState* st) const {
    EpiResidA{scaling}.finish(0.0, ss, st);
    st->rhat_ss = rss;
  }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ bool skip(DevState* st) const { return (void)st, false; }
};
struct EpiRhat {  // ||rhat||_2
  __device__ void finish(double, double ss, DevState* st) const { st->rhat_ss = ss; }
  __device__ int* flag_dst(DevState*) const { return nullptr; }
  __device__ bool skip(DevState* st) const { return (void)st, false; }
};
// s = b - A x in u_f (residual_uf, solver.cpp:190-192); max|s|, ||s||_2 and
// the scaling exponent e = ilogb(max|s|) (solver.cpp:48-53). s may be null
// (norm only: true_residual_norm, solver.cpp:194-197).
template <class Op, int PF, int VEC>
__global__ void __launch_bounds__(256) k_resid_A(Op op, const double* __restrict__ x, const double* __restrict__ b,
                                                 double* __restrict__ sv, int scaling, Geo g, Red rd,
                                                 DevState* st, int64_t wband = 0, double nsc = 1.0) {
  GADI_G;
  double m = 0.0, w0, w1;
  const bool nscale = nsc != 1.0;  // squares of s 2^-ns (norm2_64's max scaling as an exact power of two)
  auto body = [&](const Seg& s, double& d, const auto& src) {
    double acc[G], xc[G];
    load_seg<double, VEC, G>(b, s, acc);
    fold_seg<VEC, G>(op, src, s, acc, ResidAF<PF>(), xc);
    double td[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const double av = nscale ? __dmul_rn(acc[i], nsc) : acc[i];
      td[i] = __dmul_rn(av, av);
      if (GADI_LIVE(i)) m = (acc[i] == acc[i]) ? fmax(m, fabs(acc[i])) : m;
    }
    if (sv) store_seg<double, VEC, G>(sv, s, acc);
    d = seg_sum<double, G>(td, s.len);
  };
  if (VEC > 1 && wband > 0) {
    const SmemSrc<double> src = stage_window<double, VEC>(x, g, wband);
    seg_run<VEC, false, true>(g, [&](const Seg& s, double&, double& d) { body(s, d, src); }, w0, w1);
  } else {
    const PlainSrc<double> src{x};
    seg_run<VEC, false, true>(g, [&](const Seg& s, double&, double& d) { body(s, d, src); }, w0, w1);
  }
  block_max_abs(&st->maxbits, m);
  double dummy, ss;
  if (grid_finish(w0, w1, g, rd, dummy, ss)) {
    __threadfence();
    finish_red(EpiResidA{scaling}, st, dummy, ss);
  }
}

// rhat = round_{u_r}(s * 2^-e) (solver.cpp:86-92) and ||rhat||_2.
template <class T, int VEC>
__global__ void __launch_bounds__(256) k_scale_round(const double* __restrict__ sv, T* __restrict__ rhat, Geo g,
                                                     Red rd, DevState* st, double nsc = 1.0) {
  GADI_G;
  const int e = st->res_e;
  const bool nscale = nsc != 1.0;
  const double p2 = (e >= -1000 && e <= 1000) ? pow2d(-e) : 1.0;
  double w0, w1;
  seg_run<VEC, false, true>(g, [&](const Seg& s, double&, double& d) {
    double v[G], td[G];
    load_seg<double, VEC, G>(sv, s, v);
    T o[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      o[i] = from_dbl<T>(e != 0 ? ldexp_fast(v[i], -e, p2) : v[i]);
      double dv = to_dbl(o[i]);
      if (nscale) dv = __dmul_rn(dv, nsc);
      td[i] = __dmul_rn(dv, dv);
    }
    store_seg<T, VEC, G>(rhat, s, o);
    d = seg_sum<double, G>(td, s.len);
  }, w0, w1);
  double dummy, ss;
  if (grid_finish(w0, w1, g, rd, dummy, ss)) finish_red(EpiRhat{}, st, dummy, ss);
}

// x = round_u(x + round_u(2^e y)) (solver.cpp:163-166 with axpy kernels.cpp:147-164).
template <class T, int PU, int VEC>
__global__ void __launch_bounds__(256) k_update(double* __restrict__ x, const T* __restrict__ y, Geo g,
                                                DevState* st) {
  GADI_G;
  const int e = st->res_e;
  const double p2 = (e >= -1000 && e <= 1000) ? pow2d(e) : 1.0;
  int bad = 0;
  seg_each<VEC>(g, [&](const Seg& s) {
    double xv[G];
    T yv[G];
    load_seg<double, VEC, G>(x, s, xv);
    load_seg<T, VEC, G>(y, s, yv);
#pragma unroll
    for (int i = 0; i < G; ++i) {
      double yd = to_dbl(yv[i]);
      if (e != 0) yd = ldexp_fast(yd, e, p2);
      xv[i] = round_p<PU>(__dadd_rn(xv[i], round_p<PU>(__dmul_rn(1.0, yd))));
      if (GADI_LIVE(i)) bad |= isfinite(xv[i]) ? 0 : 1;
    }
    store_seg<double, VEC, G>(x, s, xv);
  });
  or_flags(&st->xbad, bad);
}

// ------------------------------------------------------------ elementwise
template <class TI, class TO, int PR>
__global__ void k_convert(const TI* __restrict__ in, TO* __restrict__ out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = from_dbl<TO>(round_p<PR>(to_dbl(in[i])));
}

static __global__ void k_fill(double* __restrict__ x, double v, int64_t n) {
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
static __global__ void k_uniform(double* __restrict__ x, uint64_t seed, double lo, double hi, int64_t n,
                                 int64_t off = 0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = uniform01(seed, (uint64_t)(i + off), lo, hi);
}

// y = Op x with the given fold, one element per thread (tests / rhs).
template <class Op, class X, class Acc, class Y, class F>
__global__ void k_apply(Op op, const X* __restrict__ x, Y* __restrict__ y, int64_t n, F f) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  Acc a[1];
  X cc[1];
  a[0] = Ar<Acc>::zero();
  op.template fold<1>(PlainSrc<X>{x}, e, a, f, cc);
  y[e] = st_t<Y, Acc>(a[0]);
}

// dot over binary64-carried values in precision C (test entry points).
template <class C>
__global__ void __launch_bounds__(256) k_dot_d(const double* __restrict__ x, const double* __restrict__ y, Geo g,
                                               Red rd, double* out) {
  constexpr int VEC = 1;
  GADI_G;
  C w0;
  double w1;
  seg_run<VEC, true, false>(g, [&](const Seg& s, C& c, double&) {
    C tc[G];
#pragma unroll
    for (int i = 0; i < G; ++i)
      tc[i] = i < s.len ? Ar<C>::mul(Ar<C>::from_d(x[s.lo + i]), Ar<C>::from_d(y[s.lo + i])) : Ar<C>::zero();
    c = seg_sum<C, G>(tc, s.len);
  }, w0, w1);
  C t;
  double dummy;
  if (grid_finish(w0, w1, g, rd, t, dummy)) *out = to_dbl(t);
}

}  // namespace gadi
