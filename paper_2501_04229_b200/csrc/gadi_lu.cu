// gadi_lu.cu — the LuDirect inner method on the device: BandLU
// (band_lu.cpp:60-172), the reference's default inner solver
// (inner_solver.hpp:21), built by prepare (solver.cpp:199-208) for H and S and
// applied by inner_solve (solver.cpp:224-231).
//
// Storage is the reference's LAPACK band layout (band_lu.cpp:83): column j at
// ab + j*ldab, A(i,j) at row kl+ku+i-j, ldab = 2kl+ku+1 (kl rows of pivot
// fill). Values are binary64 for u_r = double and binary32 otherwise
// (binary16 values carried exactly in binary32, as the reference does).
// Every scalar op is rounded once to u_r with the reference's policies
// (band_lu.cpp:12-56); the element-wise operation sequence is the
// reference's, so factors and solutions are bit for bit the reference's.
//
// Factorization, blocked right-looking without changing any element's
// operation order: for a panel of nb columns,
//   k_lu_panel  one CTA factors the panel columns in shared memory (pivot
//               search = block argmax with the reference's first-max/NaN
//               rule, row swap inside the panel, multipliers, update of the
//               remaining panel columns);
//   k_lu_trail  one warp per trailing column replays the panel's nb steps on
//               that column (swap, then x -= l*a unless a == 0), reading the
//               multipliers from shared memory. A column's replay is the
//               reference's sequence of operations on that column.
// Solves (one CTA; the recurrences are sequential in j):
//   k_lu_fwd    blocks of 32 steps: warp 0 runs the 32x32 unit-lower triangle
//               through shuffles, bringing any pivot row outside the block up
//               to date before its swap; then every thread applies the block's
//               32 updates to the positions below in step order.
//   k_lu_bwd    the same with U, blocks of 32 descending steps.
#include "gadi_host.cuh"

#include <cfloat>
#include <climits>

namespace gadi_host {
namespace {

template <int P>
struct LuPol;
template <>
struct LuPol<GADI_DOUBLE> {  // PolDouble, band_lu.cpp:12-24
  using S = double;
  static __device__ __forceinline__ S mul(S a, S b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ S sub(S a, S b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ S div(S a, S b) { return __ddiv_rn(a, b); }
  static constexpr double tiny = DBL_MIN;
};
template <>
struct LuPol<GADI_SINGLE> {  // PolSingle, band_lu.cpp:28-38
  using S = float;
  static __device__ __forceinline__ S mul(S a, S b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ S sub(S a, S b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ S div(S a, S b) { return __fdiv_rn(a, b); }
  static constexpr double tiny = FLT_MIN;
};
template <>
struct LuPol<GADI_HALF> {  // PolHalf, band_lu.cpp:44-56: binary32 op, then one RNE to binary16
  using S = float;
  static __device__ __forceinline__ S r16(S v) { return __half2float(__float2half_rn(v)); }
  static __device__ __forceinline__ S mul(S a, S b) { return r16(__fmul_rn(a, b)); }
  static __device__ __forceinline__ S sub(S a, S b) { return r16(__fsub_rn(a, b)); }
  static __device__ __forceinline__ S div(S a, S b) { return r16(__fdiv_rn(a, b)); }
  static constexpr double tiny = 6.103515625e-05;  // 2^-14
};

__device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

constexpr int kPanelThreads = 1024;
constexpr int kTrailWarps = 8;
constexpr size_t kSmemBudget = 200 * 1024;

// ------------------------------------------------------------- band assembly
// BandLU ctor (band_lu.cpp:85-90): at(i, c) = round(value) for the stored
// entries of H or S. Stencil: the 7 coefficients of the regularized operator
// (already rounded to u_r), neighbours outside the grid absent.
template <class S>
__global__ void k_band_stencil(S* __restrict__ ab, int64_t n, int64_t N, int64_t ldoff, int64_t ldab,
                               double clo, double cd, double cup) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  const int64_t nn = n * n, i = r / nn, j = (r / n) % n, k = r % n;
  auto put = [&](int64_t c, double v) { ab[c * ldab + ldoff + r - c] = (S)v; };
  if (i > 0) put(r - nn, clo);
  if (j > 0) put(r - n, clo);
  if (k > 0) put(r - 1, clo);
  put(r, cd);
  if (k + 1 < n) put(r + 1, cup);
  if (j + 1 < n) put(r + n, cup);
  if (i + 1 < n) put(r + nn, cup);
}

// CSR: the HSS union pattern (gadi_csr.cuh k_union) with the diagonal shift of
// regularize (splitting.cpp:37-47, sparse.cpp:180-183), rounded to u_r.
template <class S, int PR>
__global__ void k_band_csr(S* __restrict__ ab, int64_t N, int64_t ldoff, int64_t ldab, const int64_t* __restrict__ rp,
                           const int32_t* __restrict__ ci, const double* __restrict__ val,
                           const int64_t* __restrict__ dpos, const uint8_t* __restrict__ din, double alpha) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
    double x = val[k];
    if (k == dpos[r]) x = din[r] ? __dadd_rn(__dmul_rn(1.0, x), alpha) : alpha;
    const int64_t c = ci[k];
    ab[c * ldab + ldoff + r - c] = (S)round_p<PR>(x);
  }
}

__global__ void k_bandwidths(int64_t N, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                             unsigned long long* bw) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N || rp[r] == rp[r + 1]) return;
  const int64_t lo = r - ci[rp[r]], hi = ci[rp[r + 1] - 1] - r;
  if (lo > 0) atomicMax(bw, (unsigned long long)lo);
  if (hi > 0) atomicMax(bw + 1, (unsigned long long)hi);
}

// ------------------------------------------------------------ factorization
template <int P>
__global__ void __launch_bounds__(kPanelThreads) k_lu_panel(typename LuPol<P>::S* __restrict__ ab, int64_t N,
                                                           int64_t kl, int64_t ku, int64_t ldab, int64_t j0,
                                                           int nbw, int R, int32_t* __restrict__ ipiv,
                                                           int* __restrict__ err) {
  using Pol = LuPol<P>;
  using S = typename Pol::S;
  extern __shared__ __align__(16) unsigned char lu_smem[];
  S* Pm = reinterpret_cast<S*>(lu_smem);  // Pm[c*R + r] = A(j0+r, j0+c)
  __shared__ double rv[32];
  __shared__ int ri[32];
  __shared__ int s_p, s_bad;
  if (*(volatile int*)err) return;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int64_t ldoff = kl + ku;
  for (int c = 0; c < nbw; ++c) {
    const int64_t k = j0 + c;
    for (int r = tid; r < R; r += nt) {
      const int64_t d = ldoff + j0 + r - k;
      Pm[c * R + r] = (d >= 0 && d < ldab) ? ab[k * ldab + d] : S(0);
    }
  }
  __syncthreads();
  for (int c = 0; c < nbw; ++c) {
    const int64_t j = j0 + c;
    const int rl = (int)(lmin(N - 1, j + kl) - j0);
    S* col = Pm + c * R;
    // pivot search, band_lu.cpp:95-104: the first row of maximal |a| (NaN never wins)
    double bv = -1.0;
    int br = INT_MAX;
    for (int r = c + tid; r <= rl; r += nt) {
      const double v = fabs((double)col[r]);
      if (v > bv) {
        bv = v;
        br = r;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(~0u, bv, o);
      const int orr = __shfl_xor_sync(~0u, br, o);
      if (ov > bv || (ov == bv && orr < br)) {
        bv = ov;
        br = orr;
      }
    }
    if (lane == 0) {
      rv[warp] = bv;
      ri[warp] = br;
    }
    __syncthreads();
    if (warp == 0) {
      bv = lane < nw ? rv[lane] : -1.0;
      br = lane < nw ? ri[lane] : INT_MAX;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(~0u, bv, o);
        const int orr = __shfl_xor_sync(~0u, br, o);
        if (ov > bv || (ov == bv && orr < br)) {
          bv = ov;
          br = orr;
        }
      }
      if (lane == 0) {
        const double d0 = fabs((double)col[c]);
        int p = br;
        double pmax = bv;
        if (isnan(d0) || br == INT_MAX) {  // pmax starts at |a_jj|: NaN there keeps p = j
          p = c;
          pmax = d0;
        }
        s_bad = pmax < Pol::tiny;  // SingularInPrecision, band_lu.cpp:106-108
        s_p = p;
        if (s_bad) {
          err[1] = (int)j;
          err[0] = 1;
        } else {
          ipiv[j] = (int32_t)(j0 + p);
          if (p != c) err[3] = 1;  // a row interchange: the forward solve takes the swap-aware kernel
        }
      }
    }
    __syncthreads();
    if (s_bad) return;
    const int p = s_p;
    const int cmax = (int)lmin(nbw - 1, lmin(N - 1, j + ldoff) - j0);  // columns <= klast
    if (p != c)  // band_lu.cpp:110-113 (the trailing columns swap in k_lu_trail)
      for (int cc = c + tid; cc <= cmax; cc += nt) {
        const S t = Pm[cc * R + c];
        Pm[cc * R + c] = Pm[cc * R + p];
        Pm[cc * R + p] = t;
      }
    __syncthreads();
    const S piv = col[c];
    for (int r = c + 1 + tid; r <= rl; r += nt) {  // band_lu.cpp:115-126, one row per thread
      const S l = Pol::div(col[r], piv);
      col[r] = l;
      for (int cc = c + 1; cc <= cmax; ++cc) {
        const S a = Pm[cc * R + c];
        if (a != S(0)) Pm[cc * R + r] = Pol::sub(Pm[cc * R + r], Pol::mul(l, a));
      }
    }
    __syncthreads();
  }
  for (int c = 0; c < nbw; ++c) {
    const int64_t k = j0 + c;
    for (int r = tid; r < R; r += nt) {
      const int64_t d = ldoff + j0 + r - k;
      if (d >= 0 && d < ldab) ab[k * ldab + d] = Pm[c * R + r];
    }
  }
}

template <int P>
__global__ void __launch_bounds__(kTrailWarps * 32) k_lu_trail(typename LuPol<P>::S* __restrict__ ab, int64_t N,
                                                               int64_t kl, int64_t ku, int64_t ldab, int64_t j0,
                                                               int nbw, int R, const int32_t* __restrict__ ipiv,
                                                               const int* __restrict__ err, int64_t kfirst,
                                                               int64_t kend) {
  using Pol = LuPol<P>;
  using S = typename Pol::S;
  extern __shared__ __align__(16) unsigned char lu_smem[];
  __shared__ int pv[32];
  if (*(volatile int*)err) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  S* Lm = reinterpret_cast<S*>(lu_smem);  // the panel's multipliers, Lm[c*R + r]
  S* cb = Lm + (size_t)nbw * R + (size_t)warp * R;
  const int64_t ldoff = kl + ku;
  for (int c = 0; c < nbw; ++c) {
    const int64_t k = j0 + c;
    for (int r = c + 1 + tid; r < R; r += blockDim.x) Lm[c * R + r] = ab[k * ldab + ldoff + j0 + r - k];
  }
  if (tid < nbw) pv[tid] = ipiv[j0 + tid] - (int)j0;
  __syncthreads();
  for (int64_t k = kfirst + (int64_t)blockIdx.x * kTrailWarps + warp; k <= kend;
       k += (int64_t)gridDim.x * kTrailWarps) {
    const int rlo = (int)lmax(0, k - ldoff - j0), rhi = (int)lmin(R - 1, k + kl - j0);
    S* colk = ab + k * ldab + ldoff + j0 - k;  // colk[r] = A(j0+r, k)
    for (int r = rlo + lane; r <= rhi; r += 32) cb[r] = colk[r];
    __syncwarp();
    for (int c = 0; c < nbw; ++c) {
      const int64_t j = j0 + c;
      if (k > j + ldoff) continue;  // beyond klast(j): neither swapped nor updated at step j
      const int p = pv[c];
      if (p != c) {
        if (lane == 0) {
          const S t = cb[c];
          cb[c] = cb[p];
          cb[p] = t;
        }
        __syncwarp();
      }
      const S a = cb[c];
      if (a != S(0)) {  // band_lu.cpp:121-122
        const int rl = (int)(lmin(N - 1, j + kl) - j0);
        for (int r = c + 1 + lane; r <= rl; r += 32) cb[r] = Pol::sub(cb[r], Pol::mul(Lm[c * R + r], a));
      }
      __syncwarp();
    }
    for (int r = rlo + lane; r <= rhi; r += 32) colk[r] = cb[r];
    __syncwarp();
  }
}

template <class S>
__global__ void k_lu_nonfinite(const S* __restrict__ ab, int64_t n, int* err) {  // band_lu.cpp:132-134
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite((double)ab[t])) {
      err[0] = 2;
      return;
    }
}

// ------------------------------------------------------------------- solves
template <class T, class S>
__global__ void k_lu_in(const T* __restrict__ src, S* __restrict__ x, int64_t N) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) x[i] = (S)to_dbl(src[i]);  // from_double of a u_r value: exact
}

template <class T, class S>
__global__ void k_lu_out(const S* __restrict__ x, T* __restrict__ dst, int64_t N, int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const S v = x[i];
  dst[i] = from_dbl<T>((double)v);
  if (!isfinite((double)v)) *bad = 1;  // all_finite, solver.cpp:229
}

// forward sweep, band_lu.cpp:148-157
template <int P>
__global__ void __launch_bounds__(512, 1) k_lu_fwd(const typename LuPol<P>::S* __restrict__ ab, int64_t N,
                                                     int64_t kl, int64_t ku, int64_t ldab,
                                                     const int32_t* __restrict__ ipiv,
                                                     typename LuPol<P>::S* __restrict__ x) {
  using Pol = LuPol<P>;
  using S = typename Pol::S;
  __shared__ S xb[32];
  __shared__ int64_t tpos[32];
  __shared__ int64_t tat[32];
  __shared__ int ntab;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t ldoff = kl + ku;
  for (int64_t j0 = 0; j0 < N; j0 += 32) {
    const int nb = (int)lmin(32, N - j0);
    if (tid < 32) {
      S v = lane < nb ? x[j0 + lane] : S(0);
      S Lr[32];
#pragma unroll
      for (int c = 0; c < 32; ++c)
        Lr[c] = (c < lane && lane < nb && lane - c <= kl) ? ab[(j0 + c) * ldab + ldoff + lane - c] : S(0);
      const int pvl = lane < nb ? ipiv[j0 + lane] : 0;
      int cnt = 0;  // lane 0: swapped positions beyond the block and the step they are current through
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        if (c < nb) {
          const int64_t j = j0 + c;
          const int64_t p = __shfl_sync(~0u, pvl, c);
          if (p != j) {
            const S vc = __shfl_sync(~0u, v, c);
            if (p < j0 + nb) {
              const S vp = __shfl_sync(~0u, v, (int)(p - j0));
              if (lane == c) v = vp;
              if (lane == (int)(p - j0)) v = vc;
            } else {
              S val = S(0);
              if (lane == 0) {
                int slot = -1;
                int64_t at = j0 - 1;
                for (int t = 0; t < cnt; ++t)
                  if (tpos[t] == p) {
                    slot = t;
                    at = tat[t];
                  }
                val = x[p];
                for (int64_t jj = at + 1; jj < j; ++jj) {
                  const S xj = xb[jj - j0];
                  if (xj != S(0) && p <= jj + kl) val = Pol::sub(val, Pol::mul(ab[jj * ldab + ldoff + p - jj], xj));
                }
                x[p] = vc;
                if (slot < 0) slot = cnt++;
                tpos[slot] = p;
                tat[slot] = j - 1;
              }
              val = __shfl_sync(~0u, val, 0);
              if (lane == c) v = val;
            }
          }
          const S xj = __shfl_sync(~0u, v, c);
          if (lane == 0) xb[c] = xj;
          if (xj != S(0) && lane > c && lane < nb && lane - c <= kl) v = Pol::sub(v, Pol::mul(Lr[c], xj));
        }
      }
      if (lane < nb) x[j0 + lane] = v;
      if (lane == 0) ntab = cnt;
    }
    __syncthreads();
    const int64_t iend = lmin(N - 1, j0 + nb - 1 + kl);
    for (int64_t i = j0 + nb + tid; i <= iend; i += blockDim.x) {
      int64_t at = j0 - 1;
      for (int t = 0; t < ntab; ++t)
        if (tpos[t] == i) at = tat[t];
      const int c0 = (int)(at - j0 + 1);
      S l[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const int64_t j = j0 + c;
        l[c] = (c >= c0 && c < nb && i <= j + kl) ? ab[j * ldab + ldoff + i - j] : S(0);
      }
      S val = x[i];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const S xj = xb[c];
        if (c >= c0 && c < nb && xj != S(0) && i <= j0 + c + kl) val = Pol::sub(val, Pol::mul(l[c], xj));
      }
      x[i] = val;
    }
    __syncthreads();
  }
}

// back substitution, band_lu.cpp:159-167
template <int P>
__global__ void __launch_bounds__(512, 1) k_lu_bwd(const typename LuPol<P>::S* __restrict__ ab, int64_t N,
                                                     int64_t kl, int64_t ku, int64_t ldab,
                                                     typename LuPol<P>::S* __restrict__ x) {
  using Pol = LuPol<P>;
  using S = typename Pol::S;
  __shared__ S xb[32];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t ldoff = kl + ku;  // ubw
  for (int64_t jhi = N - 1; jhi >= 0; jhi -= 32) {
    const int64_t jlo = lmax(0, jhi - 31);
    const int nb = (int)(jhi - jlo + 1);
    if (tid < 32) {
      S v = lane < nb ? x[jlo + lane] : S(0);
      const S dg = lane < nb ? ab[(jlo + lane) * ldab + ldoff] : S(1);
      S Ur[32];
#pragma unroll
      for (int c = 0; c < 32; ++c)
        Ur[c] = (lane < c && c < nb && c - lane <= ldoff) ? ab[(jlo + c) * ldab + ldoff + lane - c] : S(0);
#pragma unroll
      for (int c = 31; c >= 0; --c) {
        if (c < nb) {
          if (lane == c) v = Pol::div(v, dg);
          const S xj = __shfl_sync(~0u, v, c);
          if (lane == 0) xb[c] = xj;
          if (xj != S(0) && lane < c && c - lane <= ldoff) v = Pol::sub(v, Pol::mul(Ur[c], xj));
        }
      }
      if (lane < nb) x[jlo + lane] = v;
    }
    __syncthreads();
    const int64_t ifirst = lmax(0, jlo - ldoff);
    for (int64_t i = ifirst + tid; i < jlo; i += blockDim.x) {
      S u[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const int64_t j = jlo + c;
        u[c] = (c < nb && j - i <= ldoff) ? ab[j * ldab + ldoff + i - j] : S(0);
      }
      S val = x[i];
#pragma unroll
      for (int c = 31; c >= 0; --c) {
        const S xj = xb[c];
        if (c < nb && xj != S(0) && jlo + c - i <= ldoff) val = Pol::sub(val, Pol::mul(u[c], xj));
      }
      x[i] = val;
    }
    __syncthreads();
  }
}

// ------------------------------------------------- pipelined solves (no swaps)
// Without row interchanges (ipiv[j] == j: every H, and S whenever it is
// column diagonally dominant) element i of the forward sweep receives exactly
// the updates x_i -= L(i,j) x_j for j = i-kl .. i-1 ascending (skipping
// x_j == 0), and element i of the back sweep x_i -= U(i,j) x_j for j =
// i+ubw .. i+1 descending, then x_i /= U(i,i) (band_lu.cpp:148-167). That
// per-element sequence does not depend on how the sweep is scheduled, so the
// 32-position blocks are processed by many CTAs at once: a CTA claims the next
// block in sweep order from a ticket (claimed blocks only wait on earlier
// claimed blocks: no deadlock whatever else runs on the device), applies the
// updates of each earlier block as soon as its flag carries this solve's
// epoch, runs its own 32 x 32 triangle through shuffles, publishes x and
// raises its flag. The band reads are coalesced: for a fixed column the 32
// lanes read 32 consecutive band rows.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int P, bool FWD, int POS>
__global__ void __launch_bounds__(32) k_lu_pipe(const typename LuPol<P>::S* __restrict__ ab, int64_t N, int64_t kl,
                                                int64_t ku, int64_t ldab, typename LuPol<P>::S* x,
                                                unsigned* __restrict__ flags, unsigned* __restrict__ ticket,
                                                unsigned epoch) {
  // a block is B = 32*POS positions; lane l owns positions B*b + l + 32p (p < POS)
  using Pol = LuPol<P>;
  using S = typename Pol::S;
  constexpr int B = 32 * POS;
  const int lane = threadIdx.x;
  const int64_t ldoff = kl + ku, nblk = (N + B - 1) / B, reach = FWD ? kl : ldoff;
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1u);
    t = __shfl_sync(~0u, t, 0);
    if ((int64_t)t >= nblk) return;
    const int64_t b = FWD ? (int64_t)t : nblk - 1 - (int64_t)t;
    int64_t ip[POS];
    S v[POS];
#pragma unroll
    for (int p = 0; p < POS; ++p) {
      ip[p] = B * b + lane + 32 * p;
      v[p] = ip[p] < N ? x[ip[p]] : S(0);
    }
    // earlier blocks in sweep order whose columns reach this block
    const int64_t dlo = FWD ? (B * b - reach > 0 ? (B * b - reach) / B : 0) : b + 1;
    const int64_t dhi = FWD ? b - 1 : (B * b + B - 1 + reach < N - 1 ? (B * b + B - 1 + reach) / B : nblk - 1);
    for (int64_t s = 0; s <= dhi - dlo; ++s) {
      const int64_t d = FWD ? dlo + s : dhi - s;  // ascending j (forward), descending j (back)
#pragma unroll
      for (int kk = 0; kk < POS; ++kk) {
        const int ch = FWD ? kk : POS - 1 - kk;  // 32-column chunk of block d
        S m[POS][32];
#pragma unroll
        for (int p = 0; p < POS; ++p)
#pragma unroll
          for (int c = 0; c < 32; ++c) {  // the band entries, issued before the wait
            const int64_t j = B * d + 32 * ch + c;
            const int64_t off = FWD ? ip[p] - j : j - ip[p];
            m[p][c] = (ip[p] < N && j < N && off >= 1 && off <= reach) ? ab[j * ldab + ldoff + ip[p] - j] : S(0);
          }
        if (kk == 0)
          while (ld_acquire(flags + d) != epoch) {
          }
        const S xd = (B * d + 32 * ch + lane < N) ? __ldcg(x + B * d + 32 * ch + lane) : S(0);
#pragma unroll
        for (int cc = 0; cc < 32; ++cc) {
          const int c = FWD ? cc : 31 - cc;
          const int64_t j = B * d + 32 * ch + c;
          const S xj = __shfl_sync(~0u, xd, c);
#pragma unroll
          for (int p = 0; p < POS; ++p) {
            const int64_t off = FWD ? ip[p] - j : j - ip[p];
            if (ip[p] < N && xj != S(0) && j < N && off >= 1 && off <= reach) v[p] = Pol::sub(v[p], Pol::mul(m[p][c], xj));
          }
        }
      }
    }
    // own triangle, chunk by chunk in sweep order
#pragma unroll
    for (int kk = 0; kk < POS; ++kk) {
      const int ch = FWD ? kk : POS - 1 - kk;
      S m[POS][32];
#pragma unroll
      for (int p = 0; p < POS; ++p)
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int64_t j = B * b + 32 * ch + c;
          const int64_t off = FWD ? ip[p] - j : j - ip[p];
          m[p][c] = (ip[p] < N && j < N && off >= 0 && off <= reach) ? ab[j * ldab + ldoff + ip[p] - j] : S(1);
        }
#pragma unroll
      for (int cc = 0; cc < 32; ++cc) {
        const int c = FWD ? cc : 31 - cc;
        const int64_t j = B * b + 32 * ch + c;
        if (j < N) {
          if (!FWD && lane == c) v[ch] = Pol::div(v[ch], m[ch][c]);  // U(j,j)
          const S xj = __shfl_sync(~0u, v[ch], c);
#pragma unroll
          for (int p = 0; p < POS; ++p) {
            const int64_t off = FWD ? ip[p] - j : j - ip[p];
            if (ip[p] < N && xj != S(0) && off >= 1 && off <= reach) v[p] = Pol::sub(v[p], Pol::mul(m[p][c], xj));
          }
        }
      }
    }
#pragma unroll
    for (int p = 0; p < POS; ++p)
      if (ip[p] < N) x[ip[p]] = v[p];
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(flags + b, epoch);
  }
}

// The same sweeps for binary32 slots (u_r = half / single) without flags or
// fences: every x value is published as one 64-bit word (value bits | epoch
// << 32), written once with a single-copy-atomic store; a consumer lane polls
// exactly the word it needs until the epoch matches. Each dependent hop is one
// L2 round trip instead of store + fence + flag + load.
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int P, bool FWD>
__global__ void __launch_bounds__(32) k_lu_pipe_t(const float* __restrict__ ab, int64_t N, int64_t kl, int64_t ku,
                                                  int64_t ldab, const float* __restrict__ x0,
                                                  unsigned long long* xt, unsigned* __restrict__ ticket,
                                                  unsigned epoch) {
  using Pol = LuPol<P>;
  const int lane = threadIdx.x;
  const int64_t ldoff = kl + ku, nblk = (N + 31) / 32, reach = FWD ? kl : ldoff;
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1u);
    t = __shfl_sync(~0u, t, 0);
    if ((int64_t)t >= nblk) return;
    const int64_t b = FWD ? (int64_t)t : nblk - 1 - (int64_t)t;
    const int64_t i = 32 * b + lane;
    const bool live = i < N;
    float v = live ? (FWD ? x0[i] : __uint_as_float((unsigned)xt[i])) : 0.f;
    const int64_t dlo = FWD ? (32 * b - reach > 0 ? (32 * b - reach) / 32 : 0) : b + 1;
    const int64_t dhi = FWD ? b - 1 : (32 * b + 31 + reach < N - 1 ? (32 * b + 31 + reach) / 32 : nblk - 1);
    for (int64_t s = 0; s <= dhi - dlo; ++s) {
      const int64_t d = FWD ? dlo + s : dhi - s;
      float m[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const int64_t j = 32 * d + c;
        const int64_t off = FWD ? i - j : j - i;
        m[c] = (live && j < N && off >= 1 && off <= reach) ? ab[j * ldab + ldoff + i - j] : 0.f;
      }
      float xd = 0.f;
      if (32 * d + lane < N) {
        unsigned long long w;
        do {
          w = ld_relaxed64(xt + 32 * d + lane);
        } while ((unsigned)(w >> 32) != epoch);
        xd = __uint_as_float((unsigned)w);
      }
#pragma unroll
      for (int cc = 0; cc < 32; ++cc) {
        const int c = FWD ? cc : 31 - cc;
        const int64_t j = 32 * d + c;
        const int64_t off = FWD ? i - j : j - i;
        const float xj = __shfl_sync(~0u, xd, c);
        if (live && xj != 0.f && j < N && off >= 1 && off <= reach) v = Pol::sub(v, Pol::mul(m[c], xj));
      }
    }
    float m[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const int64_t j = 32 * b + c;
      const int64_t off = FWD ? i - j : j - i;
      m[c] = (live && j < N && off >= 0 && off <= reach && (FWD ? off >= 1 : true)) ? ab[j * ldab + ldoff + i - j] : 1.f;
    }
#pragma unroll
    for (int cc = 0; cc < 32; ++cc) {
      const int c = FWD ? cc : 31 - cc;
      const int64_t j = 32 * b + c;
      if (j < N) {
        if (!FWD && lane == c) v = Pol::div(v, m[c]);
        const float xj = __shfl_sync(~0u, v, c);
        const int64_t off = FWD ? i - j : j - i;
        if (live && xj != 0.f && off >= 1 && off <= reach) v = Pol::sub(v, Pol::mul(m[c], xj));
      }
    }
    if (live) st_relaxed64(xt + i, ((unsigned long long)epoch << 32) | __float_as_uint(v));
  }
}

__global__ void k_lu_untag(const unsigned long long* __restrict__ xt, float* __restrict__ x, int64_t N) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) x[i] = __uint_as_float((unsigned)xt[i]);
}
__global__ void k_lu_tag(const float* __restrict__ x, unsigned long long* __restrict__ xt, int64_t N) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) xt[i] = __float_as_uint(x[i]);  // epoch 0: never a solve's epoch
}

template <class S>
inline void pick_panel(int64_t kl, int& nb) {
  nb = 32;
  while (nb > 1 && (size_t)(nb + kTrailWarps) * (size_t)(nb + kl) * sizeof(S) > kSmemBudget) nb >>= 1;
  if ((size_t)(nb + kTrailWarps) * (size_t)(nb + kl) * sizeof(S) > kSmemBudget)
    throw Err(GADI_E_UNSUPPORTED, "lu_direct: the lower bandwidth " + std::to_string(kl) +
                                      " is too wide for the device band LU (shared-memory panel)");
}

template <int P>
int factor_impl(LuFactor* f, cudaStream_t s) {
  using S = typename LuPol<P>::S;
  const int64_t N = f->N, kl = f->kl, ku = f->ku, ldab = f->ldab;
  int nb;
  pick_panel<S>(kl, nb);
  S* ab = static_cast<S*>(f->ab);
  const size_t smem_max = (size_t)(nb + kTrailWarps) * (size_t)(nb + kl) * sizeof(S);
  smem_attr(k_lu_panel<P>, smem_max);
  smem_attr(k_lu_trail<P>, smem_max);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, f->device);
  for (int64_t j0 = 0; j0 < N; j0 += nb) {
    const int nbw = (int)std::min<int64_t>(nb, N - j0);
    const int R = (int)(std::min<int64_t>(N - 1, j0 + nbw - 1 + kl) - j0 + 1);
    k_lu_panel<P><<<1, kPanelThreads, (size_t)nbw * R * sizeof(S), s>>>(ab, N, kl, ku, ldab, j0, nbw, R, f->ipiv,
                                                                        f->err);
    const int64_t kfirst = j0 + nbw, kend = std::min<int64_t>(N - 1, j0 + nbw - 1 + kl + ku);
    if (kfirst <= kend) {
      const int64_t cols = kend - kfirst + 1;
      const unsigned grid = (unsigned)std::min<int64_t>((cols + kTrailWarps - 1) / kTrailWarps, sms);
      k_lu_trail<P><<<grid, kTrailWarps * 32, (size_t)(nbw + kTrailWarps) * R * sizeof(S), s>>>(
          ab, N, kl, ku, ldab, j0, nbw, R, f->ipiv, f->err, kfirst, kend);
    }
    f->launches += 2;
  }
  CKL();
  int herr[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(herr, f->err, sizeof(herr), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (herr[0] == 1) return GADI_SINGULAR_IN_PRECISION;
  f->swaps = herr[3] != 0;
  f->sms = sms;
  k_lu_nonfinite<S><<<(unsigned)sms * 4, 256, 0, s>>>(ab, ldab * N, f->err);
  CKL();
  ++f->launches;
  CK(cudaMemcpyAsync(herr, f->err, sizeof(herr), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return herr[0] == 2 ? GADI_OVERFLOW_DETECTED : 0;
}

template <int P, class T>
void solve_impl(LuFactor* f, const void* rhs, void* x, cudaStream_t s) {
  using S = typename LuPol<P>::S;
  const int64_t N = f->N;
  S* xw = static_cast<S*>(f->xw);
  const S* ab = static_cast<const S*>(f->ab);
  const unsigned g = (unsigned)((N + 255) / 256);
  k_lu_in<T, S><<<g, 256, 0, s>>>(static_cast<const T*>(rhs), xw, N);
  // 32-position blocks (one per lane); GADI_LU_POS=2 selects 64 (two per lane: half the dependent
  // hops, but 3x slower at C1 -- register spills and twice the per-block work)
  static const int pos_env = std::getenv("GADI_LU_POS") ? std::atoi(std::getenv("GADI_LU_POS")) : 0;
  const int pos = pos_env == 2 ? 2 : 1;
  const int64_t nblk = (N + 32 * pos - 1) / (32 * pos);
  const unsigned grid = (unsigned)std::min<int64_t>(nblk, (int64_t)f->sms * 16);
  auto pipe = [&](auto fwd) {
    constexpr bool F = decltype(fwd)::value;
    CK(cudaMemsetAsync(f->ticket, 0, sizeof(unsigned), s));
    if (pos == 2)
      k_lu_pipe<P, F, 2><<<grid, 32, 0, s>>>(ab, N, f->kl, f->ku, f->ldab, xw, f->flags, f->ticket, ++f->epoch);
    else
      k_lu_pipe<P, F, 1><<<grid, 32, 0, s>>>(ab, N, f->kl, f->ku, f->ldab, xw, f->flags, f->ticket, ++f->epoch);
  };
  if constexpr (!std::is_same<S, double>::value) {  // binary32 slots: tagged words, no flags
    static const bool tagged = !(std::getenv("GADI_LU_TAGGED") && std::getenv("GADI_LU_TAGGED")[0] == '0');
    if (tagged && pos == 1) {
      const unsigned gN = (unsigned)((N + 255) / 256);
      if (f->swaps) {
        k_lu_fwd<P><<<1, 512, 0, s>>>(ab, N, f->kl, f->ku, f->ldab, f->ipiv, xw);
        k_lu_tag<<<gN, 256, 0, s>>>(xw, f->xt, N);
      } else {
        CK(cudaMemsetAsync(f->ticket, 0, sizeof(unsigned), s));
        k_lu_pipe_t<P, true><<<grid, 32, 0, s>>>(ab, N, f->kl, f->ku, f->ldab, xw, f->xt, f->ticket, ++f->epoch);
      }
      CK(cudaMemsetAsync(f->ticket, 0, sizeof(unsigned), s));
      k_lu_pipe_t<P, false><<<grid, 32, 0, s>>>(ab, N, f->kl, f->ku, f->ldab, xw, f->xt, f->ticket, ++f->epoch);
      k_lu_untag<<<gN, 256, 0, s>>>(f->xt, xw, N);
      k_lu_out<T, S><<<g, 256, 0, s>>>(xw, static_cast<T*>(x), N, f->bad);
      CKL();
      f->launches += 5;
      return;
    }
  }
  if (f->swaps)  // row interchanges in the forward sweep: one CTA (k_lu_fwd handles the swaps)
    k_lu_fwd<P><<<1, 512, 0, s>>>(ab, N, f->kl, f->ku, f->ldab, f->ipiv, xw);
  else
    pipe(std::true_type{});
  pipe(std::false_type{});
  k_lu_out<T, S><<<g, 256, 0, s>>>(xw, static_cast<T*>(x), N, f->bad);
  CKL();
  f->launches += 4;
}

// Many right-hand sides against one (small-band) factor, one thread each:
// the reference's solve_impl (band_lu.cpp:137-172) verbatim, swaps included.
// Element t of right-hand side r is X[r*rs + t*es] (binary64 slots holding
// u_r values, like the reference's Vector); bad = 1 on a non-finite result.
template <int P>
__global__ void k_lu_solve_many(const typename LuPol<P>::S* __restrict__ ab, int64_t N, int64_t kl, int64_t ku,
                                int64_t ldab, const int32_t* __restrict__ ipiv, double* __restrict__ X, int64_t es,
                                int64_t rs, int64_t nrhs, int* bad) {
  using Pol = LuPol<P>;
  using S = typename Pol::S;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrhs) return;
  double* x = X + r * rs;
  const int64_t ldoff = kl + ku;
  for (int64_t j = 0; j < N; ++j) {
    const int64_t p = ipiv[j];
    if (p != j) {
      const double t = x[j * es];
      x[j * es] = x[p * es];
      x[p * es] = t;
    }
    const S xj = (S)x[j * es];
    if (xj == S(0)) continue;
    const int64_t ilast = lmin(N - 1, j + kl);
    for (int64_t i = j + 1; i <= ilast; ++i)
      x[i * es] = (double)Pol::sub((S)x[i * es], Pol::mul(ab[j * ldab + ldoff + i - j], xj));
  }
  bool fin = true;
  for (int64_t j = N - 1; j >= 0; --j) {
    const S xj = Pol::div((S)x[j * es], ab[j * ldab + ldoff]);
    x[j * es] = (double)xj;
    fin = fin && isfinite((double)xj);
    if (xj != S(0))
      for (int64_t i = lmax(0, j - ldoff); i < j; ++i)
        x[i * es] = (double)Pol::sub((S)x[i * es], Pol::mul(ab[j * ldab + ldoff + i - j], xj));
  }
  if (!fin) *bad = 1;
}

}  // namespace

// Builds and factors the band image of H (which = 1) or S (which = 2) of the
// regularized pair in u_r (prepare, solver.cpp:204-207). Returns the factor
// and sets *status to 0 or the SolveStatus of the reference's exception.
LuFactor* lu_factor_build(gadi_handle* h, int which, double alpha, int ur, int* status) {
  if (h->sharded()) throw Err(GADI_E_UNSUPPORTED, "lu_direct: not on a shard (the band LU is one device)");
  std::unique_ptr<LuFactor> f(new LuFactor);
  f->device = h->device;
  f->prec = ur;
  f->N = h->N;
  if (h->stencil()) {
    f->kl = f->ku = h->n > 1 ? h->n * h->n : 0;  // the i-1 / i+1 neighbours
  } else {  // lower/upper_bandwidth of the union pattern (sparse.cpp:142-154)
    unsigned long long* bw = nullptr;
    CK(cudaMallocFromPoolAsync((void**)&bw, 16, engine_pool(f->device), h->stream));
    CK(cudaMemsetAsync(bw, 0, 16, h->stream));
    const auto pt = h->part(which);  // the operator's own pattern (the HSS union, or an explicit M / N)
    k_bandwidths<<<(unsigned)((h->N + 255) / 256), 256, 0, h->stream>>>(h->N, pt.rp, pt.ci, bw);
    CKL();
    unsigned long long hb[2];
    CK(cudaMemcpyAsync(hb, bw, 16, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    cudaFreeAsync(bw, h->stream);
    f->kl = (int64_t)hb[0];
    f->ku = (int64_t)hb[1];
  }
  f->ldab = 2 * f->kl + f->ku + 1;
  const size_t es = ur == GADI_DOUBLE ? 8 : 4;
  cudaStream_t s = h->stream;
  // stream-ordered allocations: concurrent handles (gadi_train.cu) never wait on each other here
  CK(cudaMallocFromPoolAsync(&f->ab, (size_t)f->ldab * (size_t)f->N * es, engine_pool(f->device), s));
  CK(cudaMemsetAsync(f->ab, 0, (size_t)f->ldab * (size_t)f->N * es, s));
  CK(cudaMallocFromPoolAsync((void**)&f->ipiv, (size_t)f->N * sizeof(int32_t), engine_pool(f->device), s));
  CK(cudaMallocFromPoolAsync(&f->xw, (size_t)f->N * es, engine_pool(f->device), s));
  CK(cudaMallocFromPoolAsync((void**)&f->err, 4 * sizeof(int), engine_pool(f->device), s));
  CK(cudaMemsetAsync(f->err, 0, 4 * sizeof(int), s));
  CK(cudaMallocFromPoolAsync((void**)&f->flags, (size_t)((f->N + 31) / 32 + 1) * sizeof(unsigned), engine_pool(f->device), s));
  CK(cudaMemsetAsync(f->flags, 0, (size_t)((f->N + 31) / 32 + 1) * sizeof(unsigned), s));
  f->ticket = f->flags + (f->N + 31) / 32;
  CK(cudaMallocFromPoolAsync((void**)&f->xt, (size_t)f->N * 8, engine_pool(f->device), s));
  CK(cudaMemsetAsync(f->xt, 0, (size_t)f->N * 8, s));  // epoch 0 on every word
  f->bad = f->err + 2;
  const int64_t ldoff = f->kl + f->ku, N = f->N;
  const unsigned g = (unsigned)((N + 255) / 256);
  if (h->stencil()) {
    // regularize of the HSS split (splitting.cpp:12-20,37-47) in closed form, as Engine::build_ops
    const double t1 = h->t1, t2 = h->t2, t3 = h->t3;
    double lo, dg, up;
    if (which == 1) {
      lo = 0.5 * t2 + 0.5 * t3;
      up = 0.5 * t3 + 0.5 * t2;
      dg = 1.0 * (0.5 * t1 + 0.5 * t1) + alpha;
    } else {
      lo = 0.5 * t2 + -0.5 * t3;
      up = 0.5 * t3 + -0.5 * t2;
      dg = 1.0 * (0.5 * t1 + -0.5 * t1) + alpha;
    }
    lo = hround(lo, ur);
    dg = hround(dg, ur);
    up = hround(up, ur);
    if (ur == GADI_DOUBLE)
      k_band_stencil<double><<<g, 256, 0, s>>>((double*)f->ab, h->n, N, ldoff, f->ldab, lo, dg, up);
    else
      k_band_stencil<float><<<g, 256, 0, s>>>((float*)f->ab, h->n, N, ldoff, f->ldab, lo, dg, up);
  } else {
    const auto pt = h->part(which);
    if (ur == GADI_DOUBLE)
      k_band_csr<double, P_DOUBLE><<<g, 256, 0, s>>>((double*)f->ab, N, ldoff, f->ldab, pt.rp, pt.ci, pt.v, pt.dpos,
                                                       pt.din, alpha);
    else if (ur == GADI_SINGLE)
      k_band_csr<float, P_SINGLE><<<g, 256, 0, s>>>((float*)f->ab, N, ldoff, f->ldab, pt.rp, pt.ci, pt.v, pt.dpos,
                                                      pt.din, alpha);
    else
      k_band_csr<float, P_HALF><<<g, 256, 0, s>>>((float*)f->ab, N, ldoff, f->ldab, pt.rp, pt.ci, pt.v, pt.dpos,
                                                    pt.din, alpha);
  }
  CKL();
  ++f->launches;
  *status = ur == GADI_DOUBLE ? factor_impl<GADI_DOUBLE>(f.get(), s)
            : ur == GADI_SINGLE ? factor_impl<GADI_SINGLE>(f.get(), s)
                                : factor_impl<GADI_HALF>(f.get(), s);
  return f.release();
}

// BandLU of shift_diagonal(M, alpha) (sparse.cpp:180-183: the diagonal is
// 1.0*M_ii + alpha, or alpha where M has none) for a small host CSR M, in u_r
// (the Sylvester coefficients' factorizations, sylvester.cpp:66-73).
LuFactor* lu_factor_host_csr(int device, cudaStream_t s, int64_t N, const int64_t* rp, const int64_t* ci,
                             const double* v, double alpha, int ur, int* status) {
  std::unique_ptr<LuFactor> f(new LuFactor);
  f->device = device;
  f->prec = ur;
  f->N = N;
  int64_t kl = 0, ku = 0;
  for (int64_t i = 0; i < N; ++i) {  // bandwidths of the shifted pattern (it has every diagonal)
    const int64_t c0 = rp[i] < rp[i + 1] ? std::min<int64_t>(ci[rp[i]], i) : i;
    const int64_t c1 = rp[i] < rp[i + 1] ? std::max<int64_t>(ci[rp[i + 1] - 1], i) : i;
    kl = std::max(kl, i - c0);
    ku = std::max(ku, c1 - i);
  }
  f->kl = kl;
  f->ku = ku;
  f->ldab = 2 * kl + ku + 1;
  const int64_t ldoff = kl + ku;
  std::vector<double> band((size_t)(f->ldab * N), 0.0);
  for (int64_t i = 0; i < N; ++i) {
    bool diag = false;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      double x = 1.0 * v[k];
      if (ci[k] == i) {
        x = 1.0 * v[k] + alpha;
        diag = true;
      }
      band[(size_t)(ci[k] * f->ldab + ldoff + i - ci[k])] = hround(x, ur);
    }
    if (!diag) band[(size_t)(i * f->ldab + ldoff)] = hround(alpha, ur);
  }
  const size_t es = ur == GADI_DOUBLE ? 8 : 4;
  CK(cudaMallocFromPoolAsync(&f->ab, band.size() * es, engine_pool(f->device), s));
  if (ur == GADI_DOUBLE) {
    CK(cudaMemcpyAsync(f->ab, band.data(), band.size() * 8, cudaMemcpyHostToDevice, s));
  } else {
    std::vector<float> bf(band.begin(), band.end());
    CK(cudaMemcpyAsync(f->ab, bf.data(), bf.size() * 4, cudaMemcpyHostToDevice, s));
  }
  CK(cudaMallocFromPoolAsync((void**)&f->ipiv, (size_t)N * sizeof(int32_t), engine_pool(f->device), s));
  CK(cudaMallocFromPoolAsync(&f->xw, (size_t)N * es, engine_pool(f->device), s));
  CK(cudaMallocFromPoolAsync((void**)&f->err, 4 * sizeof(int), engine_pool(f->device), s));
  CK(cudaMemsetAsync(f->err, 0, 4 * sizeof(int), s));
  CK(cudaMallocFromPoolAsync((void**)&f->flags, (size_t)((N + 31) / 32 + 1) * sizeof(unsigned), engine_pool(f->device), s));
  CK(cudaMemsetAsync(f->flags, 0, (size_t)((N + 31) / 32 + 1) * sizeof(unsigned), s));
  f->ticket = f->flags + (N + 31) / 32;
  CK(cudaMallocFromPoolAsync((void**)&f->xt, (size_t)N * 8, engine_pool(f->device), s));
  CK(cudaMemsetAsync(f->xt, 0, (size_t)N * 8, s));
  f->bad = f->err + 2;
  *status = ur == GADI_DOUBLE ? factor_impl<GADI_DOUBLE>(f.get(), s)
            : ur == GADI_SINGLE ? factor_impl<GADI_SINGLE>(f.get(), s)
                                : factor_impl<GADI_HALF>(f.get(), s);
  return f.release();
}

// x_r = F \ x_r for nrhs right-hand sides in place (binary64 slots of u_r
// values); element t of r at X[r*rs + t*es]. Returns true if all finite.
bool lu_solve_many(LuFactor* f, double* X, int64_t es, int64_t rs, int64_t nrhs, cudaStream_t s) {
  CK(cudaMemsetAsync(f->bad, 0, sizeof(int), s));
  const unsigned g = (unsigned)((nrhs + 127) / 128);
  if (f->prec == GADI_DOUBLE)
    k_lu_solve_many<GADI_DOUBLE><<<g, 128, 0, s>>>((const double*)f->ab, f->N, f->kl, f->ku, f->ldab, f->ipiv, X, es,
                                                  rs, nrhs, f->bad);
  else if (f->prec == GADI_SINGLE)
    k_lu_solve_many<GADI_SINGLE><<<g, 128, 0, s>>>((const float*)f->ab, f->N, f->kl, f->ku, f->ldab, f->ipiv, X, es,
                                                  rs, nrhs, f->bad);
  else
    k_lu_solve_many<GADI_HALF><<<g, 128, 0, s>>>((const float*)f->ab, f->N, f->kl, f->ku, f->ldab, f->ipiv, X, es,
                                                rs, nrhs, f->bad);
  CKL();
  ++f->launches;
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, f->bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return bad == 0;
}

void lu_release(LuFactor* f, cudaStream_t s) {
  if (!f) return;
  for (void* p : {f->ab, (void*)f->ipiv, f->xw, (void*)f->err, (void*)f->flags, (void*)f->xt})
    if (p) {
      if (s) cudaFreeAsync(p, s);
      else cudaFree(p);  // synchronous: the owner may not have synchronised its stream
    }
  delete f;
}

// inner_solve LuDirect (solver.cpp:226-231): x = solve_factored(rhs) in u_r,
// Overflow when x is not finite; rhs / x in the engine's u_r storage.
InnerOut lu_inner_solve(LuFactor* f, const void* rhs, void* x, cudaStream_t s) {
  CK(cudaMemsetAsync(f->bad, 0, sizeof(int), s));
  if (f->prec == GADI_DOUBLE) solve_impl<GADI_DOUBLE, double>(f, rhs, x, s);
  else if (f->prec == GADI_SINGLE) solve_impl<GADI_SINGLE, float>(f, rhs, x, s);
  else solve_impl<GADI_HALF, __half>(f, rhs, x, s);
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, f->bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  InnerOut o;
  o.iters = 0;
  o.status = bad ? INNER_OVERFLOW : INNER_CONVERGED;
  return o;
}

}  // namespace gadi_host
