// gadi_gpr_dense.cuh — the binary64 dense kernels of the GPR fit (gpr.cpp:84-105:
// Gram matrix, LLT, K^-1 y, log det) and of the binary64 prediction path,
// hand-written for sm_100a (no cuSOLVER / cuBLAS).
//
// Blocked right-looking Cholesky on a row-major mp x mp matrix (mp a multiple
// of 128, the lower triangle is referenced): per 128-column block
//   k_potrf128      the diagonal block, one CTA, column by column in shared memory
//   k_trsm_right    the panel below it: rows of W21 L_jj^-T by substitution
//   k_dgemm<NT>     the trailing update W22 -= L21 L21^T (lower tiles only)
// The explicit inverse factor X = L^-1 the tensor-core variance GEMM consumes
// (gadi_gpr_umma.cuh) is a right-looking block substitution on the identity:
//   k_trsm_left     X_i,: = L_ii^-1 X_i,:      k_dgemm<NN>   X_r,: -= L_r,i X_i,:
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace gpr_dev {

constexpr int NB = 128;  // block size of the factorization

// K (row-major = column-major: symmetric) = sf2 exp(-0.5 d^2), d = (x_i - x_j)/l
// (gpr.cpp:70-73); diagonal += sn2 + 1e-12 max(1, sf2) (gpr.cpp:88). Rows and
// columns >= m (padding to a multiple of 128) are those of the identity.
__global__ void k_gram(const double* __restrict__ x, int m, int mp, double sf2, double ell, double jitter,
                       double* __restrict__ K) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)mp * mp) return;
  const int i = (int)(idx / mp), j = (int)(idx % mp);
  double v;
  if (i >= m || j >= m) {
    v = i == j ? 1.0 : 0.0;
  } else {
    const double d = __ddiv_rn(__dsub_rn(x[i], x[j]), ell);
    v = __dmul_rn(sf2, exp(__dmul_rn(-0.5, __dmul_rn(d, d))));
    if (i == j) v = __dadd_rn(v, jitter);
  }
  K[idx] = v;
}

// Cholesky of the 128 x 128 diagonal block at (j0, j0), in place (lower).
// info: 0, or 1 + the first column whose pivot is not positive (Eigen's
// NumericalIssue, gpr.cpp:92). One CTA of 256 threads; shared: 128 x 129 doubles.
__global__ void __launch_bounds__(256) k_potrf128(double* __restrict__ W, int ld, int j0, int* __restrict__ info) {
  extern __shared__ double sA[];  // [128][129]
  __shared__ double scol[NB];
  __shared__ int bad;
  const int t = threadIdx.x;
  if (t == 0) bad = 0;
  for (int e = t; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    sA[r * 129 + c] = c <= r ? W[(size_t)(j0 + r) * ld + j0 + c] : 0.0;
  }
  __syncthreads();
  const int r = t & 127, half = t >> 7;
  for (int c = 0; c < NB; ++c) {
    const double d = sA[c * 129 + c];
    if (!(d > 0.0)) {  // uniform: every thread reads the same pivot
      if (t == 0) bad = c + 1;
      break;
    }
    const double sd = sqrt(d);
    if (half == 0 && r >= c) scol[r] = r == c ? sd : __ddiv_rn(sA[r * 129 + c], sd);
    __syncthreads();
    if (r > c) {
      const double lr = scol[r];
      for (int cc = c + 1 + half; cc <= r; cc += 2) sA[r * 129 + cc] = fma(-lr, scol[cc], sA[r * 129 + cc]);
    }
    if (half == 0 && r >= c) sA[r * 129 + c] = scol[r];
    __syncthreads();
  }
  __syncthreads();
  if (bad) {
    if (t == 0) atomicCAS(info, 0, j0 + bad);
    return;
  }
  for (int e = t; e < NB * NB; e += 256) {
    const int rr = e / NB, c = e % NB;
    if (c <= rr) W[(size_t)(j0 + rr) * ld + j0 + c] = sA[rr * 129 + c];
  }
}

// Lower-packed copy of a 128 x 128 diagonal block in shared memory
__device__ __forceinline__ int pk(int r, int c) { return r * (r + 1) / 2 + c; }
__device__ __forceinline__ void load_diag_packed(const double* __restrict__ W, int ld, int j0, double* sL) {
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    if (c <= r) sL[pk(r, c)] = W[(size_t)(j0 + r) * ld + j0 + c];
  }
}

// Panel: rows [r0, r0 + nrows) of the block column j0 become W21 L_jj^-T, in
// place: l_rc = (w_rc - sum_{k<c} l_rk L_ck) / L_cc. One thread per row, 64
// rows per CTA staged in shared memory. Shared: 8256 + 64*129 doubles.
__global__ void __launch_bounds__(64) k_trsm_right(double* __restrict__ W, int ld, int j0, int r0, int nrows) {
  extern __shared__ double sm[];
  double* sL = sm;
  double* sT = sm + NB * (NB + 1) / 2;  // [64][129]
  load_diag_packed(W, ld, j0, sL);
  const int rb = r0 + blockIdx.x * 64;
  for (int e = threadIdx.x; e < 64 * NB; e += 64) {
    const int r = e / NB, c = e % NB;
    sT[r * 129 + c] = rb + r < r0 + nrows ? W[(size_t)(rb + r) * ld + j0 + c] : 0.0;
  }
  __syncthreads();
  double* row = sT + threadIdx.x * 129;
  for (int c = 0; c < NB; ++c) {
    double a0 = row[c], a1 = 0.0;
    const double* Lc = sL + pk(c, 0);
    int k = 0;
    for (; k + 1 < c; k += 2) {
      a0 = fma(-row[k], Lc[k], a0);
      a1 = fma(-row[k + 1], Lc[k + 1], a1);
    }
    if (k < c) a0 = fma(-row[k], Lc[k], a0);
    row[c] = __ddiv_rn(a0 + a1, Lc[c]);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 64 * NB; e += 64) {
    const int r = e / NB, c = e % NB;
    if (rb + r < r0 + nrows) W[(size_t)(rb + r) * ld + j0 + c] = sT[r * 129 + c];
  }
}

// X[i0 .. i0+128, c0 .. c0+ncols) = L_ii^-1 X[same], in place (L_ii the
// diagonal block of L at i0): x_r = (x_r - sum_{k<r} L_rk x_k) / L_rr, one
// thread per column, 64 columns per CTA. Shared: 8256 + 128*64 doubles.
__global__ void __launch_bounds__(64) k_trsm_left(const double* __restrict__ L, int ldl, int i0, double* __restrict__ X,
                                                  int ldx, int c0, int ncols) {
  extern __shared__ double sm[];
  double* sL = sm;
  double* sT = sm + NB * (NB + 1) / 2;  // [128][64]
  load_diag_packed(L, ldl, i0, sL);
  const int cb = c0 + blockIdx.x * 64, t = threadIdx.x;
  const bool live = cb + t < c0 + ncols;
  for (int r = 0; r < NB; ++r) sT[r * 64 + t] = live ? X[(size_t)(i0 + r) * ldx + cb + t] : 0.0;
  __syncthreads();
  for (int r = 0; r < NB; ++r) {
    double a0 = sT[r * 64 + t], a1 = 0.0;
    const double* Lr = sL + pk(r, 0);
    int k = 0;
    for (; k + 1 < r; k += 2) {
      a0 = fma(-Lr[k], sT[k * 64 + t], a0);
      a1 = fma(-Lr[k + 1], sT[(k + 1) * 64 + t], a1);
    }
    if (k < r) a0 = fma(-Lr[k], sT[k * 64 + t], a0);
    sT[r * 64 + t] = __ddiv_rn(a0 + a1, Lr[r]);
  }
  if (live)
    for (int r = 0; r < NB; ++r) X[(size_t)(i0 + r) * ldx + cb + t] = sT[r * 64 + t];
}

// a[i0 .. i0+128) = L_ii^-T a[same] (one right-hand side, backward): one CTA of 128 threads.
__global__ void __launch_bounds__(128) k_trsv_diag_T(const double* __restrict__ L, int ldl, int i0, double* __restrict__ a) {
  extern __shared__ double sm[];
  double* sL = sm;  // packed lower
  __shared__ double z[NB];
  __shared__ double ar;
  load_diag_packed(L, ldl, i0, sL);
  const int t = threadIdx.x;
  z[t] = a[i0 + t];
  __syncthreads();
  for (int r = NB - 1; r >= 0; --r) {
    if (t == r) {
      ar = __ddiv_rn(z[r], sL[pk(r, r)]);
      z[r] = ar;
    }
    __syncthreads();
    if (t < r) z[t] = fma(-sL[pk(r, t)], ar, z[t]);
    __syncthreads();
  }
  a[i0 + t] = z[t];
}

// y[r0 + r] -= sum_k A[r0 + r][k0 + k] z[k0 + k], k < 128, r < nrows: one warp per row
__global__ void k_gemv_sub(const double* __restrict__ A, int lda, int r0, int nrows, int k0, const double* z,
                           double* y) {  // z and y may be disjoint ranges of one vector
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= nrows) return;
  const double* row = A + (size_t)(r0 + r) * lda + k0;
  double s = 0.0;
#pragma unroll
  for (int k = lane; k < NB; k += 32) s = fma(row[k], z[k0 + k], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[r0 + r] -= s;
}
// z[c] -= sum_r A[r0 + r][c] a[r0 + r], r < 128, c < ncols (the transposed update of the backward solve)
__global__ void k_gemvT_sub(const double* __restrict__ A, int lda, int r0, int ncols, const double* a, double* z) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  __shared__ double sa[NB];
  if (threadIdx.x < NB) sa[threadIdx.x] = a[r0 + threadIdx.x];
  __syncthreads();
  if (c >= ncols) return;
  double s0 = 0.0, s1 = 0.0;
  for (int r = 0; r < NB; r += 2) {
    s0 = fma(A[(size_t)(r0 + r) * lda + c], sa[r], s0);
    s1 = fma(A[(size_t)(r0 + r + 1) * lda + c], sa[r + 1], s1);
  }
  z[c] -= s0 + s1;
}

// C[M x N] -= A[M x K] op(B): NT: B is [N][K]; NN: B is [K][N]. Row-major,
// 64 x 64 tiles, K steps of 16, 256 threads x (4 x 4). LOWER: tiles entirely
// above the diagonal of the square region are skipped (SYRK); ncut > 0: tile
// columns >= the tile's row0 + ncut are skipped (triangular right-hand sides).
template <bool NN, bool LOWER>
__global__ void __launch_bounds__(256) k_dgemm(double* __restrict__ C, int ldc, const double* __restrict__ A, int lda,
                                               const double* __restrict__ B, int ldb, int M, int N, int K) {
  const int row0 = blockIdx.y * 64, col0 = blockIdx.x * 64;
  if (LOWER && col0 > row0 + 63) return;
  __shared__ double As[16][64 + 4];
  __shared__ double Bs[16][64 + 4];
  const int t = threadIdx.x, ty = t >> 4, tx = t & 15;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k0 = 0; k0 < K; k0 += 16) {
    {  // A tile: 64 rows x 16 k
      const int r = t >> 2, kk = (t & 3) * 4;
      const double* src = A + (size_t)(row0 + r) * lda + k0 + kk;
      const bool ok = row0 + r < M;
#pragma unroll
      for (int u = 0; u < 4; ++u) As[kk + u][r] = (ok && k0 + kk + u < K) ? src[u] : 0.0;
    }
    if (NN) {  // B tile: 16 k x 64 n
      const int kk = t >> 4, n = (t & 15) * 4;
      const double* src = B + (size_t)(k0 + kk) * ldb + col0 + n;
      const bool ok = k0 + kk < K;
#pragma unroll
      for (int u = 0; u < 4; ++u) Bs[kk][n + u] = (ok && col0 + n + u < N) ? src[u] : 0.0;
    } else {   // B tile: 64 n x 16 k
      const int n = t >> 2, kk = (t & 3) * 4;
      const double* src = B + (size_t)(col0 + n) * ldb + k0 + kk;
      const bool ok = col0 + n < N;
#pragma unroll
      for (int u = 0; u < 4; ++u) Bs[kk + u][n] = (ok && k0 + kk + u < K) ? src[u] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = row0 + ty * 4 + i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = col0 + tx * 4 + j;
      if (c < N) C[(size_t)r * ldc + c] -= acc[i][j];
    }
  }
}

// sum_i log L_ii over the first m rows
__global__ void k_logdiag(const double* __restrict__ L, int ld, int m, double* __restrict__ out) {
  __shared__ double sm[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) s += log(L[(size_t)i * ld + i]);
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

// max |X_ij| over the lower triangle (bit pattern of a non-negative double: atomicMax on the integer image)
__global__ void k_maxabs_lower(const double* __restrict__ X, int mp, unsigned long long* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (idx < (int64_t)mp * mp && (idx % mp) <= (idx / mp)) v = fabs(X[idx]);
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(v));
}

// X = identity (mp x mp)
__global__ void k_eye(double* __restrict__ X, int mp) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)mp * mp) return;
  X[idx] = (idx / mp) == (idx % mp) ? 1.0 : 0.0;
}

// double -> (hi, lo) float pairs (the variance kernel's double-float inputs); entries >= n are 0
__global__ void k_split_f2(const double* __restrict__ x, int n, int np, float2* __restrict__ o) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np) return;
  const double v = i < n ? x[i] : 0.0;
  const float h = (float)v;
  o[i] = make_float2(h, (float)(v - (double)h));
}

// mean_t = max(mu + sum_i k(xq_t, x_i) a_i, floor) in binary64, the kernel
// values formed on the fly (predict_alpha, gpr.cpp:153-158,166): one warp per query.
__global__ void k_mean(const double* __restrict__ x, const double* __restrict__ a, int m, const double* __restrict__ xq,
                       int q, double sf2, double ell, double mu, double floor_mean, double* __restrict__ mean) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= q) return;
  const double xt = xq[t];
  double s = 0.0;
  for (int i = lane; i < m; i += 32) {
    const double d = __ddiv_rn(__dsub_rn(xt, x[i]), ell);
    s = fma(__dmul_rn(sf2, exp(__dmul_rn(-0.5, __dmul_rn(d, d)))), a[i], s);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const double mn = mu + s;
    mean[t] = mn < floor_mean ? floor_mean : mn;
  }
}

// binary64 variance path: Ks[k][t] = k(x_k, xq_t) for a block of queries (mp x qb, row-major; rows >= m zero)
__global__ void k_cross(const double* __restrict__ x, int m, int mp, const double* __restrict__ xq, int qb, int ldq,
                        double sf2, double ell, double* __restrict__ Ks) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)mp * qb) return;
  const int k = (int)(idx / qb), t = (int)(idx % qb);
  double v = 0.0;
  if (k < m) {
    const double d = __ddiv_rn(__dsub_rn(xq[t], x[k]), ell);
    v = __dmul_rn(sf2, exp(__dmul_rn(-0.5, __dmul_rn(d, d))));
  }
  Ks[(size_t)k * ldq + t] = v;
}
// var_t = max(sfsn - sum_i V[i][t]^2, 0): thread per query, coalesced over t
__global__ void k_colsumsq(const double* __restrict__ V, int mp, int qb, int ldq, double sfsn, double* __restrict__ var) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= qb) return;
  double s0 = 0.0, s1 = 0.0;
  int i = 0;
  for (; i + 1 < mp; i += 2) {
    const double a = V[(size_t)i * ldq + t], b = V[(size_t)(i + 1) * ldq + t];
    s0 = fma(a, a, s0);
    s1 = fma(b, b, s1);
  }
  if (i < mp) s0 = fma(V[(size_t)i * ldq + t], V[(size_t)i * ldq + t], s0);
  const double v = sfsn - (s0 + s1);
  var[t] = v < 0.0 ? 0.0 : v;
}

}  // namespace gpr_dev
