// gadi_gpr_dense.cuh — the binary64 dense kernels of the GPR fit (gpr.cpp:84-105:
// Gram matrix, LLT, K^-1 y, log det) and of the binary64 prediction path,
// hand-written for sm_100a (no cuSOLVER / cuBLAS).
//
// Blocked right-looking Cholesky on a row-major mp x mp matrix (mp a multiple
// of 128, the lower triangle is referenced): per 128-column block
//   k_potinv128     the diagonal block L_jj and its inverse D_j, one CTA
//   k_dgemm<NT,SET> the panel below it: L21 = W21 D_j^T
//   k_dgemm<NT>     the trailing update W22 -= L21 L21^T (lower tiles only)
// The explicit inverse factor X = L^-1 the tensor-core variance GEMM consumes
// (gadi_gpr_umma.cuh) is a right-looking block substitution on the identity:
//   k_dgemm<NN,SET> X_i,: = D_i R_i,:          k_dgemm<NN>   R_r,: -= L_r,i X_i,:
// and K^-1 y the same substitution on one vector (k_diag_apply, k_gemv[T]_sub).
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

// 64-bit warp shuffle
__device__ __forceinline__ double shfl_d(double v, int src) {
  int lo = __double2loint(v), hi = __double2hiint(v);
  lo = __shfl_sync(0xffffffffu, lo, src);
  hi = __shfl_sync(0xffffffffu, hi, src);
  return __hiloint2double(hi, lo);
}

// Cholesky of the 128 x 128 diagonal block at (j0, j0), in place (lower), and
// its inverse D = L_jj^-1 (128 x 128 row-major, zeros above the diagonal): the
// panel below the block, the inverse factor and the triangular solves then
// all run as GEMMs / GEMVs against D instead of substitutions.
// info: 0, or 1 + the first column whose pivot is not positive (Eigen's
// NumericalIssue, gpr.cpp:92). One CTA of 256 threads, shared: 128 x 129
// doubles. Blocked by 32:
//   factor   per 32-column block: the 32 x 32 diagonal block in one warp's
//            registers (column broadcasts by shuffle, 1/sqrt by rsqrt: no
//            division on the pivot chain), the rows below it one thread per
//            row, the trailing update of the block on 16 x 16 threads;
//   invert   in place, last 32-block first: X_kk in one warp's registers,
//            X_ik = -(sum_j X_ij L_jk) X_kk on all threads.
__global__ void __launch_bounds__(256) k_potinv128(double* __restrict__ W, int ld, int j0, double* __restrict__ D,
                                                   int* __restrict__ info) {
  extern __shared__ double sA[];  // [128][129]; the strict upper triangle stays zero
  __shared__ double sinv[NB];     // 1 / L_cc
  __shared__ double scol[32];
  __shared__ int bad;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) bad = 0;
  for (int e = t; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    sA[r * 129 + c] = c <= r ? W[(size_t)(j0 + r) * ld + j0 + c] : 0.0;
  }
  __syncthreads();
  // ------------------------------------------------------------- factor
  for (int c0 = 0; c0 < NB; c0 += 32) {
    if (warp == 0) {  // diagonal 32 x 32 block: lane = row, the row in registers
      double a[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) a[c] = sA[(c0 + lane) * 129 + c0 + c];
      int isbad = 0;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        scol[lane] = a[c];  // column c of the block, unscaled: broadcast through shared memory
        __syncwarp();
        const double piv = scol[c];
        if (!(piv > 0.0) && !isbad) isbad = c0 + c + 1;
        const double rs = rsqrt(piv);
        const double l = lane == c ? piv * rs : a[c] * rs;
        a[c] = l;
        if (lane == c) sinv[c0 + c] = rs;
#pragma unroll
        for (int cc = c + 1; cc < 32; ++cc) {
          // l_cc,c = raw * rs, the value lane cc stores as its own a[c]; rows above cc are not updated
          const double lcc = lane >= cc ? scol[cc] * rs : 0.0;
          a[cc] = fma(-l, lcc, a[cc]);
        }
        __syncwarp();
      }
      if (isbad && lane == 0) bad = isbad;
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c <= lane) sA[(c0 + lane) * 129 + c0 + c] = a[c];
    }
    __syncthreads();
    if (bad) break;
    const int below = NB - c0 - 32;  // rows under the diagonal block
    if (t < below) {                 // l_r,: = a_r,: L_kk^-T, one thread per row
      double x[32];
      const int r = c0 + 32 + t;
#pragma unroll
      for (int c = 0; c < 32; ++c) x[c] = sA[r * 129 + c0 + c];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        double acc = x[c];
#pragma unroll
        for (int k = 0; k < c; ++k) acc = fma(-x[k], sA[(c0 + c) * 129 + c0 + k], acc);
        x[c] = acc * sinv[c0 + c];
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) sA[r * 129 + c0 + c] = x[c];
    }
    __syncthreads();
    if (below > 0) {  // trailing update of the block: a_r,cc -= sum_k l_r,k l_cc,k
      const int ty = t >> 4, tx = t & 15, b0 = c0 + 32;
      double acc[6][6];
#pragma unroll
      for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) acc[i][j] = 0.0;
      for (int k = 0; k < 32; ++k) {
        double rv[6], cv[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const int r = b0 + ty + 16 * i, c = b0 + tx + 16 * i;
          rv[i] = r < NB ? sA[r * 129 + c0 + k] : 0.0;
          cv[i] = c < NB ? sA[c * 129 + c0 + k] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
          for (int j = 0; j < 6; ++j) acc[i][j] = fma(rv[i], cv[j], acc[i][j]);
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const int r = b0 + ty + 16 * i, c = b0 + tx + 16 * j;
          if (r < NB && c <= r) sA[r * 129 + c] -= acc[i][j];
        }
    }
    __syncthreads();
  }
  if (bad) {
    if (t == 0) atomicCAS(info, 0, j0 + bad);
    return;
  }
  for (int e = t; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    if (c <= r) W[(size_t)(j0 + r) * ld + j0 + c] = sA[r * 129 + c];
  }
  __syncthreads();
  // ------------------------------------------------------------- invert
  for (int c0 = NB - 32; c0 >= 0; c0 -= 32) {
    if (warp == 0) {  // X_kk = L_kk^-1: lane = column
      double x[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        double acc = i == lane ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < i; ++k) acc = fma(-sA[(c0 + i) * 129 + c0 + k], x[k], acc);
        x[i] = i < lane ? 0.0 : acc * sinv[c0 + i];
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i >= lane) sA[(c0 + i) * 129 + c0 + lane] = x[i];
    }
    __syncthreads();
    const int b0 = c0 + 32, below = NB - b0;
    if (below > 0) {
      const int c = t & 31, g = t >> 5;  // column of the block, row group
      double acc[12];
      // T = X22 L21: rows b0 + g + 8 u, inner index j over the inverted trailing block (upper part is zero)
#pragma unroll
      for (int u = 0; u < 12; ++u) acc[u] = 0.0;
      for (int j = b0; j < NB; ++j) {
        const double lj = sA[j * 129 + c0 + c];
#pragma unroll
        for (int u = 0; u < 12; ++u) {
          const int i = b0 + g + 8 * u;
          if (i < NB) acc[u] = fma(sA[i * 129 + j], lj, acc[u]);
        }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 12; ++u) {
        const int i = b0 + g + 8 * u;
        if (i < NB) sA[i * 129 + c0 + c] = acc[u];
      }
      __syncthreads();
      // X21 = -T X_kk (X_kk lower: its upper part is zero)
#pragma unroll
      for (int u = 0; u < 12; ++u) acc[u] = 0.0;
      for (int k = 0; k < 32; ++k) {
        const double xk = sA[(c0 + k) * 129 + c0 + c];
#pragma unroll
        for (int u = 0; u < 12; ++u) {
          const int i = b0 + g + 8 * u;
          if (i < NB) acc[u] = fma(sA[i * 129 + c0 + k], xk, acc[u]);
        }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 12; ++u) {
        const int i = b0 + g + 8 * u;
        if (i < NB) sA[i * 129 + c0 + c] = -acc[u];
      }
    }
    __syncthreads();
  }
  for (int e = t; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    D[e] = c <= r ? sA[r * 129 + c] : 0.0;
  }
}

// v[0..128) = D v (TRANS = false) or D^T v (TRANS = true), D a 128 x 128
// lower-triangular block: one CTA of 128 threads.
template <bool TRANS>
__global__ void __launch_bounds__(128) k_diag_apply(const double* __restrict__ D, double* __restrict__ v) {
  __shared__ double sv[NB];
  const int t = threadIdx.x;
  sv[t] = v[t];
  __syncthreads();
  double s = 0.0;
  if (TRANS) {
    for (int k = t; k < NB; ++k) s = fma(D[k * NB + t], sv[k], s);  // coalesced over t
    v[t] = s;
  } else {
    const int warp = t >> 5, lane = t & 31;
    for (int r = warp; r < NB; r += 4) {  // a warp per row, lanes over k
      double a = 0.0;
      for (int k = lane; k <= r; k += 32) a = fma(D[r * NB + k], sv[k], a);
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) v[r] = a;
    }
  }
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

// C[M x N] -= A[M x K] op(B) (SET: C = A op(B)): NT: B is [N][K]; NN: B is [K][N]. Row-major,
// 64 x 64 tiles, K steps of 16, 256 threads x (4 x 4). LOWER: tiles entirely
// above the diagonal of the square region are skipped (SYRK); ncut > 0: tile
// columns >= the tile's row0 + ncut are skipped (triangular right-hand sides).
template <bool NN, bool LOWER, bool SET = false>
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
      if (c < N) {
        if (SET) C[(size_t)r * ldc + c] = acc[i][j];
        else C[(size_t)r * ldc + c] -= acc[i][j];
      }
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
