// gadi_csr.cuh — general sparse operators on the device (BASELINE configs[3]).
//
//  * k_band_gen: the C4 generator (26 distinct off-diagonals uniform in
//    [i-4096, i+4096] \ {i}, values U[-1,1], diagonal 1.1 * sum|off|), bit for
//    bit the oracle's orc_band_csr (counter RNG, same draw order).
//  * the HSS split on the device (splitting.cpp:12-20 with sparse.cpp:104-117
//    transpose and :166-178 pattern-union add, explicit zeros kept): column
//    counts -> scan -> scatter -> per-row sort gives A^T; a per-row merge of
//    A and A^T (plus the diagonal, shift_diagonal sparse.cpp:180-183) gives
//    the union pattern with M = (A+A^T)/2 and N = (A-A^T)/2 in binary64, the
//    same two-term sums the reference's from_triplets forms.
//  * Sell<V>: a sliced-ELL image of a CSR matrix. A slice is 32*R rows
//    (R = rows per lane); its entries are stored k-major: entry k of row
//    (lane*R + v) at slice_base + k*32*R + lane*R + v, so at fold step k a
//    lane reads its R rows' entries as one contiguous vector and a warp reads
//    32*R contiguous entries. Each row still folds its entries in stored
//    column order (kernels.cpp:47-52), so results are bit-identical to CSR.
#pragma once

#include "gadi_kernels.cuh"

namespace gadi {

template <class V>
struct Sell {
  using value_type = V;  // the storage format's values (exact: they are rounded to u_r)
  int64_t N;
  int lgSR;                              // log2(rows per slice)
  const int64_t* __restrict__ soff;      // slice start offsets (entries)
  const uint16_t* __restrict__ len;      // row lengths
  const int32_t* __restrict__ col;       // absolute columns, or null and
  const V* __restrict__ val;
  const int16_t* __restrict__ off;       // column - row (narrow band: 2 bytes per entry)
  const uint8_t* __restrict__ zf = nullptr;  // per-row zflag summary (k_sell_zflags), when built

  __device__ __forceinline__ int zflags(int64_t row) const { return zf[row]; }
  template <int VEC>
  __device__ __forceinline__ void zflags_vec(int64_t e0, int (&f)[VEC]) const {
    uint8_t z[VEC];
    ld_vec<uint8_t, VEC>(zf, e0, z);
#pragma unroll
    for (int v = 0; v < VEC; ++v) f[v] = z[v];
  }

  template <int VEC, class Src, class X, class Acc, class F>
  __device__ __forceinline__ void fold(const Src& x, int64_t e0, Acc (&acc)[VEC], F f, X (&cc)[VEC]) const {
    x.template vec<VEC>(e0, cc);
    const int64_t SR = int64_t(1) << lgSR;
    const int64_t s = e0 >> lgSR;
    const int64_t base = soff[s] + (e0 & (SR - 1));
    const int width = (int)((soff[s + 1] - soff[s]) >> lgSR);
    int ln[VEC];
    uint16_t lv[VEC];
    ld_vec<uint16_t, VEC>(len, e0, lv);
    int lmax = 0;  // this lane's longest row: the padding beyond it is never read
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      ln[v] = lv[v];
      lmax = max(lmax, ln[v]);
    }
    if (lmax > width) lmax = width;
    if (off) {
#pragma unroll 2
      for (int k = 0; k < lmax; ++k) {
        const int64_t pos = base + (int64_t)k * SR;
        int16_t ov[VEC];
        V vv[VEC];
        ld_vec<int16_t, VEC>(off, pos, ov);
        ld_vec<V, VEC>(val, pos, vv);
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          if (k < ln[v]) acc[v] = f(acc[v], ld_c<V, Acc>(vv[v]), x.at(e0 + v + ov[v]));
      }
      return;
    }
    for (int k = 0; k < lmax; ++k) {
      const int64_t pos = base + (int64_t)k * SR;
      int32_t cv[VEC];
      V vv[VEC];
      if constexpr (VEC * 4 % 16 == 0) {
#pragma unroll
        for (int b = 0; b < VEC / 4; ++b) {
          const int4 c4 = __ldg(reinterpret_cast<const int4*>(col + pos) + b);
          cv[4 * b] = c4.x;
          cv[4 * b + 1] = c4.y;
          cv[4 * b + 2] = c4.z;
          cv[4 * b + 3] = c4.w;
        }
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) cv[v] = col[pos + v];
      }
      ld_vec<V, VEC>(val, pos, vv);
#pragma unroll
      for (int v = 0; v < VEC; ++v)
        if (k < ln[v]) acc[v] = f(acc[v], ld_c<V, Acc>(vv[v]), x.at(cv[v]));
    }
  }
};

// Per-row OR of zflag over the stored coefficients of a SELL image.
template <class V>
__global__ void k_sell_zflags(int64_t N, int lgSR, const int64_t* __restrict__ soff, const uint16_t* __restrict__ len,
                              const V* __restrict__ val, uint8_t* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  const int64_t SR = int64_t(1) << lgSR;
  const int64_t base = soff[r >> lgSR] + (r & (SR - 1));
  int f = 0;
  for (int k = 0; k < len[r]; ++k) f |= zflag(val[base + (int64_t)k * SR]);
  out[r] = (uint8_t)f;
}

// ------------------------------------------------------------ generator
#define GADI_VALSALT 0x5851F42D4C957F2Dull
// rows [row0, row0 + rows) of the N x N matrix (global columns), row i - row0
// at (i - row0) * (k_off + 1): a row block generates its own rows (+ the band)
static __global__ void k_band_gen(int64_t N, int k_off, int64_t band, uint64_t seed, int32_t* __restrict__ ci,
                                  double* __restrict__ v, int64_t row0, int64_t rows) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows) return;
  const int64_t i = row0 + t;
  int64_t cols[32];
  int cnt = 0;
  for (uint64_t draw = 0; cnt < k_off && draw < (1u << 20); ++draw) {
    const uint64_t z = splitmix64(seed, ((uint64_t)i << 20) | draw);
    const int64_t off = (int64_t)(z % (uint64_t)(2 * band + 1)) - band;
    const int64_t c = i + off;
    if (off == 0 || c < 0 || c >= N) continue;
    bool dup = false;
    for (int t = 0; t < cnt; ++t) dup |= cols[t] == c;
    if (dup) continue;
    cols[cnt++] = c;
  }
  for (int a = 1; a < cnt; ++a) {  // insertion sort (ascending columns)
    const int64_t key = cols[a];
    int b = a - 1;
    while (b >= 0 && cols[b] > key) {
      cols[b + 1] = cols[b];
      --b;
    }
    cols[b + 1] = key;
  }
  const int64_t base = t * (int64_t)(k_off + 1);
  double sum = 0.0;
  int64_t dpos = -1, w = base;
  int slot = 0;
  for (int t = 0; t <= cnt; ++t) {
    if (dpos < 0 && (t == cnt || cols[t] > i)) {
      dpos = w;
      ci[w++] = (int32_t)i;
    }
    if (t == cnt) break;
    const double val = uniform01(seed ^ GADI_VALSALT, ((uint64_t)i << 8) | (uint64_t)slot, -1.0, 1.0);
    ++slot;
    sum = __dadd_rn(sum, fabs(val));
    ci[w] = (int32_t)cols[t];
    v[w] = val;
    ++w;
  }
  v[dpos] = __dmul_rn(1.1, sum);
}

// rp[i] = i * step (fixed-width rows of the generator)
static __global__ void k_iota_scaled(int64_t* __restrict__ rp, int64_t n, int64_t step) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rp[i] = i * step;
}

static __global__ void k_i32_to_i64(const int* __restrict__ a, int64_t* __restrict__ b, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

// ------------------------------------------------------------ row blocks
// The square window [lo, hi)^2 of a CSR holding rows [lo, hi) with global
// columns (a sharded row block's rows plus the band on each side): per-row
// counts of the columns inside, then the entries with columns shifted by -lo.
static __global__ void k_window_count(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t rows,
                                      int64_t lo, int64_t hi, int64_t* __restrict__ cnt) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  int64_t c = 0;
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) c += (ci[k] >= lo && ci[k] < hi) ? 1 : 0;
  cnt[r] = c;
}
static __global__ void k_window_fill(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                     const double* __restrict__ v, int64_t rows, int64_t lo, int64_t hi,
                                     const int64_t* __restrict__ nrp, int32_t* __restrict__ nci,
                                     double* __restrict__ nv) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  int64_t w = nrp[r];
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k)
    if (ci[k] >= lo && ci[k] < hi) {
      nci[w] = (int32_t)(ci[k] - lo);
      nv[w] = v[k];
      ++w;
    }
}
// out[i] = in[i] - d (row pointers / entry positions of a cropped row range)
static __global__ void k_sub_i64(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n, int64_t d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] - d;
}
// out[k] = in[k] - d (column indices relative to a cropped row range's first row)
static __global__ void k_sub_i32(const int32_t* __restrict__ in, int32_t* __restrict__ out, int64_t n, int32_t d) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = in[k] - d;
}

// ------------------------------------------------------------ transpose
static __global__ void k_count_cols(const int32_t* __restrict__ ci, int64_t nnz, int* __restrict__ cnt) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nnz) atomicAdd(&cnt[ci[k]], 1);
}

static __global__ void k_scatter_t(int64_t N, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ v, unsigned long long* __restrict__ next,
                            int32_t* __restrict__ tci, double* __restrict__ tv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
    const int64_t q = (int64_t)atomicAdd(&next[ci[k]], 1ull);
    tci[q] = (int32_t)i;
    tv[q] = v[k];
  }
}

// sort each row of A^T by (original) row index; keys are unique per row
static __global__ void k_sort_rows(int64_t N, const int64_t* __restrict__ rp, int32_t* __restrict__ c,
                            double* __restrict__ v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int64_t b = rp[i], e = rp[i + 1];
  for (int64_t a = b + 1; a < e; ++a) {
    const int32_t key = c[a];
    const double kv = v[a];
    int64_t t = a - 1;
    while (t >= b && c[t] > key) {
      c[t + 1] = c[t];
      v[t + 1] = v[t];
      --t;
    }
    c[t + 1] = key;
    v[t + 1] = kv;
  }
}

// ------------------------------------------------------------ pattern union
// One row of the union of A, A^T and the diagonal; WRITE = false counts.
template <bool WRITE>
__global__ void k_union(int64_t N, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                        const double* __restrict__ v, const int64_t* __restrict__ trp,
                        const int32_t* __restrict__ tci, const double* __restrict__ tv, int64_t* __restrict__ ulen,
                        const int64_t* __restrict__ urp, int32_t* __restrict__ uci, double* __restrict__ mv,
                        double* __restrict__ nv, int64_t* __restrict__ dpos, uint8_t* __restrict__ din) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int64_t a = rp[i], ae = rp[i + 1], t = trp[i], te = trp[i + 1];
  int64_t w = WRITE ? urp[i] : 0, cnt = 0;
  bool diag_done = false;
  while (a < ae || t < te || !diag_done) {
    const int64_t ca = a < ae ? ci[a] : INT64_MAX, ct = t < te ? tci[t] : INT64_MAX;
    int64_t c = ca < ct ? ca : ct;
    if (!diag_done && i <= c) c = i;
    const bool hA = ca == c, hT = ct == c;
    if (WRITE) {
      double m = 0.0, nn = 0.0;
      if (hA && hT) {  // add(0.5,A,±0.5,A^T): two triplets summed (sparse.cpp:36-58)
        m = __dadd_rn(__dmul_rn(0.5, v[a]), __dmul_rn(0.5, tv[t]));
        nn = __dadd_rn(__dmul_rn(0.5, v[a]), __dmul_rn(-0.5, tv[t]));
      } else if (hA) {
        m = __dmul_rn(0.5, v[a]);
        nn = m;
      } else if (hT) {
        m = __dmul_rn(0.5, tv[t]);
        nn = __dmul_rn(-0.5, tv[t]);
      }
      if (c == i) {
        dpos[i] = w;
        din[i] = (hA || hT) ? 1 : 0;
      }
      uci[w] = (int32_t)c;
      mv[w] = m;
      nv[w] = nn;
      ++w;
    }
    if (c == i) diag_done = true;
    ++cnt;
    if (hA) ++a;
    if (hT) ++t;
  }
  if (!WRITE) ulen[i] = cnt;
}

// ------------------------------------------------------------ SELL image
// width of each slice (max row length) and the row lengths
static __global__ void k_sell_width(int64_t N, int lgSR, const int64_t* __restrict__ rp, int64_t* __restrict__ wid,
                             uint16_t* __restrict__ len) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t SR = int64_t(1) << lgSR;
  if (s * SR >= N) return;
  int64_t m = 0;
  for (int64_t r = s * SR; r < (s + 1) * SR && r < N; ++r) {
    const int64_t l = rp[r + 1] - rp[r];
    len[r] = (uint16_t)l;
    m = l > m ? l : m;
  }
  wid[s] = m * SR;
}

// entries of CSR values (or just the pattern when val == nullptr) into the
// SELL image; vout receives round_{u_r}(val) (+ alpha on the diagonal when
// dpos is given: shift_diagonal, sparse.cpp:180-183; splitting.cpp:37-47).
template <class VO, int PR>
__global__ void k_sell_fill(int64_t N, int lgSR, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ val, const int64_t* __restrict__ soff,
                            int32_t* __restrict__ cout, int16_t* __restrict__ oout, VO* __restrict__ vout,
                            const int64_t* __restrict__ dpos, const uint8_t* __restrict__ din, double alpha) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  const int64_t SR = int64_t(1) << lgSR;
  const int64_t base = soff[r >> lgSR] + (r & (SR - 1));
  const int64_t b = rp[r], e = rp[r + 1];
  for (int64_t k = b; k < e; ++k) {
    const int64_t pos = base + (k - b) * SR;
    if (cout) cout[pos] = ci[k];
    if (oout) oout[pos] = (int16_t)(ci[k] - r);
    if (vout) {
      double x = val[k];
      if (dpos && k == dpos[r]) x = din[r] ? __dadd_rn(__dmul_rn(1.0, x), alpha) : alpha;
      vout[pos] = from_dbl<VO>(round_p<PR>(x));
    }
  }
}

}  // namespace gadi
