// gadi_gpr_umma.cuh — the GPR predictive variances on the 5th-generation
// tensor cores (tcgen05.mma, accumulators in TMEM), sm_100a only.
//
// predict_alpha (gpr.cpp:151-169) needs, per query x_q,
//     var_q = sf2 + sn2 - || L^-1 k_q ||^2,   k_q[i] = sf2 exp(-(x_q - x_i)^2 / (2 l^2)),
// m^2 flops per query: 1.1e12 for BASELINE configs[4] (m = 4096, q = 65,536),
// the one dense contraction of the solver. Here it is ONE GEMM against the
// explicit inverse factor: with X = sf2 L^-1 (binary64, gadi_gpr.cu) and
// k'_q = k_q / sf2 = exp(.) in (0, 1],
//     || L^-1 k_q ||^2 = || X k'_q ||^2,
// D = X K'_* (m x q) is accumulated in TMEM and never stored: the epilogue
// squares it and reduces over the rows.
//
// Precision: fp16 tensor-core inputs carry 11 bits, too few for a difference
// sf2 + sn2 - ||.||^2 that cancels; every operand is therefore split
// v = hi + lo (two fp16, ~22 bits) and each product takes three MMAs
// (hi*hi + hi*lo + lo*hi) into the same fp32 accumulator -- "FP16 panels, FP32
// accumulate". A (= 2^ea X, ea chosen so max|A| is in [256, 512): the lo halves
// stay clear of the fp16 subnormals) is split once by k_pack_linv into the exact
// shared-memory image of its tiles, so a stage's A operands are one 1-D bulk
// copy (cp.async.bulk + mbarrier complete_tx); B (= 2^8 K'_*) is generated on
// the fly by the producer warps (double-float difference, ex2.approx) and
// written straight into the swizzled operand layout.
//
// Tiling: one CTA owns 256 queries (UMMA N = 256) and walks the row blocks of
// X in passes of 256 rows = two 128 x 256 fp32 accumulators = all 512 TMEM
// columns. X is lower triangular: pass p only needs k < 256 (p + 1). K blocks
// of 32 (64-byte rows, SWIZZLE_64B), 3-stage ring:
//   warps 0-3   epilogue: tcgen05.ld, square, 32x32 transpose-reduce, per-query sums
//   warp  4     MMA issuer (one lane): 12 tcgen05.mma per stage, tcgen05.commit
//   warp  5     bulk-copy issuer for the A tiles
//   warps 6-13  B generators: thread = query row, 32 kernel values per stage
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace gpr_dev {

constexpr int UM_BM = 128;     // rows of X per accumulator (UMMA M)
constexpr int UM_NQ = 256;     // queries per CTA (UMMA N)
constexpr int UM_BK = 32;      // k per stage (64-byte operand rows)
constexpr int UM_STAGES = 3;
constexpr int UM_PASS_ROWS = 2 * UM_BM;
constexpr int UM_A_TILE = UM_BM * UM_BK * 2;        // 8 KB: one 128 x 32 fp16 tile
constexpr int UM_A_STAGE = 4 * UM_A_TILE;           // [tile 0/1][hi/lo]
constexpr int UM_B_TILE = UM_NQ * UM_BK * 2;        // 16 KB
constexpr int UM_STAGE_BYTES = UM_A_STAGE + 2 * UM_B_TILE;  // 64 KB
constexpr int UM_THREADS = 14 * 32;
constexpr int UM_GEN_WARPS = 8;
constexpr float UM_SCALE_B_LOG2 = 8.0f;             // 2^8
constexpr int UM_SMEM = UM_STAGES * UM_STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + 4 * UM_NQ * 8;

__device__ __forceinline__ uint32_t um_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void um_bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(um_smem(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void um_bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(um_smem(b)) : "memory");
}
__device__ __forceinline__ void um_bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(um_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void um_bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(um_smem(b)), "r"(parity)
                 : "memory");
  } while (!ok);
}
__device__ __forceinline__ void um_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   um_smem(dst)),
               "l"(src), "r"(bytes), "r"(um_smem(bar))
               : "memory");
}

// K-major operand tile with 64-byte rows, SWIZZLE_64B: byte offset of 16-byte
// chunk c (0..3) of row r; 8-row groups are 512 bytes apart (the descriptor's
// stride byte offset), the chunk index is XORed with bits 7-8 of the address.
__host__ __device__ __forceinline__ uint32_t um_sw64(uint32_t r, uint32_t c) {
  return r * 64u + ((c ^ ((r >> 1) & 3u)) << 4);
}

// Shared-memory matrix descriptor (PTX ISA "tcgen05 shared memory descriptor"):
// start address >> 4 [0,14), leading byte offset >> 4 [16,30) (unused for a
// swizzled K-major tile whose K extent is one swizzle row), stride byte offset
// >> 4 [32,46) = 512 B between 8-row groups, version 1 [46,48), layout type
// [61,64) = 4 (SWIZZLE_64B).
__device__ __forceinline__ uint64_t um_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(512u >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
// Instruction descriptor, kind::f16: D = fp32 [4,6) = 1, A = B = fp16 (0),
// both K-major, N >> 3 at [17,23), M >> 4 at [24,29).
__host__ __device__ constexpr uint32_t um_idesc() { return (1u << 4) | ((uint32_t)(UM_NQ >> 3) << 17) | ((uint32_t)(UM_BM >> 4) << 24); }

__device__ __forceinline__ void um_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void um_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(um_smem(bar))
               : "memory");
}
__device__ __forceinline__ void um_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void um_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void um_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// X (binary64, row-major mp x mp, lower triangular) -> the operand image:
// for pass p, k-block kb < 8 (p + 1): [tile 0 hi][tile 0 lo][tile 1 hi][tile 1 lo],
// each tile the SWIZZLE_64B image of scale * X[256 p + 128 t + r][32 kb + c].
// Stage s of pass p lives at offset (8 * p (p + 1) / 2 + kb) * UM_A_STAGE.
__global__ void k_pack_linv(const double* __restrict__ X, int mp, int ld, double scale, uint8_t* __restrict__ img) {
  const int p = blockIdx.y, kb = blockIdx.x;
  if (kb >= 8 * (p + 1)) return;
  uint8_t* dst = img + ((size_t)(4 * p * (p + 1) + kb)) * UM_A_STAGE;
  for (int e = threadIdx.x; e < 2 * UM_BM * 4; e += blockDim.x) {  // (tile, row, 16-byte chunk)
    const int t = e / (UM_BM * 4), r = (e / 4) % UM_BM, c = e % 4;
    const int row = UM_PASS_ROWS * p + UM_BM * t + r, col = UM_BK * kb + 8 * c;
    __align__(16) __half hi[8], lo[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double v = (col + j <= row) ? X[(size_t)row * ld + col + j] * scale : 0.0;
      const float f = (float)v;
      hi[j] = __float2half_rn(f);
      lo[j] = __float2half_rn((float)(v - (double)__half2float(hi[j])));
    }
    uint8_t* tb = dst + (size_t)t * 2 * UM_A_TILE;
    *reinterpret_cast<uint4*>(tb + um_sw64(r, c)) = *reinterpret_cast<const uint4*>(hi);
    *reinterpret_cast<uint4*>(tb + UM_A_TILE + um_sw64(r, c)) = *reinterpret_cast<const uint4*>(lo);
  }
}

struct VarParams {
  const uint8_t* img;   // k_pack_linv image
  const float2* xs;     // training inputs as double-float (hi, lo), mp entries (padding arbitrary)
  const float2* xq;     // query inputs as double-float, q entries
  int mp, m, q;
  float inv_ell;
  double mult, sfsn;    // var = max(sfsn - mult * sum, 0), mult = the operand scalings squared, inverted
  double* var_out;      // q
};

__global__ void __launch_bounds__(UM_THREADS, 1) k_var_umma(VarParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + UM_STAGES * UM_STAGE_BYTES);
  uint64_t* full = bars;                  // [STAGES] A bytes landed + B generated
  uint64_t* empty = bars + UM_STAGES;     // [STAGES] MMAs that read the stage have completed
  uint64_t* acc_full = bars + 2 * UM_STAGES;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  double* colsum = reinterpret_cast<double*>(smem + UM_STAGES * UM_STAGE_BYTES + 256);  // [4][NQ]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npass = P.mp / UM_PASS_ROWS;
  const int q0 = blockIdx.x * UM_NQ;

  if (threadIdx.x == 0) {
    for (int s = 0; s < UM_STAGES; ++s) {
      um_bar_init(&full[s], 1 + UM_GEN_WARPS);
      um_bar_init(&empty[s], 1);
    }
    um_bar_init(acc_full, 1);
    um_bar_init(acc_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {  // the MMA warp owns the TMEM allocation: all 512 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(um_smem(tmem_slot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  um_fence_before();
  __syncthreads();
  um_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ------------------------------------------------------------ epilogue
    double sums[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) sums[c] = 0.0;
    for (int p = 0; p < npass; ++p) {
      um_bar_wait(acc_full, p & 1);
      um_fence_after();
#pragma unroll 1
      for (int a = 0; a < 2; ++a) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float v[32];
          um_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(a * UM_NQ + 32 * c), v);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] *= v[i];
          // transpose-reduce: lane l ends with the sum over the warp's 32 rows of column 32 c + l
#pragma unroll
          for (int off = 16, n = 32; off >= 1; off >>= 1, n >>= 1) {
            const bool up = (lane & off) != 0;
#pragma unroll
            for (int j = 0; j < n / 2; ++j) {
              const float send = up ? v[j] : v[j + n / 2];
              const float keep = up ? v[j + n / 2] : v[j];
              v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
          }
          sums[c] += (double)v[0];
        }
      }
      um_fence_before();
      __syncwarp();
      if (lane == 0) um_bar_arrive(acc_empty);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) colsum[warp * UM_NQ + 32 * c + lane] = sums[c];
    asm volatile("bar.sync 1, 128;" ::: "memory");
    for (int j = threadIdx.x; j < UM_NQ; j += 128) {
      const double s = colsum[j] + colsum[UM_NQ + j] + colsum[2 * UM_NQ + j] + colsum[3 * UM_NQ + j];
      if (q0 + j < P.q) {
        const double v = P.sfsn - P.mult * s;
        P.var_out[q0 + j] = v < 0.0 ? 0.0 : v;
      }
    }
  } else if (warp == 4) {
    // ---------------------------------------------------------- MMA issuer
    const uint32_t idesc = um_idesc();
    uint32_t it = 0;
    for (int p = 0; p < npass; ++p) {
      if (p > 0) {
        um_bar_wait(acc_empty, (p - 1) & 1);  // the epilogue has drained both accumulators
        um_fence_after();
      }
      const int nkb = 8 * (p + 1);
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % UM_STAGES;
        um_bar_wait(&full[s], (it / UM_STAGES) & 1);
        um_fence_after();
        if (lane == 0) {
          const uint32_t sa = um_smem(smem + (size_t)s * UM_STAGE_BYTES);
          const uint32_t sb = sa + UM_A_STAGE;
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            const uint32_t ah = sa + a * 2 * UM_A_TILE, al = ah + UM_A_TILE;
            const uint32_t bh = sb, bl = sb + UM_B_TILE;
            const uint32_t d = tmem + (uint32_t)(a * UM_NQ);
#pragma unroll
            for (int ks = 0; ks < UM_BK / 16; ++ks) {  // K = 16 per MMA: 32 bytes along the swizzled row
              const uint32_t o = ks * 32;
              um_mma(d, um_desc(ah + o), um_desc(bh + o), idesc, (kb | ks) != 0);
              um_mma(d, um_desc(ah + o), um_desc(bl + o), idesc, 1);
              um_mma(d, um_desc(al + o), um_desc(bh + o), idesc, 1);
            }
          }
          um_commit(&empty[s]);                      // frees the stage when these MMAs retire
          if (kb == nkb - 1) um_commit(acc_full);    // ... and hands the accumulators to the epilogue
        }
        __syncwarp();
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------ A tiles: 1-D bulk copies
    if (lane == 0) {
      uint32_t it = 0;
      for (int p = 0; p < npass; ++p) {
        const uint8_t* src = P.img + (size_t)(4 * p * (p + 1)) * UM_A_STAGE;
        for (int kb = 0; kb < 8 * (p + 1); ++kb, ++it) {
          const int s = it % UM_STAGES;
          if (it >= UM_STAGES) um_bar_wait(&empty[s], ((it / UM_STAGES) - 1) & 1);
          um_bar_expect(&full[s], UM_A_STAGE);
          um_bulk_g2s(smem + (size_t)s * UM_STAGE_BYTES, src + (size_t)kb * UM_A_STAGE, UM_A_STAGE, &full[s]);
        }
      }
    }
  } else {
    // ------------------------------------- B tiles: K'_* generated on the fly
    const int row = (warp - 6) * 32 + lane;  // query row of the tile
    const int qi = q0 + row;
    const float2 xq = qi < P.q ? P.xq[qi] : make_float2(0.f, 0.f);
    const bool live = qi < P.q;
    const float cexp = -0.72134752044448170368f;  // -0.5 log2(e)
    uint32_t it = 0;
    for (int p = 0; p < npass; ++p) {
      for (int kb = 0; kb < 8 * (p + 1); ++kb, ++it) {
        const int s = it % UM_STAGES;
        if (it >= UM_STAGES) um_bar_wait(&empty[s], ((it / UM_STAGES) - 1) & 1);
        uint8_t* bh = smem + (size_t)s * UM_STAGE_BYTES + UM_A_STAGE;
        uint8_t* bl = bh + UM_B_TILE;
        const int k0 = UM_BK * kb;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          __align__(16) __half2 hi[4], lo[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 xx = __ldg(reinterpret_cast<const float4*>(P.xs + k0 + 8 * c + 2 * j));  // two (hi, lo) pairs
            const float d0 = ((xq.x - xx.x) + (xq.y - xx.y)) * P.inv_ell;
            const float d1 = ((xq.x - xx.z) + (xq.y - xx.w)) * P.inv_ell;
            float v0 = exp2f(fmaf(cexp * d0, d0, UM_SCALE_B_LOG2));
            float v1 = exp2f(fmaf(cexp * d1, d1, UM_SCALE_B_LOG2));
            if (!live || k0 + 8 * c + 2 * j >= P.m) v0 = 0.f;
            if (!live || k0 + 8 * c + 2 * j + 1 >= P.m) v1 = 0.f;
            hi[j] = __floats2half2_rn(v0, v1);
            const float2 hf = __half22float2(hi[j]);
            lo[j] = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
          }
          *reinterpret_cast<uint4*>(bh + um_sw64(row, c)) = *reinterpret_cast<const uint4*>(hi);
          *reinterpret_cast<uint4*>(bl + um_sw64(row, c)) = *reinterpret_cast<const uint4*>(lo);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> visible to the MMA (async proxy)
        __syncwarp();
        if (lane == 0) um_bar_arrive(&full[s]);
      }
    }
  }

  um_fence_before();
  __syncthreads();
  if (warp == 4) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

}  // namespace gpr_dev
