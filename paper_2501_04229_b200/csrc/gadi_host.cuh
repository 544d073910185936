// gadi_host.cuh — host-side engine of the B200 GADI-IR solver (shared by the
// per-format translation units gadi_engine_*.cu and the C ABI in gadi_api.cu).
//
// run_gadi_ir (solver.cpp:57-179) is restated over device-resident vectors:
// x, b, s in binary64, the inner vectors in u_r storage. Per outer step the
// host issues CG on H, the p-scaling, GMRES on S, the update and the new
// residual. Inside CG the host only keeps the launch queue a few iterations
// ahead of the device (the recurrences and stop tests run on the device,
// gadi_kernels.cuh); GMRES reads one small Hessenberg column per Arnoldi step
// (the Givens rotations run on the host in the inner format's rounding).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cub/device/device_scan.cuh>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/gadi_cuda.h"
#include "gadi_kernels.cuh"
#include "gadi_st25.cuh"
#include "gadi_resid64.cuh"
#include "gadi_dist.cuh"
#include "gadi_csr.cuh"

using namespace gadi;

namespace gadi_host {

inline thread_local std::string g_last_error;
void set_last_error(const std::string& m);  // gadi_api.cu

struct Err : std::runtime_error {
  int code;
  Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(x)                                                                                     \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess)                                                                        \
      throw Err(e_ == cudaErrorMemoryAllocation ? GADI_E_OOM : GADI_E_CUDA,                       \
                std::string(#x) + ": " + cudaGetErrorString(e_));                                 \
  } while (0)

#define CKL() CK(cudaGetLastError())

// ---------------------------------------------------------------- host rounding
// round_to (precision.hpp:54-87): one RNE rounding of a binary64 to binary16 /
// binary32, used for the Givens/back-solve scalars that run on the host.
inline double hround(double x, int p) {
  if (p == GADI_SINGLE) return (double)(float)x;
  if (p != GADI_HALF) return x;
  if (std::isnan(x) || std::isinf(x) || x == 0.0) return x;
  const double ax = std::fabs(x);
  if (ax >= 65520.0) return std::copysign(INFINITY, x);
  const int e = std::ilogb(ax);
  const int q = e < -14 ? -24 : e - 10;
  return std::copysign(std::ldexp(std::nearbyint(std::ldexp(ax, -q)), q), x);
}

inline double unit_roundoff(int p) {
  return p == GADI_HALF ? std::ldexp(1.0, -11) : p == GADI_SINGLE ? std::ldexp(1.0, -24) : std::ldexp(1.0, -53);
}

inline bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
inline int ilog2(int64_t v) {
  int d = 0;
  while ((int64_t(1) << (d + 1)) <= v) ++d;
  return d;
}
inline int lg_of(int64_t n) { return is_pow2(n) ? ilog2(n) : -1; }

// 2^D segments -> lanes x warps x segments-per-lane x blocks (gadi_kernels.cuh).
// Up to RMAX segments per lane while that still leaves >= 4 blocks per SM.
inline Geo make_geo(int64_t N, int vec) {
  Geo g;
  g.N = N;
  int64_t nseg;
  if (vec > 1) {
    nseg = N / vec;
    g.D = ilog2(nseg);
  } else {
    g.D = N < 4 ? 0 : ilog2(N) - 1;
    nseg = int64_t(1) << g.D;
  }
  g.L = (int)std::min<int64_t>(32, nseg);
  g.W = (int)std::min<int64_t>(8, nseg / g.L);
  g.R = RMAX;
  if (const char* e = std::getenv("GADI_GEO_R"))  // tuning knob: segments per lane (<= RMAX)
    g.R = std::max(1, std::min(RMAX, std::atoi(e)));
  while (g.R > 1 && nseg / ((int64_t)g.L * g.W * g.R) < 592) g.R /= 2;
  g.nblk = (int)(nseg / ((int64_t)g.L * g.W * g.R));
  return g;
}


// Operand window of a banded sparse operator staged in shared memory
// (gadi_kernels.cuh stage_window): the band passed to the kernel (0 = read the
// operand from global memory) and the dynamic shared memory it needs. Used
// when the window is small and not dominated by the halo (band <= 2 block rows).
struct Window {
  int64_t band = 0;
  size_t bytes = 0;
};
inline Window window_for(const Geo& g, int vec, size_t tsize, int64_t max_band, bool aligned) {
  Window w;
  static const bool disabled = std::getenv("GADI_NO_WINDOW") != nullptr;  // A/B measurement knob
  if (disabled || !aligned || vec <= 1 || max_band == INT64_MAX) return w;
  const int64_t br = (int64_t)g.W * g.R * g.L * vec;
  const int64_t band = std::max<int64_t>(max_band, 1);
  const size_t bytes = (size_t)(br + 2 * band + vec) * tsize;
  // > 64 KB costs more occupancy than the gathers gain (measured: the binary64
  // residual on A with a 96 KB window ran 1.65 ms vs 1.28 ms reading x from L1/L2)
  if (band > 2 * br || bytes > 64 * 1024) return w;
  w.band = band;
  w.bytes = bytes;
  return w;
}
// The dynamic shared-memory cap is one value per kernel for the whole
// process, while handles of different shapes launch concurrently from
// several host threads (gadi_train.cu): the cap only ever grows, under a lock,
// so no launch can find it lowered below its own request.
inline std::mutex& smem_attr_mu() {
  static std::mutex m;
  return m;
}
inline std::map<std::pair<int, const void*>, size_t>& smem_attr_set() {
  static std::map<std::pair<int, const void*>, size_t> s;
  return s;
}
template <class K>
inline void smem_attr(K kern, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  int dev = 0;
  CK(cudaGetDevice(&dev));  // the attribute is per device
  std::lock_guard<std::mutex> g(smem_attr_mu());
  size_t& cur = smem_attr_set()[{dev, (const void*)kern}];
  if (bytes <= cur) return;
  CK(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  cur = bytes;
}

inline bool aligned_for(int64_t N, int64_t n, bool stencil, int vec) {
  return (N % vec == 0) && is_pow2(N / vec) && (!stencil || n % vec == 0);
}

// Geometry of the 2.5D plane-marching stencil kernels (gadi_st25.cuh) for a
// grid of n^3 points stored as `tsize`-byte values with `nin` staged inputs.
// ok = false when the shape does not fit (then the generic kernels run).
inline bool make_st25(int64_t n, int tsize, int nin, St25Geo& g, int64_t target_chunks = 512,
                      bool ident = false, int ring_tsize = 0, int64_t i0 = 0, int64_t i1 = -1,
                      int ring_planes = 4, int64_t max_threads_in = 256) {
  if (i1 < 0) i1 = n;
  const int64_t nloc = i1 - i0;
  if (nloc < 1 || !is_pow2(nloc)) return false;
  g.i0 = (int)i0;
  g.i1 = (int)i1;
  if (ring_tsize == 0) ring_tsize = tsize;
  if (const char* e = std::getenv("GADI_ST25_CHUNKS")) target_chunks = std::max(32, std::atoi(e));  // tuning knob
  const int vec = 16 / tsize;
  if (!is_pow2(n) || n % vec != 0 || n < 8) return false;
  const int64_t TR = n / vec;
  if (TR > 1024) return false;
  g.n = (int)n;
  g.lg = ilog2(n);
  g.nn = n * n;
  g.TR = (int)TR;
  g.lgTR = ilog2(TR);
  int64_t TJ = std::max<int64_t>(1, target_chunks / TR);
  TJ = std::min<int64_t>(TJ, n);
  const int64_t chunks = TJ * TR;
  int64_t max_threads = max_threads_in;
  if (const char* e = std::getenv("GADI_ST25_THREADS")) max_threads = std::atoi(e);  // tuning knob
  g.threads = (int)std::min<int64_t>(std::min<int64_t>(max_threads, 32 * ST25_MAXW), chunks);
  g.CPT = (int)(chunks / g.threads);
  if (g.CPT > ST25_CPT_MAX || g.threads < 32) return false;
  g.TJ = (int)TJ;
  g.lgTJ = ilog2(TJ);
  g.njt = (int)(n / TJ);
  int64_t IL = 32;
  while (IL > 4 && g.njt * (nloc / IL) < 2048) IL /= 2;
  IL = std::min<int64_t>(IL, nloc);
  g.IL = (int)IL;
  g.nblk = (int)(g.njt * (nloc / IL));
  // operand-ring kernels: raw stages + a 4-plane operand ring; identity-
  // operand kernels fold from the stages directly and need 4 of them
  g.stages = 4;
  const int64_t pe = (TJ + 2) * n;
  auto bytes = [&]() {
    return 128 + (size_t)g.stages * nin * pe * tsize + (ident ? 0 : (size_t)ring_planes * pe * ring_tsize);
  };
  // stages in [2 (3 for identity operands), 4]: the most CTAs per SM (228 KB
  // of shared memory, ~5 KB static + 1 KB reserved per CTA), then the most stages
  auto ctas = [&]() { return (int)((228 * 1024) / (bytes() + 6 * 1024)); };
  int best = g.stages, bc = ctas();
  for (int st = g.stages - 1; st >= (ident ? 3 : 2); --st) {
    g.stages = st;
    if (ctas() > bc) {
      bc = ctas();
      best = st;
    }
  }
  g.stages = best;
  if (const char* e = std::getenv("GADI_ST25_STAGES")) g.stages = std::max(2, std::atoi(e));  // tuning knob
  g.smem = bytes();
  if (g.smem > 200 * 1024) return false;
  return true;
}

template <class P, int CPT>
inline void launch_st25_cpt(const P& pol, const St25Geo& g, cudaStream_t s, const Red& rd, DevState* st) {
  smem_attr(k_st25<P, CPT>, 200 * 1024);  // per device, once (monotonic cap, locked)
  k_st25<P, CPT><<<g.nblk, g.threads, g.smem, s>>>(pol, g, rd, st);
}
template <class P>
inline void launch_st25(const P& pol, const St25Geo& g, cudaStream_t s, const Red& rd, DevState* st) {
  switch (g.CPT) {  // chunks per thread per plane, a compile-time loop count
    case 1: return launch_st25_cpt<P, 1>(pol, g, s, rd, st);
    case 2: return launch_st25_cpt<P, 2>(pol, g, s, rd, st);
    default: return launch_st25_cpt<P, 4>(pol, g, s, rd, st);
  }
}

// k_resid64 (gadi_resid64.cuh): tile of threads*CPT 16-byte chunks per plane,
// S staged planes of TJ+2 rows. Variants (threads, CPT, CTAs per SM) are
// compile-time; GADI_R64 picks one (0: off, the k_st25 passes run).
inline int r64_variant() {  // read per launch (a test switch; one getenv per outer step)
  const char* e = std::getenv("GADI_R64");
  return e ? std::atoi(e) : 4;
}
inline bool make_r64(int64_t n, int64_t i0, int64_t i1, int threads, int cpt, int S, St25Geo& g) {
  if (i1 < 0) i1 = n;
  const int64_t nloc = i1 - i0;
  if (nloc < 1 || !is_pow2(nloc) || !is_pow2(n) || n < 64) return false;
  const int64_t TR = n / 2, chunks = (int64_t)threads * cpt;
  if (chunks % TR != 0) return false;
  const int64_t TJ = chunks / TR;
  if (TJ < 1 || TJ > n) return false;
  g.i0 = (int)i0;
  g.i1 = (int)i1;
  g.n = (int)n;
  g.lg = ilog2(n);
  g.nn = n * n;
  g.TR = (int)TR;
  g.lgTR = ilog2(TR);
  g.CPT = cpt;
  g.TJ = (int)TJ;
  g.lgTJ = ilog2(TJ);
  g.njt = (int)(n / TJ);
  int64_t IL = 32;
  while (IL > 4 && g.njt * (nloc / IL) < 2048) IL /= 2;
  if (const char* e = std::getenv("GADI_R64_IL")) IL = std::min(32, std::max(1, std::atoi(e)));  // tuning knob
  IL = std::min<int64_t>(IL, nloc);
  g.IL = (int)IL;
  g.nblk = (int)(g.njt * (nloc / IL));
  g.threads = threads;
  g.stages = S;
  g.smem = 128 + (size_t)S * ((TJ + 2) * n + 2) * sizeof(double);
  return g.smem <= 200 * 1024;
}
// the variant's (threads, CPT) and whether the shape and coefficients fit
inline bool r64_fits(int64_t n, int64_t i0, int64_t i1, const double (&c7)[7], St25Geo& g) {
  static const int TH[6] = {0, 512, 256, 256, 512, 512}, CP[6] = {0, 2, 4, 2, 4, 2}, SS[6] = {0, 4, 4, 4, 4, 8};
  const int v = r64_variant();
  if (v < 1 || v > 5) return false;
  for (int k = 0; k < 7; ++k)
    if (!std::isfinite(c7[k])) return false;
  return make_r64(n, i0, i1, TH[v], CP[v], SS[v], g);
}
template <class P, int CPT, int THREADS, int MINB, int S>
inline void launch_resid64_v(const P& pol, const St25Geo& g, cudaStream_t s, const Red& rd, DevState* st) {
  smem_attr(k_resid64<P, CPT, THREADS, MINB, S>, 200 * 1024);
  k_resid64<P, CPT, THREADS, MINB, S><<<g.nblk, THREADS, g.smem, s>>>(pol, g, rd, st);
}
template <class P>
inline void launch_resid64(const P& pol, const St25Geo& g, cudaStream_t s, const Red& rd, DevState* st) {
  // the variant r64_fits built g for (threads, chunks per thread, stages)
  if (g.threads == 512 && g.CPT == 2 && g.stages == 4) return launch_resid64_v<P, 2, 512, 1, 4>(pol, g, s, rd, st);
  if (g.threads == 256 && g.CPT == 4) return launch_resid64_v<P, 4, 256, 2, 4>(pol, g, s, rd, st);
  if (g.threads == 256 && g.CPT == 2) return launch_resid64_v<P, 2, 256, 2, 4>(pol, g, s, rd, st);
  if (g.threads == 512 && g.CPT == 2) return launch_resid64_v<P, 2, 512, 1, 8>(pol, g, s, rd, st);
  return launch_resid64_v<P, 4, 512, 1, 4>(pol, g, s, rd, st);
}

// k_st25h geometry: the k_st25 tiling with a padded 3-plane operand ring;
// stages chosen for the most CTAs per SM, then the most stages
inline bool make_st25h(int64_t n, int nin, St25Geo& g, int64_t i0, int64_t i1) {
  if (!make_st25(n, 2, nin, g, 512, false, 2, i0, i1, 3)) return false;
  if (g.TR < 32) return false;  // a warp's 32 chunks lie in one grid row
  const size_t pe = (size_t)(g.TJ + 2) * n, pr = (size_t)st25h_plane(g.TJ, (int)n);
  auto bytes = [&](int st) { return 128 + (size_t)st * nin * pe * 2 + 3 * pr * 2; };
  auto ctas = [&](int st) { return (int)((228 * 1024) / (bytes(st) + 4 * 1024)); };
  int best = 2;
  for (int st = 3; st <= 4; ++st)
    if (ctas(st) >= ctas(best)) best = st;
  if (const char* e = std::getenv("GADI_ST25_STAGES")) best = std::max(2, std::atoi(e));  // tuning knob
  g.stages = best;
  g.smem = bytes(best);
  return g.smem <= 200 * 1024;
}

template <class P, int CPT, int MINB>
inline void launch_st25h_cpt(const P& pol, const St25Geo& g, cudaStream_t s, const Red& rd, DevState* st) {
  smem_attr(k_st25h<P, CPT, MINB>, 200 * 1024);
  // persistent CTAs: as many as are resident at once, cached per (device,
  // shared memory, threads) under a lock (handles on several devices, and the
  // training-set probe threads, launch concurrently)
  int c_res = 0;
  {
    static std::mutex mu;
    static std::map<std::tuple<int, size_t, int>, int> cache;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, g.smem, g.threads});
    if (it == cache.end()) {
      int sms = 0, per = 0;
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_st25h<P, CPT, MINB>, g.threads, g.smem));
      int res = std::max(1, per) * sms;
      if (const char* e = std::getenv("GADI_ST25H_GRID")) res = std::max(1, std::atoi(e));  // tuning knob
      it = cache.emplace(std::make_tuple(dev, g.smem, g.threads), res).first;
    }
    c_res = it->second;
  }
  const int grid = std::min(g.nblk, c_res);
  k_st25h<P, CPT, MINB><<<grid, g.threads, g.smem, s>>>(pol, g, rd, st);
}
template <class P>
inline void launch_st25h(const P& pol, const St25Geo& g, cudaStream_t s, const Red& rd, DevState* st) {
  static const int minb = [] {  // tuning knob: register budget (CTAs per SM)
    const char* e = std::getenv("GADI_ST25H_MINB");
    return e ? std::atoi(e) : 2;
  }();
  if (minb == 2) {
    switch (g.CPT) {
      case 1: return launch_st25h_cpt<P, 1, 2>(pol, g, s, rd, st);
      case 2: return launch_st25h_cpt<P, 2, 2>(pol, g, s, rd, st);
      default: return launch_st25h_cpt<P, 4, 2>(pol, g, s, rd, st);
    }
  }
  switch (g.CPT) {
    case 1: return launch_st25h_cpt<P, 1, 3>(pol, g, s, rd, st);
    case 2: return launch_st25h_cpt<P, 2, 3>(pol, g, s, rd, st);
    default: return launch_st25h_cpt<P, 4, 3>(pol, g, s, rd, st);
  }
}

template <int V>
struct VecTag {
  static constexpr int v = V;
};

inline dim3 ew_grid(int64_t n) { return dim3((unsigned)((n + 255) / 256)); }

template <class T>
constexpr int prec_of() {
  return std::is_same<T, __half>::value ? GADI_HALF : std::is_same<T, float>::value ? GADI_SINGLE : GADI_DOUBLE;
}

}  // namespace gadi_host

// ==================================================================== handle
struct EngineBase;

// A SELL image (gadi_csr.cuh) owned on the device.
struct SellImage {
  int lgSR = 0;
  int64_t entries = 0;
  int64_t* soff = nullptr;
  uint16_t* len = nullptr;
  int32_t* col = nullptr;  // absolute columns, or
  int16_t* off = nullptr;  // column - row when every |column - row| < 2^15 (4 B/nnz instead of 6 in fp16)
  void* val = nullptr;
  void release() {
    for (void* p : {(void*)soff, (void*)len, (void*)col, (void*)off, val})
      if (p) cudaFree(p);
    soff = nullptr;
    len = nullptr;
    col = nullptr;
    off = nullptr;
    val = nullptr;
  }
};

struct gadi_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  int kind = GADI_PROBLEM_STENCIL7;
  int64_t N = 0, n = 0;
  double t1 = 0, t2 = 0, t3 = 0;
  // sparse A (CSR, device) and its SELL image for the binary64 residual
  int64_t* d_rpA = nullptr;
  int32_t* d_ciA = nullptr;
  double* d_vA = nullptr;
  int64_t nnzA = 0, nnzHS = 0;
  int64_t max_band = INT64_MAX;  // max |column - row| of A (the HSS union has the same band)
  SellImage sellA;
  // the HSS split on the union pattern (device): M, N in binary64, the
  // position of each diagonal entry and whether M's own pattern had it
  int64_t* d_urp = nullptr;
  int32_t* d_uci = nullptr;
  double *d_mv = nullptr, *d_nv = nullptr;
  int64_t* d_dpos = nullptr;
  uint8_t* d_din = nullptr;
  // explicit_splitting(A, M, N) (splitting.cpp:22-35; gadi_cuda_set_split): M
  // and N on their own patterns, each with the diagonal inserted where it has
  // none (shift_diagonal's pattern, sparse.cpp:180-183)
  struct SplitPart {
    int64_t* rp = nullptr;
    int32_t* ci = nullptr;
    double* v = nullptr;
    int64_t* dpos = nullptr;  // position of the diagonal entry of each row
    uint8_t* din = nullptr;   // 1: the matrix's own pattern had it
    int64_t nnz = 0;
  };
  bool explicit_split = false;
  SplitPart ex[2];
  int64_t ex_band = 0;  // max |column - row| over A, M and N
  int64_t hs_band() const { return explicit_split ? ex_band : max_band; }  // band of the H / S operators
  // M (which = 1) or N (which = 2) of the active split
  SplitPart part(int which) const {
    if (explicit_split) return ex[which - 1];
    return SplitPart{d_urp, d_uci, which == 1 ? d_mv : d_nv, d_dpos, d_din, nnzHS};
  }
  // outer vectors (binary64)
  double *d_x = nullptr, *d_b = nullptr, *d_s = nullptr, *d_t64 = nullptr;
  // reductions / state
  DevState* st = nullptr;
  DevState* h_st = nullptr;  // pinned mirror
  double *d_part0 = nullptr, *d_part1 = nullptr;
  double* d_partm = nullptr;  // block partials of the multi-dot pass (4 channels)
  int64_t partm_stride = 0;
  unsigned* d_ticket = nullptr;
  int* h_done = nullptr;  // mapped pinned flag (CG done)
  int* d_h_done = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evA = nullptr, evB = nullptr, evC = nullptr;
  std::vector<cudaEvent_t> ring;
  int64_t launches = 0;
  // Binary64 norms of the outer residual (norm2_64, kernels.cpp:184-194, scales
  // by max|s| so the squares neither underflow nor overflow): the passes sum
  // the squares of s 2^-ns, an exact scaling, and the host returns
  // 2^ns sqrt(sum). ns stays 0 while |ilogb(max|s|)| <= 400; beyond that the
  // pass is rerun with ns = ilogb(max|s|) (res_norm_ok).
  int ns = 0;
  // prepared inner engine
  std::unique_ptr<EngineBase> eng;
  double stop_norm = 1.0;
  std::vector<double> history;
  // sharded solves (gadi_dist.cuh): this rank's z-slab [i0, i1) of the n
  // planes (every slab vector has gh = n^2 ghost entries on each side), or
  // its CSR row block [row0, row0 + N) (gh = the band)
  int world = 1, rank = 0;
  int64_t i0 = 0, i1 = 0, gh = 0;
  std::unique_ptr<gadi_host::Comm> comm;
  uint64_t dist_seq = 0;
  std::vector<void*> raw;  // ghosted allocations (freed at destroy)

  bool stencil() const { return kind == GADI_PROBLEM_STENCIL7; }
  bool sharded() const { return comm != nullptr; }
  int64_t row0 = 0;  // CSR row block: first owned row
  int64_t e_off() const { return stencil() ? i0 * n * n : row0; }  // global index of local entry 0
};

namespace gadi_host {

template <class T>
T* dalloc(int64_t n);

// exclusive prefix sum of n int64 values (in -> out, out[n] = total when in[n] = 0)
inline void scan_i64(cudaStream_t s, const int64_t* in, int64_t* out, int64_t n) {
  size_t tmp = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
  void* t = nullptr;
  CK(cudaMalloc(&t, tmp));
  CK(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n, s));
  CK(cudaStreamSynchronize(s));
  cudaFree(t);
}

// SELL layout (slice offsets, row lengths, column image) of a device CSR
// pattern with 2^lgSR rows per slice (gadi_csr.cuh).
inline void build_sell_layout(cudaStream_t s, int64_t N, int lgSR, const int64_t* rp, const int32_t* ci,
                              SellImage& L, bool rel) {
  const int64_t SR = int64_t(1) << lgSR, ns = (N + SR - 1) / SR;
  L.lgSR = lgSR;
  int64_t* wid = dalloc<int64_t>(ns + 1);
  CK(cudaMemsetAsync(wid, 0, (ns + 1) * 8, s));
  L.len = dalloc<uint16_t>(N);
  k_sell_width<<<(unsigned)((ns + 255) / 256), 256, 0, s>>>(N, lgSR, rp, wid, L.len);
  CKL();
  L.soff = dalloc<int64_t>(ns + 1);
  scan_i64(s, wid, L.soff, ns + 1);
  cudaFree(wid);
  CK(cudaMemcpy(&L.entries, L.soff + ns, 8, cudaMemcpyDeviceToHost));
  if (rel) {
    L.off = dalloc<int16_t>(L.entries);
    CK(cudaMemsetAsync(L.off, 0, L.entries * 2, s));
  } else {
    L.col = dalloc<int32_t>(L.entries);
    CK(cudaMemsetAsync(L.col, 0, L.entries * 4, s));
  }
  k_sell_fill<double, P_DOUBLE><<<(unsigned)((N + 255) / 256), 256, 0, s>>>(
      N, lgSR, rp, ci, nullptr, L.soff, L.col, L.off, (double*)nullptr, nullptr, nullptr, 0.0);
  CKL();
  CK(cudaStreamSynchronize(s));
}

// values of a device CSR (binary64) into a SELL layout as VO, rounded to
// precision PR, the diagonal shifted by alpha when dpos is given.
template <class VO, int PR>
inline VO* fill_sell_values(cudaStream_t s, int64_t N, const SellImage& L, const int64_t* rp, const double* val,
                            const int64_t* dpos, const uint8_t* din, double alpha) {
  VO* out = dalloc<VO>(L.entries);
  CK(cudaMemsetAsync(out, 0, L.entries * sizeof(VO), s));
  k_sell_fill<VO, PR><<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, L.lgSR, rp, nullptr, val, L.soff, nullptr,
                                                                  nullptr, out, dpos, din, alpha);
  CKL();
  CK(cudaStreamSynchronize(s));
  return out;
}

}  // namespace gadi_host

namespace gadi_host {

template <class T>
T* dalloc(int64_t n) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<int64_t>(n, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

// The scalar head of the device state (cols = 0), plus the Arnoldi column (cols = 1) or the
// columns of a speculative window as well (cols = 2).
inline void read_state(gadi_handle* h, int cols = 0) {
  const size_t bytes = cols == 0 ? offsetof(DevState, hcol) : cols == 1 ? offsetof(DevState, hhist) : offsetof(DevState, ycoef);
  CK(cudaMemcpyAsync(h->h_st, h->st, bytes, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
}

inline Red red_of(gadi_handle* h) { return Red{h->d_part0, h->d_part1, h->d_ticket}; }

// 2^-ns for the residual passes; the norms they reduced (after read_state)
inline double nsc_of(int ns) { return ns == 0 ? 1.0 : std::ldexp(1.0, -ns); }
inline double res_norm(const gadi_handle* h) { return std::ldexp(std::sqrt(h->h_st->res_ss), h->ns); }
// After a residual pass and read_state: true when max|s| lies within 2^+-400
// of the scale the squares were taken at (the sum is then the exact scaled
// sum); otherwise ns is moved to ilogb(max|s|) and the caller reruns the pass.
inline bool res_norm_ok(gadi_handle* h) {
  const double mx = h->h_st->res_max;
  if (!(mx > 0.0) || !std::isfinite(mx)) return true;
  const int e = std::ilogb(mx);
  if (std::abs(e - h->ns) <= 400) return true;
  h->ns = std::abs(e) <= 400 ? 0 : e;
  return false;
}

// A slab vector of the handle: N entries with h->gh ghost entries on each
// side (zero-filled), the interior pointer returned.
template <class T>
T* hvec(gadi_handle* h, int64_t n_extra = 0) {
  T* p = dalloc<T>(h->N + 2 * h->gh + n_extra);
  CK(cudaMemset(p, 0, (h->N + 2 * h->gh + n_extra) * sizeof(T)));
  h->raw.push_back(p);
  return p + h->gh;
}

// Sharded solves: complete a reduction whose kernel parked its record
// (finish_red) -- all-gather the records, fold them in rank order and apply
// the epilogue on every rank. A no-op on one device.
template <class C0, class Epi>
inline void coll(gadi_handle* h, const Epi& e) {
  if (!h->sharded()) return;
  const int half = (int)(h->dist_seq++ & 1);
  h->comm->allgather4(h->st->dist_loc[half], h->st->dist_all[half], h->stream);
  k_dist_finish<Epi, C0><<<1, 1, 0, h->stream>>>(e, h->st, h->world, half);
  CKL();
}
// flag / max words only (kernels without a grid reduction)
inline void coll_flags(gadi_handle* h, int* flags) {
  if (!h->sharded()) return;
  k_dist_pack<<<1, 1, 0, h->stream>>>(h->st, flags);
  coll<double>(h, EpiNone{flags});
}
// the ghost entries of a shard vector (a plane of a z-slab, the band of a
// CSR row block) before an operator pass reads them
template <class T>
inline void halo(gadi_handle* h, const T* interior) {
  if (!h->sharded()) return;
  h->comm->halo(reinterpret_cast<char*>(const_cast<T*>(interior)), h->gh * (int64_t)sizeof(T),
                h->N * (int64_t)sizeof(T), h->stream);
}

// ------------------------------------------------------------ outer kernels on A
struct OuterA {
  // s = b - A x in u_f; s == nullptr computes the norm only.
  static void resid(gadi_handle* h, const double* x, double* s, int uf, bool scaling) {
    CK(cudaMemsetAsync(&h->st->maxbits, 0, sizeof(unsigned long long), h->stream));
    halo(h, x);
    const int64_t eo = h->e_off();  // stencil kernels index by global row
    const bool al = aligned_for(h->N, h->n, h->stencil(), 2);
    Geo g = make_geo(h->N, al ? 2 : 1);
    g.gh = h->gh;
    const Window win = h->stencil() ? Window{} : window_for(g, 2, sizeof(double), h->max_band, al);
    auto go = [&](auto op) {
      auto L = [&](auto pt, auto vt) {
        constexpr int PF = decltype(pt)::v, V = decltype(vt)::v;
        auto kern = k_resid_A<decltype(op), PF, V>;
        smem_attr(kern, win.bytes);
        kern<<<g.nblk, g.threads(), win.bytes, h->stream>>>(op, x, h->d_b, s, scaling ? 1 : 0, g, red_of(h), h->st,
                                                            win.band, nsc_of(h->ns));
      };
      auto LV = [&](auto pt) {
        if (al) L(pt, VecTag<2>{});
        else L(pt, VecTag<1>{});
      };
      if (uf == GADI_HALF) LV(VecTag<P_HALF>{});
      else if (uf == GADI_SINGLE) LV(VecTag<P_SINGLE>{});
      else LV(VecTag<P_DOUBLE>{});
    };
    St25Geo g25;
    bool done64 = false;
    if (h->stencil() && uf == GADI_DOUBLE) {
      PolResidA<P_DOUBLE> pol{{h->t2, h->t2, h->t2, h->t1, h->t3, h->t3, h->t3}, x - eo, h->d_b - eo,
                              s ? s - eo : nullptr, scaling ? 1 : 0, nsc_of(h->ns)};
      if ((done64 = r64_fits(h->n, h->i0, h->i1, pol.c7, g25)))
        launch_resid64(pol, g25, h->stream, red_of(h), h->st);
    }
    if (done64) {
    } else if (h->stencil() && make_st25(h->n, 8, 1, g25, 1024, true, 0, h->i0, h->i1)) {
      auto L = [&](auto pt) {
        constexpr int PF = decltype(pt)::v;
        PolResidA<PF> pol{{h->t2, h->t2, h->t2, h->t1, h->t3, h->t3, h->t3}, x - eo, h->d_b - eo,
                          s ? s - eo : nullptr, scaling ? 1 : 0, nsc_of(h->ns)};
        launch_st25(pol, g25, h->stream, red_of(h), h->st);
      };
      if (uf == GADI_HALF) L(VecTag<P_HALF>{});
      else if (uf == GADI_SINGLE) L(VecTag<P_SINGLE>{});
      else L(VecTag<P_DOUBLE>{});
    } else if (h->stencil()) {
      Stencil7<double> op{h->n, h->n * h->n, h->N, {h->t2, h->t2, h->t2, h->t1, h->t3, h->t3, h->t3}, lg_of(h->n)};
      op.i_off = h->i0;
      go(op);
    } else {
      Sell<double> op{h->N, h->sellA.lgSR, h->sellA.soff, h->sellA.len, h->sellA.col,
                      static_cast<const double*>(h->sellA.val), h->sellA.off};
      go(op);
    }
    CKL();
    ++h->launches;
    coll<double>(h, EpiResidA{scaling ? 1 : 0});
  }
  // resid + read_state, rerun once if max|s| is far from the norm scale
  static void resid_sync(gadi_handle* h, const double* x, double* s, int uf, bool scaling) {
    for (int pass = 0; pass < 2; ++pass) {
      resid(h, x, s, uf, scaling);
      read_state(h);
      if (res_norm_ok(h)) return;
    }
  }
  static void apply(gadi_handle* h, const double* x, double* y) {
    auto go = [&](auto op) {
      k_apply<decltype(op), double, double, double><<<ew_grid(h->N), 256, 0, h->stream>>>(op, x, y, h->N,
                                                                                          MatvecAF());
    };
    if (h->stencil()) {
      Stencil7<double> op{h->n, h->n * h->n, h->N, {h->t2, h->t2, h->t2, h->t1, h->t3, h->t3, h->t3}, lg_of(h->n)};
      op.i_off = h->i0;
      go(op);
    } else {
      Sell<double> op{h->N, h->sellA.lgSR, h->sellA.soff, h->sellA.len, h->sellA.col,
                      static_cast<const double*>(h->sellA.val), h->sellA.off};
      go(op);
    }
    CKL();
    ++h->launches;
  }
};

}  // namespace gadi_host

// ================================================================== engines
struct InnerOut {
  int iters = 0;
  int status = INNER_CONVERGED;
};

// A device band LU factorization (gadi_lu.cu; BandLU, band_lu.cpp).
struct LuFactor {
  int device = 0, prec = GADI_DOUBLE;
  int64_t N = 0, kl = 0, ku = 0, ldab = 1;
  void* ab = nullptr;         // ldab x N band (binary64, or binary32 for single/half)
  int32_t* ipiv = nullptr;    // N pivot rows
  void* xw = nullptr;         // solve work vector (N)
  int* err = nullptr;         // [0] 1 singular / 2 non-finite, [1] column, [2] solve non-finite
  int* bad = nullptr;
  unsigned* flags = nullptr;  // pipelined solves: per-block epoch flags, then the block ticket
  unsigned* ticket = nullptr;
  unsigned long long* xt = nullptr;  // binary32 sweeps: (value | epoch << 32) words
  unsigned epoch = 0;
  bool swaps = false;         // any row interchange (forward solve needs the swap-aware kernel)
  int sms = 148;
  int64_t launches = 0;
};
namespace gadi_host {
LuFactor* lu_factor_build(gadi_handle* h, int which, double alpha, int ur, int* status);
void lu_release(LuFactor* f, cudaStream_t s = nullptr);  // stream-ordered free (no device sync)
InnerOut lu_inner_solve(LuFactor* f, const void* rhs, void* x, cudaStream_t s);
LuFactor* lu_factor_host_csr(int device, cudaStream_t s, int64_t N, const int64_t* rp, const int64_t* ci,
                             const double* v, double alpha, int ur, int* status);
bool lu_solve_many(LuFactor* f, double* X, int64_t es, int64_t rs, int64_t nrhs, cudaStream_t s);
}  // namespace gadi_host

// The inner solvers for one (operator, storage, arithmetic) choice.
struct EngineBase {
  virtual ~EngineBase() {
    for (LuFactor*& f : lu) {
      gadi_host::lu_release(f, nullptr);
      f = nullptr;
    }
  }
  LuFactor* lu[3] = {nullptr, nullptr, nullptr};  // LuDirect factors of H (1) and S (2)
  int u_r = GADI_DOUBLE, accum = 0, cprec = GADI_DOUBLE;
  size_t tsize = 8;
  gadi_inner_spec spec{};
  double alpha = 1, omega = 1;
  // inner-format device vectors (type-erased)
  void *rhat = nullptr, *z = nullptr, *pz = nullptr, *y = nullptr;
  // set by the outer loop right before cg(): rhs is the rhat an outer residual pass just
  // produced, and st->rhat_ss holds its binary64 sum of squares at scale 2^0 (consumed by cg)
  bool rhs_ss_known = false;
  // H/S solves on inner-format device vectors; CG consumes rhs (r in place)
  virtual InnerOut cg(int which, void* rhs, void* x, double target) = 0;
  virtual InnerOut gmres(int which, const void* rhs, void* x, double target) = 0;
  // rhat = round(s 2^-e); the squares of rhat are taken at 2^-ns_r (0 when
  // the residual scaling put max|rhat| in [1, 2), else the residual's ns)
  virtual void scale_round(const double* s, int ns_r) = 0;
  // rhat = round(s 2^-ep) straight from the residual pass (u_f binary64,
  // stencil operators); false: not available for this operator / shape
  virtual bool resid_spec(const double* x, int ep, bool scaling) = 0;
  virtual void scale_pz(double phat) = 0;                   // pz = round(phat z)
  // pz = round(phat z) deferred: gmres(2, pz) forms it inside its zero-start
  // residual pass and stores pz only if a later pass needs it (restart /
  // happy-breakdown residual).
  void defer_pz(double phat) {
    pz_phat = phat;
    pz_lazy = true;
  }
  double pz_phat = 0.0;
  bool pz_lazy = false;
  virtual void update(double* x, int pu) = 0;               // x += 2^e y
  virtual void to_inner(const double* src, void* dst) = 0;  // round_vec to u_r
  virtual void to_double(const void* src, double* dst) = 0;
  virtual void apply(int which, const void* x, void* yv) = 0;
  virtual bool set_alpha(double a, double om) = 0;  // false: rebuild the engine
};

namespace gadi_host {

// The engines' work vectors come from a library-owned stream-ordered pool per
// device (the process's default pool and its attributes are left alone). It
// keeps what a solve used for the next one; gadi_cuda_destroy trims it to 256 MB
// (engine_pool_trim) so a destroyed C3-sized engine does not hold its GBs.
inline cudaMemPool_t engine_pool(int dev) {
  static cudaMemPool_t pools[64] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  cudaMemPool_t& p = pools[dev & 63];
  if (!p) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    CK(cudaMemPoolCreate(&p, &props));
    uint64_t keep = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  return p;
}
inline void engine_pool_trim(int dev) { cudaMemPoolTrimTo(engine_pool(dev), (size_t)256 << 20); }  // keep 256 MB for the next small handle

template <class Op, class T, class C>
struct Engine final : EngineBase {
  gadi_handle* h;
  Op opH, opS;
  bool aligned;
  Geo geo;
  static constexpr int VA = 16 / sizeof(T);
  static constexpr bool SPARSE = !std::is_same<Op, Stencil7<C>>::value;
  // binary16 storage with binary32 arithmetic (GADI_ACCUM_FP32): the fused two-pass Gram-Schmidt
  static constexpr bool FUSED_GS = std::is_same<T, __half>::value && std::is_same<C, float>::value;
  // CG / GMRES work vectors
  T *pA = nullptr, *pB = nullptr, *q = nullptr, *wA = nullptr, *wB = nullptr, *gr = nullptr, *V = nullptr;
  int64_t ldv = 0;  // basis stride
  using OV = typename Op::value_type;
  OV* dH = nullptr;  // sparse operators: H / S values in the SELL image sHS
  OV* dS = nullptr;
  uint8_t *zfH = nullptr, *zfS = nullptr;  // per-row zflag summaries of H / S (residual from x = 0)
  SellImage sHS, sS2;
  int m_restart = 30;
  std::vector<T*> owned;
  bool st25 = false;  // 2.5D TMA stencil kernels (gadi_st25.cuh) for the operator passes
  St25Geo g25;        // CG p-update + SpMV: two staged inputs + operand ring
  St25Geo g25m;       // Arnoldi matvec: one staged input + operand ring
  St25Geo g25i;       // GMRES residual: identity operand, folded from the stages
  bool st25h = false;  // binary16 operator passes with register-resident operands (k_st25h)
  bool st25h_geo = false;
  St25Geo g25h, g25mh;  // their geometries (3-plane operand ring)
  Window win;         // sparse operators: operand window in shared memory

  // Work vectors come from the device's stream-ordered memory pool (kept,
  // not released, between solves): re-preparing an engine -- every
  // gadi_ir_solve does (solver.cpp:75) -- costs no cudaMalloc/cudaFree and no
  // device-wide synchronisation.
  T* salloc(int64_t n) {
    T* p = nullptr;
    CK(cudaMallocFromPoolAsync((void**)&p, (size_t)n * sizeof(T), engine_pool(h->device), h->stream));
    return p;
  }

  T* vec() {  // a slab vector (ghost planes when sharded)
    T* v = salloc(h->N + 2 * h->gh);
    if (h->gh) CK(cudaMemsetAsync(v, 0, (h->N + 2 * h->gh) * sizeof(T), h->stream));
    owned.push_back(v);
    return v + h->gh;
  }

  Engine(gadi_handle* hh, const gadi_inner_spec& sp, double a, double om, int ur, int acc) : h(hh) {
    u_r = ur;
    accum = acc;
    cprec = std::is_same<C, __half>::value ? GADI_HALF : std::is_same<C, float>::value ? GADI_SINGLE : GADI_DOUBLE;
    tsize = sizeof(T);
    spec = sp;
    alpha = a;
    omega = om;
    const int64_t N = h->N;
    aligned = aligned_for(N, h->n, h->stencil(), VA);
    geo = make_geo(N, aligned ? VA : 1);
    geo.gh = h->gh;
    if constexpr (SPARSE) win = window_for(geo, VA, sizeof(T), h->hs_band(), aligned);
    if constexpr (std::is_same<Op, Stencil7<C>>::value) {
      constexpr int rsz = sizeof(typename RingOf<T, C>::type);
      st25 = make_st25(h->n, sizeof(T), 2, g25, 512, false, rsz, h->i0, h->i1) &&
             make_st25(h->n, sizeof(T), 1, g25m, 512, false, rsz, h->i0, h->i1) &&
             make_st25(h->n, sizeof(T), 1, g25i, 512, true, 0, h->i0, h->i1);
      if constexpr (PolSpmvp<T, C>::FASTH) {
        const char* e = std::getenv("GADI_ST25H");
        st25h = st25 && !(e && e[0] == '0') &&
                make_st25h(h->n, 2, g25h, h->i0, h->i1) && make_st25h(h->n, 1, g25mh, h->i0, h->i1);
        st25h_geo = st25h;
      }
    }
    if (h->sharded() && !SPARSE && !st25)
      throw Err(GADI_E_UNSUPPORTED, "sharded solve: the slab shape needs the st25 kernels");
    m_restart = std::max(1, spec.restart);
    rhat = vec();
    z = vec();
    pz = vec();
    y = vec();
    pA = vec();
    pB = vec();
    q = vec();
    wA = vec();
    wB = vec();
    gr = vec();
    // basis: m+1 vectors of ldv = N + 2 gh entries (a sharded sparse matvec
    // reads its operand v_j, a basis vector, at the ghost entries)
    ldv = N + 2 * h->gh;
    T* vb = salloc((int64_t)(m_restart + 1) * ldv);
    if (h->gh) CK(cudaMemsetAsync(vb, 0, (int64_t)(m_restart + 1) * ldv * sizeof(T), h->stream));
    owned.push_back(vb);
    V = vb + h->gh;
    build_ops();
    check_st25h();
  }

  void check_st25h() {
    if constexpr (std::is_same<Op, Stencil7<C>>::value && PolSpmvp<T, C>::FASTH) {
      st25h = st25h_geo;
      for (int k = 0; k < 7; ++k)  // k_st25h folds neutral operands at the boundary: finite coefficients only
        if (!std::isfinite((double)opH.c[k]) || !std::isfinite((double)opS.c[k])) st25h = false;
    }
  }

  // A new (alpha, omega) on the same vectors: the stencil operators are seven
  // coefficients, rebuilt in place (no device allocation, so no implicit
  // device-wide synchronisation between concurrent handles).
  bool set_alpha(double a, double om) override {
    if constexpr (SPARSE) {
      return false;
    } else {
      alpha = a;
      omega = om;
      build_ops();
      check_st25h();
      return true;
    }
  }

  ~Engine() override {
    for (T* v : owned) cudaFreeAsync(v, h->stream);  // allocation bases, back to the pool
    if (dH) cudaFree(dH);
    if (dS) cudaFree(dS);
    sHS.release();
    sS2.release();
    if (zfH) cudaFree(zfH);
    if (zfS) cudaFree(zfS);
  }

  static C cval(double v, int ur) {
    // matrix values are rounded to u_r (rounded_copy, inner_solver.cpp:41-45)
    const double r = hround(v, ur);
    if constexpr (std::is_same<C, __half>::value) return __double2half(r);
    else return (C)r;
  }

  void build_ops() {
    // regularize (splitting.cpp:37-47): H = shift_diagonal(M, alpha), S = shift_diagonal(N, alpha),
    // the shift being 1.0*M_ii + alpha (sparse.cpp:166-183).
    if constexpr (std::is_same<Op, Stencil7<C>>::value) {
      const double t1 = h->t1, t2 = h->t2, t3 = h->t3;
      const double ml = 0.5 * t2 + 0.5 * t3, mc = 0.5 * t1 + 0.5 * t1, mu = 0.5 * t3 + 0.5 * t2;
      const double nl = 0.5 * t2 + -0.5 * t3, nc = 0.5 * t1 + -0.5 * t1, nu = 0.5 * t3 + -0.5 * t2;
      const double hc = 1.0 * mc + alpha, sc = 1.0 * nc + alpha;
      const double Hc[7] = {ml, ml, ml, hc, mu, mu, mu};
      const double Sc[7] = {nl, nl, nl, sc, nu, nu, nu};
      opH.n = opS.n = h->n;
      opH.nn = opS.nn = h->n * h->n;
      opH.N = opS.N = h->N;
      opH.lg = opS.lg = lg_of(h->n);
      opH.i_off = opS.i_off = h->i0;
      auto zf = [&](double v) {  // zflag of the u_r-rounded coefficient (gadi_ops.cuh)
        const double r = hround(v, u_r);
        return (uint8_t)((std::signbit(r) ? 1 : 0) | (std::isfinite(r) ? 0 : 2));
      };
      for (int k = 0; k < 7; ++k) {
        opH.c[k] = cval(Hc[k], u_r);
        opS.c[k] = cval(Sc[k], u_r);
        opH.zc[k] = zf(Hc[k]);
        opS.zc[k] = zf(Sc[k]);
      }
    } else {
      // SELL image of the union pattern with VA rows per lane, values of
      // H / S rounded to u_r (rounded_copy, inner_solver.cpp:41-45) on the device
      // (an explicit split has one pattern per operator: S gets its own image sS2)
      const auto pH = h->part(1), pS = h->part(2);
      const bool rel = h->hs_band() < 32768;
      build_sell_layout(h->stream, h->N, ilog2(32 * VA), pH.rp, pH.ci, sHS, rel);
      if (h->explicit_split) build_sell_layout(h->stream, h->N, ilog2(32 * VA), pS.rp, pS.ci, sS2, rel);
      const SellImage& iS = h->explicit_split ? sS2 : sHS;
      auto fill = [&](const SellImage& im, const gadi_handle::SplitPart& pt) -> OV* {
        if (u_r == GADI_HALF)
          return fill_sell_values<OV, P_HALF>(h->stream, h->N, im, pt.rp, pt.v, pt.dpos, pt.din, alpha);
        if (u_r == GADI_SINGLE)
          return fill_sell_values<OV, P_SINGLE>(h->stream, h->N, im, pt.rp, pt.v, pt.dpos, pt.din, alpha);
        return fill_sell_values<OV, P_DOUBLE>(h->stream, h->N, im, pt.rp, pt.v, pt.dpos, pt.din, alpha);
      };
      dH = fill(sHS, pH);
      dS = fill(iS, pS);
      auto zflags = [&](const SellImage& im, const OV* v) {
        uint8_t* z = dalloc<uint8_t>(h->N);
        k_sell_zflags<OV><<<(unsigned)((h->N + 255) / 256), 256, 0, h->stream>>>(h->N, im.lgSR, im.soff, im.len, v, z);
        CKL();
        return z;
      };
      zfH = zflags(sHS, dH);
      zfS = zflags(iS, dS);
      opH = Op{h->N, sHS.lgSR, sHS.soff, sHS.len, sHS.col, dH, sHS.off, zfH};
      opS = Op{h->N, iS.lgSR, iS.soff, iS.len, iS.col, dS, iS.off, zfS};
    }
  }

  template <class F>
  void V2(F&& f) {
    if (aligned) f(VecTag<VA>{});
    else f(VecTag<1>{});
  }

  const Op& op(int which) const { return which == 1 ? opH : opS; }

  // The 2.5D TMA stencil versions of the operator passes (gadi_st25.cuh);
  // each returns false when it does not apply (CSR, or a grid shape the
  // plane marcher does not cover) and the generic kernel runs instead.
  bool spmvp25(const Op& o, const T* r, const T* p_in, T* p_out, int first) {
    if constexpr (std::is_same<Op, Stencil7<C>>::value) {
      if (!st25) return false;
      const int64_t eo = h->e_off();  // the st25 kernels index by global row
      PolSpmvp<T, C> pol{{o.c[0], o.c[1], o.c[2], o.c[3], o.c[4], o.c[5], o.c[6]},
                         r - eo, p_in - eo, p_out - eo, q - eo, Ar_beta(), first};
      if constexpr (PolSpmvp<T, C>::FASTH)
        if (st25h) {
          launch_st25h(pol, g25h, h->stream, red_of(h), h->st);
          return true;
        }
      launch_st25(pol, g25, h->stream, red_of(h), h->st);
      return true;
    } else {
      return false;
    }
  }
  bool gmmatvec25(const Op& o, const T* wprev, double inv, T* vj, T* w, bool inv_dev = false) {
    if constexpr (std::is_same<Op, Stencil7<C>>::value) {
      if (!st25) return false;
      const int64_t eo = h->e_off();
      PolGmMatvec<T, C> pol{{o.c[0], o.c[1], o.c[2], o.c[3], o.c[4], o.c[5], o.c[6]}, wprev - eo, inv, vj - eo,
                            V - eo, w - eo};
      pol.inv_dev = inv_dev ? 1 : 0;
      if constexpr (PolGmMatvec<T, C>::FASTH)
        if (st25h) {
          launch_st25h(pol, g25mh, h->stream, red_of(h), h->st);
          return true;
        }
      launch_st25(pol, g25m, h->stream, red_of(h), h->st);
      return true;
    } else {
      return false;
    }
  }
  bool gmresid25(const Op& o, const T* x, const T* rhs) {
    if constexpr (std::is_same<Op, Stencil7<C>>::value) {
      if (!st25) return false;
      const int64_t eo = h->e_off();
      PolGmResid<T, C> pol{{o.c[0], o.c[1], o.c[2], o.c[3], o.c[4], o.c[5], o.c[6]}, x - eo, rhs - eo, gr - eo};
      launch_st25(pol, g25i, h->stream, red_of(h), h->st);
      return true;
    } else {
      return false;
    }
  }
  // beta for the fused p-update is read by the kernel from the device state;
  // the policy carries a placeholder the kernel overwrites (see PolSpmvp::beta).
  static C Ar_beta() { return C(); }

  // ------------------------------------------------------------------ CG
  // inner_solver.cpp:47-83 on the device: per iteration one fused
  // (p-update + SpMV + p.q) pass and one fused (two axpys + r.r + ||r||)
  // pass. The host keeps at most ring.size() iterations queued ahead and stops
  // queueing once the device raises the mapped done flag.
  InnerOut cg(int which, void* rhs_v, void* x_v, double target) override {
    T* r = static_cast<T*>(rhs_v);
    T* x = static_cast<T*>(x_v);
    cudaStream_t s = h->stream;
    const Red rd = red_of(h);
    const Op& o = op(which);
    const int nt = geo.threads();
    *(volatile int*)h->h_done = 0;
    bool known = rhs_ss_known && rhs_v == rhat;
    rhs_ss_known = false;
    if (known && std::getenv("GADI_CHECK_SS")) {
      // self-check (tests): reduce the binary64 sum here too and compare it with the outer pass's
      V2([&](auto vt) {
        constexpr int V_ = decltype(vt)::v;
        k_cg_init<T, C, V_, true><<<geo.nblk, nt, 0, s>>>(r, spec.max_inner_iters, target, geo, rd, h->st);
      });
      CKL();
      coll<C>(h, EpiCgInit{spec.max_inner_iters, target, 0});
      read_state(h);
      if (std::memcmp(&h->h_st->red_d, &h->h_st->rhat_ss, sizeof(double)) != 0)
        throw Err{GADI_E_STATE, "k_cg_init: the outer pass's sum of squares of rhat differs from the CG pass's"};
    }
    V2([&](auto vt) {
      constexpr int V_ = decltype(vt)::v;
      if (known) k_cg_init<T, C, V_, false><<<geo.nblk, nt, 0, s>>>(r, spec.max_inner_iters, target, geo, rd, h->st);
      else k_cg_init<T, C, V_, true><<<geo.nblk, nt, 0, s>>>(r, spec.max_inner_iters, target, geo, rd, h->st);
    });
    CKL();
    ++h->launches;
    coll<C>(h, EpiCgInit{spec.max_inner_iters, target, known ? 1 : 0});
    const int kAhead = (int)h->ring.size();
    for (int it = 0; it < spec.max_inner_iters; ++it) {
      if (it >= kAhead) {
        CK(cudaEventSynchronize(h->ring[it % kAhead]));
        const int hd = *(volatile int*)h->h_done;
        // sharded: stop where the decision was made at or before the synced
        // iteration, so every rank queues the same collectives
        if (h->sharded() ? (hd && hd - 2 <= it - kAhead) : hd != 0) break;
      }
      T* p_in = (it & 1) ? pA : pB;
      T* p_out = (it & 1) ? pB : pA;
      const int first = it == 0;
      if (h->sharded() && !SPARSE) {  // the stencil pass reads r and p_old on the neighbours' boundary planes
        halo(h, r);
        if (!first) halo(h, p_in);
      }
      V2([&](auto vt) {
        constexpr int V_ = decltype(vt)::v;
        if constexpr (SPARSE) {  // p-update as its own pass: a gathered operand is not re-formed per nonzero
          k_cg_pupd<T, C, V_><<<geo.nblk, nt, 0, s>>>(r, p_in, p_out, first, geo, h->st);
          halo(h, p_out);  // a row block's SpMV reads p at the band beyond its rows
          auto kern = k_cg_spmvp<Op, T, C, V_, false>;
          smem_attr(kern, win.bytes);
          kern<<<geo.nblk, nt, win.bytes, s>>>(o, r, p_out, p_out, q, first, geo, rd, h->st, win.band);
          ++h->launches;
        } else if (!spmvp25(o, r, p_in, p_out, first)) {
          k_cg_spmvp<Op, T, C, V_><<<geo.nblk, nt, 0, s>>>(o, r, p_in, p_out, q, first, geo, rd, h->st);
        }
        coll<C>(h, EpiCgPap{});
        // the residual vector is dead after the last possible iteration (the next outer step rewrites rhat)
        k_cg_update<T, C, V_><<<geo.nblk, nt, 0, s>>>(x, r, p_out, q, first, geo, rd, h->st,
                                                      it + 1 < spec.max_inner_iters ? 1 : 0);
        coll<C>(h, EpiCgUpdate{});
      });
      CKL();
      h->launches += 2;
      CK(cudaEventRecord(h->ring[it % kAhead], s));
    }
    read_state(h);
    if (!h->h_st->cg_xvalid) CK(cudaMemsetAsync(x, 0, h->N * sizeof(T), s));  // x = 0 (:51)
    InnerOut out;
    out.iters = h->h_st->cg_iters;
    out.status = h->h_st->cg_status;
    return out;
  }

  // --------------------------------------------------------------- GMRES
  // inner_solver.cpp:85-194: vector work on the device (the basis scaling
  // fused into the next matvec, MGS fused with the next Arnoldi dot), the
  // (m+1) x m Hessenberg / Givens / back-solve on the host in the inner
  // format's rounding, exactly as the reference orders them.
  InnerOut gmres(int which, const void* rhs_v, void* x_v, double target) override {
    const T* rhs = static_cast<const T*>(rhs_v);
    T* x = static_cast<T*>(x_v);
    cudaStream_t s = h->stream;
    const Red rd = red_of(h);
    const Op& o = op(which);
    const int64_t N = h->N;
    const int m = m_restart, fmt = cprec, nt = geo.threads();
    auto Rf = [&](double v) { return hround(v, fmt); };
    std::vector<double> Hc((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), yv(m + 1);
    auto HC = [&](int i, int j) -> double& { return Hc[(size_t)i * m + j]; };
    int total = 0, status = -1;
    bool x_zero = true;  // x = 0 until the first update (inner_solver.cpp:92)
    bool lazy = rhs_v == pz && pz_lazy;  // rhs = round(pz_phat z), not stored yet
    pz_lazy = false;
    // Speculative Arnoldi windows (fused mode on the st25 passes): the steps of a window are
    // queued back to back -- each step's basis scaling 1 / h(j+1, j) is formed on the device
    // (gm_inv) and its column kept in hhist -- and the host reads the whole window with one
    // sync, then rotates the columns in order. A step past the one where the host stops
    // (convergence, breakdown, overflow) only wrote basis / work vectors nobody reads.
    const char* spec_e = std::getenv("GADI_GM_SPEC");  // a test switch, read per solve
    const bool spec_env = !spec_e || std::atoi(spec_e) != 0;
    const bool spec_ok = FUSED_GS && !SPARSE && st25 && spec_env;
    auto resid = [&](bool sync = true) {  // r = rhs - S x ; flags, max, ||r||_2 (binary64), norm2 in fmt
      if (lazy && !x_zero) {
        scale_pz(pz_phat);
        lazy = false;
      }
      CK(cudaMemsetAsync(&h->st->maxbits, 0, 8, s));
      CK(cudaMemsetAsync(&h->st->flags, 0, 4, s));
      if constexpr (FUSED_GS) {
        if (x_zero) {  // one pass: r, ||r|| (binary64), beta = sqrt(dot(r, r)) (binary32), finiteness
          V2([&](auto vt) {
            constexpr int V_ = decltype(vt)::v;
            if constexpr (V_ == 8 && !SPARSE) {
              // packed pass: phat is a binary16 value (solver.cpp:117 rounds it to u_r), so HMUL2 scales
              const __half ph = __float2half_rn((float)pz_phat);
              if (!lazy || (double)__half2float(ph) == pz_phat) {
                const uint32_t pb = __half_as_ushort(ph);
                k_gm_resid0p<Op><<<geo.nblk, nt, 0, s>>>(o, lazy ? static_cast<const T*>(z) : rhs, gr, geo, rd, h->st,
                                                         lazy ? 1 : 0, pb | (pb << 16));
                return;
              }
            }
            k_gm_resid0<Op, V_><<<geo.nblk, nt, 0, s>>>(o, rhs, gr, geo, rd, h->st,
                                                        lazy ? static_cast<const T*>(z) : nullptr, pz_phat);
          });
          coll<C>(h, EpiResidF{});
          CKL();
          ++h->launches;
          if (sync) read_state(h);
          return;
        }
      }
      V2([&](auto vt) {
        constexpr int V_ = decltype(vt)::v;
        if (!x_zero) halo(h, x);
        if (x_zero || !gmresid25(o, x, rhs)) {
          auto kern = k_gm_resid<Op, T, C, V_>;
          const size_t sm = x_zero ? 0 : win.bytes;
          smem_attr(kern, sm);
          kern<<<geo.nblk, nt, sm, s>>>(o, x, x_zero ? 1 : 0, rhs, gr, geo, rd, h->st, x_zero ? 0 : win.band,
                                        lazy ? static_cast<const T*>(z) : nullptr, pz_phat);
        }
        coll<C>(h, EpiRedD{});
        if constexpr (FUSED_GS) {  // the fused mode's norm: beta = sqrt(dot(r, r))
          k_selfdot<T, C, V_><<<geo.nblk, nt, 0, s>>>(gr, geo, rd, h->st);
          coll<C>(h, EpiSqrtRedC{});
        } else {
          k_norm2<T, C, V_><<<geo.nblk, nt, 0, s>>>(gr, &h->st->red_c, geo, rd, h->st);
          coll<C>(h, EpiNorm2{&h->st->red_c});
        }
      });
      CKL();
      h->launches += 2;
      if (sync) read_state(h);
    };
    // one Arnoldi step's kernels: v_j = w_prev * inv, w = S v_j, the column h(., j)
    auto arnoldi = [&](int j, double inv, bool inv_dev, int slot, bool last) {  // last: no step follows in this cycle
      const T* wprev = j == 0 ? gr : (((j - 1) & 1) ? wB : wA);
      T* vj = V + (int64_t)j * ldv;
      T* w = (j & 1) ? wB : wA;
      V2([&](auto vt) {
        constexpr int V_ = decltype(vt)::v;
        if constexpr (SPARSE) {  // v_j = w / h as its own pass, then the gathered matvec
          k_scale<T, V_, FUSED_GS><<<geo.nblk, nt, 0, s>>>(wprev, vj, inv, geo);
          halo(h, vj);  // a row block's matvec reads v_j at the band beyond its rows
          auto kern = k_gm_matvec<Op, T, C, V_, false>;
          smem_attr(kern, win.bytes);
          kern<<<geo.nblk, nt, win.bytes, s>>>(o, nullptr, 0.0, vj, V, w, geo, rd, h->st, win.band);
          ++h->launches;
        } else {
          halo(h, wprev);
          if (!gmmatvec25(o, wprev, inv, vj, w, inv_dev))
            k_gm_matvec<Op, T, C, V_, true><<<geo.nblk, nt, 0, s>>>(o, wprev, inv, vj, V, w, geo, rd, h->st);
        }
        coll<C>(h, EpiHcol{0});
        if constexpr (FUSED_GS) {
          // accum = FP32: classical Gram-Schmidt in two passes (gadi_kernels.cuh)
          const int64_t ps = h->partm_stride;
          for (int i0 = 1; i0 <= j;) {
            const int left = j - i0 + 1, J = h->sharded() ? 1 : std::min(left, 4);
            if (J == 4) k_gm_dots<T, C, V_, 4><<<geo.nblk, nt, 0, s>>>(w, V, ldv, i0, geo, rd, h->d_partm, ps, h->st);
            else if (J == 3) k_gm_dots<T, C, V_, 3><<<geo.nblk, nt, 0, s>>>(w, V, ldv, i0, geo, rd, h->d_partm, ps, h->st);
            else if (J == 2) k_gm_dots<T, C, V_, 2><<<geo.nblk, nt, 0, s>>>(w, V, ldv, i0, geo, rd, h->d_partm, ps, h->st);
            else k_gm_dots<T, C, V_, 1><<<geo.nblk, nt, 0, s>>>(w, V, ldv, i0, geo, rd, h->d_partm, ps, h->st);
            if (J == 1) coll<C>(h, EpiHcol{i0});
            i0 += J;
            ++h->launches;
          }
          if constexpr (V_ > 1) {
            auto few = [&](auto nbt) {  // the last step of a cycle reduces the updated w without storing it
              constexpr int NB = decltype(nbt)::value;
              if (last) k_gm_cgs_few<T, C, V_, NB, false><<<geo.nblk, nt, 0, s>>>(w, V, ldv, geo, rd, h->st);
              else k_gm_cgs_few<T, C, V_, NB, true><<<geo.nblk, nt, 0, s>>>(w, V, ldv, geo, rd, h->st);
            };
            if (j == 0) few(std::integral_constant<int, 1>{});
            else if (j == 1) few(std::integral_constant<int, 2>{});
            else if (j == 2) few(std::integral_constant<int, 3>{});
            else if (j == 3) few(std::integral_constant<int, 4>{});
            else if (j == 4) few(std::integral_constant<int, 5>{});
            else if (j == 5) few(std::integral_constant<int, 6>{});
            else if (j == 6) few(std::integral_constant<int, 7>{});
            else k_gm_cgs<T, C, V_><<<geo.nblk, nt, 0, s>>>(w, V, ldv, j, geo, rd, h->st);
          } else {
            k_gm_cgs<T, C, V_><<<geo.nblk, nt, 0, s>>>(w, V, ldv, j, geo, rd, h->st);
          }
          coll<C>(h, EpiCgsNorm{j});
          if (slot >= 0) {
            k_gm_column_done<<<1, 1, 0, s>>>(h->st, j, slot);
            ++h->launches;
          }
          h->launches += 2;
        } else {
          for (int i = 0; i <= j; ++i) {
            T* vi = V + (int64_t)i * ldv;
            if (i < j) {
              k_gm_mgs<T, C, V_, false><<<geo.nblk, nt, 0, s>>>(w, vi, vi + ldv, i, geo, rd, h->st);
              coll<C>(h, EpiHcol{i + 1});
            } else {
              CK(cudaMemsetAsync(&h->st->maxbits, 0, 8, s));
              k_gm_mgs<T, C, V_, true><<<geo.nblk, nt, 0, s>>>(w, vi, nullptr, i, geo, rd, h->st);
              coll_flags(h, nullptr);  // max|w| over all ranks
            }
          }
          k_norm2<T, C, V_><<<geo.nblk, nt, 0, s>>>(w, &h->st->hcol[j + 1], geo, rd, h->st);
          coll<C>(h, EpiNorm2{&h->st->hcol[j + 1]});
          h->launches += j + 3;
        }
      });
      CKL();
    };
    while (total < spec.max_inner_iters) {
      // spec: the restart residual and the first window go out together
      int jq = 0, win0 = 0;  // steps queued so far in this cycle; first step of the current window
      auto queue_window = [&](int j0) {
        const int hi = std::min({m, j0 + GM_SPEC_MAX, j0 + (spec.max_inner_iters - total)});
        for (int jj = j0; jj < hi; ++jj)
          arnoldi(jj, 0.0, true, jj - j0, jj + 1 == m || total + (jj - j0) + 1 == spec.max_inner_iters);
        win0 = j0;
        jq = hi;
        read_state(h, 2);
      };
      resid(!spec_ok);
      if (spec_ok) queue_window(0);
      if (h->h_st->flags & 1) {
        status = INNER_OVERFLOW;
        break;
      }
      const double beta = h->h_st->red_c;
      if (std::sqrt(h->h_st->red_d) <= target) {
        status = INNER_CONVERGED;
        break;
      }
      if (beta == 0.0) break;
      std::fill(Hc.begin(), Hc.end(), 0.0);
      std::fill(cs.begin(), cs.end(), 0.0);
      std::fill(sn.begin(), sn.end(), 0.0);
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      int j = 0;
      bool happy = false;
      double inv = 1.0 / beta;  // v_0 = r / beta (scale with a binary64 factor)
      for (; j < m && total < spec.max_inner_iters; ++j, ++total) {
        const double* col = h->h_st->hcol;
        if (spec_ok) {
          if (j == jq) queue_window(j);
          col = h->h_st->hhist[j - win0];
        } else {
          arnoldi(j, inv, false, -1, j + 1 == m || total + 1 == spec.max_inner_iters);
          read_state(h, 1);
        }
        for (int i = 0; i <= j + 1; ++i) HC(i, j) = col[i];
        const double h1 = HC(j + 1, j);
        if (!std::isfinite(h1)) {
          status = INNER_OVERFLOW;
          goto done;
        }
        // v_{j+1} = w / h1 happens inside the next matvec (skipped if h1 == 0:
        // the loop then ends at this step, below).
        inv = h1 != 0.0 ? 1.0 / h1 : 0.0;
        for (int i = 0; i < j; ++i) {
          const double t1 = Rf(Rf(cs[i] * HC(i, j)) + Rf(sn[i] * HC(i + 1, j)));
          const double t2 = Rf(Rf(cs[i] * HC(i + 1, j)) - Rf(sn[i] * HC(i, j)));
          HC(i, j) = t1;
          HC(i + 1, j) = t2;
        }
        {
          const double a = HC(j, j), b = HC(j + 1, j);
          const double denom = Rf(std::hypot(a, b));
          if (denom == 0.0) {
            happy = true;
            ++j;
            ++total;
            break;
          }
          cs[j] = Rf(a / denom);
          sn[j] = Rf(b / denom);
          HC(j, j) = denom;
          HC(j + 1, j) = 0.0;
          const double gj = g[j];
          g[j] = Rf(cs[j] * gj);
          g[j + 1] = Rf(-sn[j] * gj);
          if (std::fabs(g[j + 1]) <= target || h1 == 0.0) {
            happy = true;
            ++j;
            ++total;
            break;
          }
        }
      }
      for (int i = j - 1; i >= 0; --i) {
        double acc = g[i];
        for (int k = i + 1; k < j; ++k) acc = Rf(acc - Rf(HC(i, k) * yv[k]));
        yv[i] = Rf(acc / HC(i, i));
      }
      if (j > 0) {
        for (int i = 0; i < j; ++i) h->h_st->ycoef[i] = yv[i];
        CK(cudaMemcpyAsync(h->st->ycoef, h->h_st->ycoef, j * sizeof(double), cudaMemcpyHostToDevice, s));
      }
      CK(cudaMemsetAsync(&h->st->flags, 0, 4, s));
      V2([&](auto vt) {
        constexpr int V_ = decltype(vt)::v;
        const int xz = x_zero ? 1 : 0;
        if constexpr (V_ > 1) {
          switch (j) {
            case 1: k_gm_update_few<T, C, V_, 1><<<geo.nblk, nt, 0, s>>>(x, xz, V, ldv, geo, h->st); break;
            case 2: k_gm_update_few<T, C, V_, 2><<<geo.nblk, nt, 0, s>>>(x, xz, V, ldv, geo, h->st); break;
            case 3: k_gm_update_few<T, C, V_, 3><<<geo.nblk, nt, 0, s>>>(x, xz, V, ldv, geo, h->st); break;
            case 4: k_gm_update_few<T, C, V_, 4><<<geo.nblk, nt, 0, s>>>(x, xz, V, ldv, geo, h->st); break;
            case 5: k_gm_update_few<T, C, V_, 5><<<geo.nblk, nt, 0, s>>>(x, xz, V, ldv, geo, h->st); break;
            case 6: k_gm_update_few<T, C, V_, 6><<<geo.nblk, nt, 0, s>>>(x, xz, V, ldv, geo, h->st); break;
            case 7: k_gm_update_few<T, C, V_, 7><<<geo.nblk, nt, 0, s>>>(x, xz, V, ldv, geo, h->st); break;
            default: k_gm_update<T, C, V_><<<geo.nblk, nt, 0, s>>>(x, xz, V, ldv, j, geo, h->st);
          }
        } else {
          k_gm_update<T, C, V_><<<geo.nblk, nt, 0, s>>>(x, xz, V, ldv, j, geo, h->st);
        }
      });
      CKL();
      ++h->launches;
      coll_flags(h, &h->st->flags);
      x_zero = false;
      read_state(h);
      if (h->h_st->flags & 1) {
        status = INNER_OVERFLOW;
        break;
      }
      if (happy) {
        resid();
        if (std::sqrt(h->h_st->red_d) <= target) {
          status = INNER_CONVERGED;
          break;
        }
      }
    }
  done:
    if (x_zero) CK(cudaMemsetAsync(x, 0, N * sizeof(T), s));
    // all_finite(x) (inner_solver.cpp:192): every update of x was checked above
    if (status < 0) status = INNER_STAGNATED;
    InnerOut out;
    out.iters = total;
    out.status = status;
    return out;
  }

  // ----------------------------------------------------------- outer pieces
  // Outer elementwise passes: 8-element segments (4 x 128-bit binary64
  // accesses per lane) where the shape allows -- the same pairwise tree,
  // a quarter of the per-segment warp-tree work of 2-element segments.
  int outer_vec() const {
    return aligned_for(h->N, h->n, h->stencil(), 8) ? 8 : aligned_for(h->N, h->n, h->stencil(), 2) ? 2 : 1;
  }
  void scale_round(const double* sv, int ns_r) override {
    const Red rd = red_of(h);
    const int ov = outer_vec();
    const Geo g = make_geo(h->N, ov);
    const double nr = nsc_of(ns_r);
    T* rh = static_cast<T*>(rhat);
    if (ov == 8) k_scale_round<T, 8><<<g.nblk, g.threads(), 0, h->stream>>>(sv, rh, g, rd, h->st, nr);
    else if (ov == 2) k_scale_round<T, 2><<<g.nblk, g.threads(), 0, h->stream>>>(sv, rh, g, rd, h->st, nr);
    else k_scale_round<T, 1><<<g.nblk, g.threads(), 0, h->stream>>>(sv, rh, g, rd, h->st, nr);
    CKL();
    ++h->launches;
    coll<double>(h, EpiRhat{});
  }
  bool resid_spec(const double* x, int ep, bool scaling) override {
    if constexpr (SPARSE) {
      return false;
    } else {
      St25Geo gs;
      // k_resid64 where the shape fits; else k_st25 on 2048-chunk tiles, 16 warps x 4 chunks
      const double c7[7] = {h->t2, h->t2, h->t2, h->t1, h->t3, h->t3, h->t3};
      const bool fits64 = r64_fits(h->n, h->i0, h->i1, c7, gs);
      if (!fits64 && !make_st25(h->n, 8, 1, gs, 2048, true, 0, h->i0, h->i1, 4, 512) &&
          !make_st25(h->n, 8, 1, gs, 1024, true, 0, h->i0, h->i1))
        return false;
      CK(cudaMemsetAsync(&h->st->maxbits, 0, sizeof(unsigned long long), h->stream));
      halo(h, x);
      const int64_t eo = h->e_off();
      PolResidSpec<T> pol{{h->t2, h->t2, h->t2, h->t1, h->t3, h->t3, h->t3},
                          x - eo,
                          h->d_b - eo,
                          static_cast<T*>(rhat) - eo,
                          ep,
                          (ep >= -1000 && ep <= 1000) ? std::ldexp(1.0, -ep) : 1.0,
                          scaling ? 1 : 0,
                          nsc_of(h->ns),
                          nsc_of(scaling ? 0 : h->ns)};
      if (fits64) launch_resid64(pol, gs, h->stream, red_of(h), h->st);
      else launch_st25(pol, gs, h->stream, red_of(h), h->st);
      CKL();
      ++h->launches;
      coll<double>(h, EpiResidSpec{scaling ? 1 : 0});
      return true;
    }
  }
  void scale_pz(double phat) override {
    V2([&](auto vt) {
      constexpr int V_ = decltype(vt)::v;
      k_scale<T, V_><<<geo.nblk, geo.threads(), 0, h->stream>>>(static_cast<T*>(z), static_cast<T*>(pz), phat, geo);
    });
    CKL();
    ++h->launches;
  }
  void update(double* x, int pu) override {
    const int ov = std::min(outer_vec(), 2);  // no reduction here: 2-element segments stream best (measured)
    const Geo g = make_geo(h->N, ov);
    auto L = [&](auto pt, auto vt) {
      constexpr int PU = decltype(pt)::v, V_ = decltype(vt)::v;
      k_update<T, PU, V_><<<g.nblk, g.threads(), 0, h->stream>>>(x, static_cast<const T*>(y), g, h->st);
    };
    auto LV = [&](auto pt) {
      if (ov == 2) L(pt, VecTag<2>{});
      else L(pt, VecTag<1>{});
    };
    if (pu == GADI_HALF) LV(VecTag<P_HALF>{});
    else if (pu == GADI_SINGLE) LV(VecTag<P_SINGLE>{});
    else LV(VecTag<P_DOUBLE>{});
    CKL();
    ++h->launches;
    coll_flags(h, &h->st->xbad);
  }
  void to_inner(const double* src, void* dst) override {
    constexpr int PT = prec_of<T>();
    k_convert<double, T, PT><<<ew_grid(h->N), 256, 0, h->stream>>>(src, static_cast<T*>(dst), h->N);
    CKL();
    ++h->launches;
  }
  void to_double(const void* src, double* dst) override {
    k_convert<T, double, P_DOUBLE><<<ew_grid(h->N), 256, 0, h->stream>>>(static_cast<const T*>(src), dst, h->N);
    CKL();
    ++h->launches;
  }
  void apply(int which, const void* xv, void* yv_) override {
    k_apply<Op, T, C, T><<<ew_grid(h->N), 256, 0, h->stream>>>(op(which), static_cast<const T*>(xv),
                                                               static_cast<T*>(yv_), h->N, MatvecF<C, T>());
    CKL();
    ++h->launches;
  }
};

// One translation unit per (operator, storage, arithmetic) instantiates each
// engine (gadi_engine_*.cu) so the build compiles them in parallel.
#define GADI_ENGINE_FACTORY(name) \
  EngineBase* name(gadi_handle* h, const gadi_inner_spec& sp, double a, double om, int ur, int acc)
GADI_ENGINE_FACTORY(make_engine_st_d64);
GADI_ENGINE_FACTORY(make_engine_st_f32);
GADI_ENGINE_FACTORY(make_engine_st_h16);
GADI_ENGINE_FACTORY(make_engine_st_h32);
GADI_ENGINE_FACTORY(make_engine_csr_d64);
GADI_ENGINE_FACTORY(make_engine_csr_f32);
GADI_ENGINE_FACTORY(make_engine_csr_h16);
GADI_ENGINE_FACTORY(make_engine_csr_h32);

}  // namespace gadi_host
