// Stencil pass design exploration (not product code): times candidate
// structures of the fused CG pass p = r + beta p, q = H p, p.q on an n^3 grid
// in binary16 storage / binary32 arithmetic against a plain streaming copy.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/stmb tools/st_microbench.cu && /tmp/stmb 512
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <type_traits>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ float fhfma(__half a, __half b, float c) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(__half_as_ushort(a)), "h"(__half_as_ushort(b)), "f"(c));
  return d;
}
struct H8 { __half v[8]; };
__device__ __forceinline__ void pf_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ H8 ldh8(const __half* p) { uint4 u = __ldg(reinterpret_cast<const uint4*>(p)); return *reinterpret_cast<H8*>(&u); }
__device__ __forceinline__ H8 ldh8cs(const __half* p) { uint4 u = __ldcs(reinterpret_cast<const uint4*>(p)); return *reinterpret_cast<H8*>(&u); }
__device__ __forceinline__ void sth8(__half* p, const H8& h) { *reinterpret_cast<uint4*>(p) = *reinterpret_cast<const uint4*>(&h); }

__device__ __forceinline__ H8 pupd(const H8& r, const H8& p, float beta) {
  H8 o;
#pragma unroll
  for (int e = 0; e < 8; ++e) o.v[e] = __float2half_rn(__fadd_rn(__half2float(r.v[e]), __fmul_rn(beta, __half2float(p.v[e]))));
  return o;
}

__global__ void k_copy(const uint4* a, const uint4* b, uint4* c, uint4* d, long n16) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n16; i += (long)gridDim.x * blockDim.x) {
    uint4 x = __ldcs(a + i), y = __ldcs(b + i);
    c[i] = x; d[i] = y;
  }
}

// V1: register marching along i, j-neighbours recomputed from r, p (L1/L2), k-edges by shuffles.
// CTA = 8 warps = 4 rows x 512 points (n = 512: 64 chunks per row, 2 warps per row).
template <int IL, int PF>
__global__ void __launch_bounds__(256) k_v1(const __half* __restrict__ r, const __half* __restrict__ p, __half* __restrict__ pn,
                                            __half* __restrict__ q, float beta, __half c0, __half c1, __half c2, __half c3,
                                            __half c4, __half c5, __half c6, int n, double* part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rows = blockDim.x / (n / 8);
  const int ngj = n / rows;
  const int jg = blockIdx.x % ngj, ic = blockIdx.x / ngj;
  const int c = threadIdx.x;  // chunk in tile
  const int jl = c / (n / 8), k0 = (c % (n / 8)) * 8;
  const int j = jg * rows + jl;
  const long nn = (long)n * n;
  const int ib = ic * IL, ie = ib + IL;
  auto at = [&](int i, int jj) -> long { return (long)i * nn + (long)jj * n + k0; };
  auto mk = [&](int i, int jj) -> H8 { long e = at(i, jj); return pupd(ldh8(r + e), ldh8(p + e), beta); };
  H8 zero; for (int e = 0; e < 8; ++e) zero.v[e] = __float2half_rn(0.f);
  H8 prv = ib > 0 ? mk(ib - 1, j) : zero;
  H8 cur = mk(ib, j);
  // prefetch raw of plane ib+1
  H8 rn = ldh8(r + at(ib + 1 < n ? ib + 1 : ib, j)), pnx = ldh8(p + at(ib + 1 < n ? ib + 1 : ib, j));
  float dsum = 0.f;
  const long tile = (long)jg * rows * n;
  if (PF > 0 && threadIdx.x == 0)
    for (int d = 2; d < 2 + PF && ib + d < n; ++d) { pf_l2(r + (ib + d) * nn + tile, rows * n * 2); pf_l2(p + (ib + d) * nn + tile, rows * n * 2); }
  for (int i = ib; i < ie; ++i) {
    if (PF > 0 && threadIdx.x == 0 && i + 2 + PF < n && i + 2 + PF <= ie) { pf_l2(r + (i + 2 + PF) * nn + tile, rows * n * 2); pf_l2(p + (i + 2 + PF) * nn + tile, rows * n * 2); }
    H8 nxt = pupd(rn, pnx, beta);
    if (i + 2 < n) { rn = ldh8(r + at(i + 2, j)); pnx = ldh8(p + at(i + 2, j)); }
    H8 jm = j > 0 ? mk(i, j - 1) : zero;
    H8 jp = j < n - 1 ? mk(i, j + 1) : zero;
    // k edges
    __half left = __shfl_up_sync(0xffffffffu, cur.v[7], 1);
    __half right = __shfl_down_sync(0xffffffffu, cur.v[0], 1);
    if (lane == 0 && k0 > 0) { long e = at(i, j) - 1; left = __float2half_rn(__fadd_rn(__half2float(r[e]), __fmul_rn(beta, __half2float(p[e])))); }
    if (lane == 31 && k0 + 8 < n) { long e = at(i, j) + 8; right = __float2half_rn(__fadd_rn(__half2float(r[e]), __fmul_rn(beta, __half2float(p[e])))); }
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float a = 0.f;
      if (i > 0) a = fhfma(c0, prv.v[e], a);
      if (j > 0) a = fhfma(c1, jm.v[e], a);
      __half km = e > 0 ? cur.v[e - 1] : left;
      if (e > 0 || k0 > 0) a = fhfma(c2, km, a);
      a = fhfma(c3, cur.v[e], a);
      __half kp = e < 7 ? cur.v[e + 1] : right;
      if (e < 7 || k0 + 8 < n) a = fhfma(c4, kp, a);
      if (j < n - 1) a = fhfma(c5, jp.v[e], a);
      if (i < n - 1) a = fhfma(c6, nxt.v[e], a);
      acc[e] = a;
    }
    H8 qv;
#pragma unroll
    for (int e = 0; e < 8; ++e) qv.v[e] = __float2half_rn(acc[e]);
    sth8(q + at(i, j), qv);
    sth8(pn + at(i, j), cur);
    float t[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) t[e] = fhfma(cur.v[e], qv.v[e], -0.f);
#pragma unroll
    for (int s = 1; s < 8; s <<= 1)
#pragma unroll
      for (int e = 0; e < 8; e += 2 * s) t[e] = __fadd_rn(t[e], t[e + s]);
    float w = t[0];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) w = __fadd_rn(w, __shfl_xor_sync(0xffffffffu, w, o));
    dsum = __fadd_rn(dsum, w);
    prv = cur;
    cur = nxt;
  }
  if (lane == 0) part[(long)blockIdx.x * 8 + warp] = dsum;
}

// V2a: plain p-update pass (streaming).
__global__ void k_pupd(const __half* __restrict__ r, const __half* __restrict__ p, __half* __restrict__ pn, float beta, long n8) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n8; i += (long)gridDim.x * blockDim.x) {
    H8 a = ldh8cs(r + i * 8), b = ldh8cs(p + i * 8);
    sth8(pn + i * 8, pupd(a, b, beta));
  }
}
// V2b: plain SpMV + dot, register marching, neighbours straight from global.
template <int IL, int PF>
__global__ void __launch_bounds__(256) k_v2(const __half* __restrict__ x, __half* __restrict__ q, __half c0, __half c1,
                                            __half c2, __half c3, __half c4, __half c5, __half c6, int n, double* part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rows = blockDim.x / (n / 8);
  const int ngj = n / rows;
  const int jg = blockIdx.x % ngj, ic = blockIdx.x / ngj;
  const int c = threadIdx.x;
  const int jl = c / (n / 8), k0 = (c % (n / 8)) * 8;
  const int j = jg * rows + jl;
  const long nn = (long)n * n;
  const int ib = ic * IL, ie = ib + IL;
  auto at = [&](int i, int jj) -> long { return (long)i * nn + (long)jj * n + k0; };
  H8 zero; for (int e = 0; e < 8; ++e) zero.v[e] = __float2half_rn(0.f);
  H8 prv = ib > 0 ? ldh8(x + at(ib - 1, j)) : zero;
  H8 cur = ldh8(x + at(ib, j));
  H8 nxt = ldh8(x + at(ib + 1 < n ? ib + 1 : ib, j));
  float dsum = 0.f;
  const long tile = (long)jg * rows * n;
  if (PF > 0 && threadIdx.x == 0)
    for (int d = 2; d < 2 + PF && ib + d < n; ++d) pf_l2(x + (ib + d) * nn + tile, rows * n * 2);
  for (int i = ib; i < ie; ++i) {
    if (PF > 0 && threadIdx.x == 0 && i + 2 + PF < n && i + 2 + PF <= ie) pf_l2(x + (i + 2 + PF) * nn + tile, rows * n * 2);
    H8 nn2 = i + 2 < n ? ldh8(x + at(i + 2, j)) : zero;
    H8 jm = j > 0 ? ldh8(x + at(i, j - 1)) : zero;
    H8 jp = j < n - 1 ? ldh8(x + at(i, j + 1)) : zero;
    __half left = __shfl_up_sync(0xffffffffu, cur.v[7], 1);
    __half right = __shfl_down_sync(0xffffffffu, cur.v[0], 1);
    if (lane == 0 && k0 > 0) left = x[at(i, j) - 1];
    if (lane == 31 && k0 + 8 < n) right = x[at(i, j) + 8];
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float a = 0.f;
      if (i > 0) a = fhfma(c0, prv.v[e], a);
      if (j > 0) a = fhfma(c1, jm.v[e], a);
      __half km = e > 0 ? cur.v[e - 1] : left;
      if (e > 0 || k0 > 0) a = fhfma(c2, km, a);
      a = fhfma(c3, cur.v[e], a);
      __half kp = e < 7 ? cur.v[e + 1] : right;
      if (e < 7 || k0 + 8 < n) a = fhfma(c4, kp, a);
      if (j < n - 1) a = fhfma(c5, jp.v[e], a);
      if (i < n - 1) a = fhfma(c6, nxt.v[e], a);
      acc[e] = a;
    }
    H8 qv;
#pragma unroll
    for (int e = 0; e < 8; ++e) qv.v[e] = __float2half_rn(acc[e]);
    sth8(q + at(i, j), qv);
    float t[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) t[e] = fhfma(cur.v[e], qv.v[e], -0.f);
#pragma unroll
    for (int s = 1; s < 8; s <<= 1)
#pragma unroll
      for (int e = 0; e < 8; e += 2 * s) t[e] = __fadd_rn(t[e], t[e + s]);
    float w = t[0];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) w = __fadd_rn(w, __shfl_xor_sync(0xffffffffu, w, o));
    dsum = __fadd_rn(dsum, w);
    prv = cur;
    cur = nxt;
    nxt = nn2;
  }
  if (lane == 0) part[(long)blockIdx.x * 8 + warp] = dsum;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 512;
  const long N = (long)n * n * n;
  __half *r, *p, *pn, *q;
  CK(cudaMalloc(&r, N * 2)); CK(cudaMalloc(&p, N * 2)); CK(cudaMalloc(&pn, N * 2)); CK(cudaMalloc(&q, N * 2));
  CK(cudaMemset(r, 0x3c, N * 2)); CK(cudaMemset(p, 0x3a, N * 2));
  double* part; CK(cudaMalloc(&part, (N / 8 + 1024) * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const __half c0 = __float2half(-1.f), c3 = __float2half(6.2f), c6 = __float2half(-0.95f);
  auto time = [&](const char* name, double bytes, auto&& f) {
    for (int w = 0; w < 3; ++w) f();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    const int R = 20;
    for (int k = 0; k < R; ++k) f();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / R;
    printf("%-34s %8.1f us  %7.0f GB/s (algorithmic %.3f GB)\n", name, us, bytes / us * 1e-3, bytes * 1e-9);
  };
  const double V = N * 2.0;
  time("copy 2 in 2 out", 4 * V, [&] { k_copy<<<148 * 16, 256>>>((uint4*)r, (uint4*)p, (uint4*)pn, (uint4*)q, N / 8); });
  time("pupd (r,p -> pn)", 3 * V, [&] { k_pupd<<<148 * 16, 256>>>(r, p, pn, 0.5f, N / 8); });
  const int rows = 256 / (n / 8);
  auto run = [&](auto ilc, auto pfc) {
    constexpr int IL = decltype(ilc)::value, PF = decltype(pfc)::value;
    const int grid = (n / rows) * (n / IL);
    char nm[64];
    snprintf(nm, 64, "v1 fused recompute IL=%d PF=%d", IL, PF);
    time(nm, 4 * V, [&] { k_v1<IL, PF><<<grid, 256>>>(r, p, pn, q, 0.5f, c0, c0, c0, c3, c6, c6, c6, n, part); });
    snprintf(nm, 64, "v2 spmv only IL=%d PF=%d", IL, PF);
    time(nm, 2 * V, [&] { k_v2<IL, PF><<<grid, 256>>>(pn, q, c0, c0, c0, c3, c6, c6, c6, n, part); });
  };
  using namespace std;
  run(integral_constant<int, 16>{}, integral_constant<int, 0>{});
  run(integral_constant<int, 16>{}, integral_constant<int, 2>{});
  run(integral_constant<int, 16>{}, integral_constant<int, 4>{});
  run(integral_constant<int, 16>{}, integral_constant<int, 8>{});
  run(integral_constant<int, 32>{}, integral_constant<int, 4>{});
  run(integral_constant<int, 32>{}, integral_constant<int, 8>{});
  run(integral_constant<int, 64>{}, integral_constant<int, 8>{});
  return 0;
}
