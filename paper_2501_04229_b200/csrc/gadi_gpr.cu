// gadi_gpr.cu — the GPR alpha predictor on the device (gpr.hpp:60-87;
// fit gpr.cpp:109-149 with try_fit :84-105, predict_alpha :151-169).
//
// Inputs are ln(size) (gpr.cpp:114), targets centred on their mean, the
// squared-exponential Gram matrix K_ij = sf2 exp(-(x_i - x_j)^2 / (2 l^2))
// plus (sn2 + 1e-12 max(1, sf2)) on the diagonal, all in binary64. fit()
// either searches the reference's 27-point grid (sf2 in {1/4,1,4} var,
// l in {1/2,1,2} spacing, sn2 in {1e-10,1e-8,1e-6} var; strict '>' keeps the
// first maximum of the log marginal likelihood) or takes fixed (sf2, l, sn2)
// (BASELINE configs[4]: l = 1, sn2 = 1e-4). The Gram matrix is built by a
// device kernel and factored by cuSOLVER's Dpotrf (a plain library
// factorization); predictions build K_* on the device, the mean is a fused
// kernel-vector pass and the variance sf2 + sn2 - ||L^-1 k_*||^2 is one
// cuBLAS Dtrsm over a block of queries followed by a fused column-norm pass.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gadi_cuda.h"

namespace gadi_host {
void set_last_error(const std::string& m);  // gadi_api.cu: shared by gadi_last_error()
}

namespace {

struct GErr : std::runtime_error {
  int code;
  GErr(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define GCK(x)                                                                            \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) throw GErr(GADI_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define BCK(x)                                                                     \
  do {                                                                             \
    if ((x) != CUBLAS_STATUS_SUCCESS) throw GErr(GADI_E_CUDA, std::string(#x));    \
  } while (0)
#define SCK(x)                                                                     \
  do {                                                                             \
    if ((x) != CUSOLVER_STATUS_SUCCESS) throw GErr(GADI_E_CUDA, std::string(#x));  \
  } while (0)

// K (column major, m x m) = sf2 * exp(-0.5 d^2), d = (x_i - x_j) / l (gpr.cpp:70-73),
// diagonal += sn2 + 1e-12 * max(1, sf2) (gpr.cpp:88)
__global__ void k_gram(const double* __restrict__ x, int m, double sf2, double ell, double jitter,
                       double* __restrict__ K) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)m * m) return;
  const int i = (int)(idx % m), j = (int)(idx / m);
  const double d = __ddiv_rn(__dsub_rn(x[i], x[j]), ell);
  double v = __dmul_rn(sf2, exp(__dmul_rn(-0.5, __dmul_rn(d, d))));
  if (i == j) v = __dadd_rn(v, jitter);
  K[idx] = v;
}

// K_*^T block (m x qb, column major): k(x_i, xq_t)
__global__ void k_cross(const double* __restrict__ x, int m, const double* __restrict__ xq, int qb, double sf2,
                        double ell, double* __restrict__ Ks) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)m * qb) return;
  const int i = (int)(idx % m), t = (int)(idx / m);
  const double d = __ddiv_rn(__dsub_rn(xq[t], x[i]), ell);
  Ks[idx] = __dmul_rn(sf2, exp(__dmul_rn(-0.5, __dmul_rn(d, d))));
}

// per query column t: mean = mu + k.a, and ||v||^2 of the solved column (one warp each)
__global__ void k_pred_cols(const double* __restrict__ Ks, const double* __restrict__ V, const double* __restrict__ a,
                            int m, int qb, double mu, double sfsn, double floor_mean, double* __restrict__ mean,
                            double* __restrict__ sd) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= qb) return;
  double kd = 0.0, vn = 0.0;
  for (int i = lane; i < m; i += 32) {
    kd = fma(Ks[(int64_t)t * m + i], a[i], kd);
    const double v = V[(int64_t)t * m + i];
    vn = fma(v, v, vn);
  }
  for (int o = 16; o > 0; o >>= 1) {
    kd += __shfl_xor_sync(0xffffffffu, kd, o);
    vn += __shfl_xor_sync(0xffffffffu, vn, o);
  }
  if (lane == 0) {
    double mn = mu + kd;
    double var = sfsn - vn;
    if (var < 0.0) var = 0.0;
    if (mn < floor_mean) mn = floor_mean;
    mean[t] = mn;
    sd[t] = sqrt(var);
  }
}

__global__ void k_logdiag(const double* __restrict__ L, int m, double* __restrict__ out) {
  __shared__ double sm[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) s += log(L[(int64_t)i * m + i]);
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

template <class T>
T* galloc(size_t n) {
  void* p = nullptr;
  GCK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

}  // namespace

struct gadi_gpr {
  int device = 0, m = 0;
  cudaStream_t s = nullptr;
  cublasHandle_t cb = nullptr;
  cusolverDnHandle_t cs = nullptr;
  double mu = 0, sf2 = 1, ell = 1, sn2 = 1e-8, lml = 0, tmin = 0;
  double* d_x = nullptr;  // ln(size)
  double* d_L = nullptr;  // lower Cholesky factor of K (column major)
  double* d_a = nullptr;  // K^-1 (y - mu)
  double fit_ms = 0.0;
  ~gadi_gpr() {
    for (void* p : {(void*)d_x, (void*)d_L, (void*)d_a})
      if (p) cudaFree(p);
    if (cb) cublasDestroy(cb);
    if (cs) cusolverDnDestroy(cs);
    if (s) cudaStreamDestroy(s);
  }
};

namespace {

// try_fit (gpr.cpp:84-105) for one hyperparameter triple; false when K is
// not positive definite after jitter or the LML is not finite.
bool try_fit(gadi_gpr* g, const std::vector<double>& y, double sf2, double ell, double sn2, double* d_K,
             double* d_work, int lwork, int* d_info, double* d_tmp, double& lml) {
  const int m = g->m;
  const double jitter = sn2 + 1e-12 * std::max(1.0, sf2);
  const int64_t mm = (int64_t)m * m;
  k_gram<<<(unsigned)((mm + 255) / 256), 256, 0, g->s>>>(g->d_x, m, sf2, ell, jitter, d_K);
  GCK(cudaGetLastError());
  SCK(cusolverDnDpotrf(g->cs, CUBLAS_FILL_MODE_LOWER, m, d_K, m, d_work, lwork, d_info));
  int info = 0;
  GCK(cudaMemcpyAsync(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost, g->s));
  GCK(cudaStreamSynchronize(g->s));
  if (info != 0) return false;
  GCK(cudaMemcpyAsync(d_tmp, y.data(), m * sizeof(double), cudaMemcpyHostToDevice, g->s));
  SCK(cusolverDnDpotrs(g->cs, CUBLAS_FILL_MODE_LOWER, m, 1, d_K, m, d_tmp, m, d_info));
  k_logdiag<<<1, 256, 0, g->s>>>(d_K, m, d_tmp + m);
  std::vector<double> a(m + 1);
  GCK(cudaMemcpyAsync(a.data(), d_tmp, (m + 1) * sizeof(double), cudaMemcpyDeviceToHost, g->s));
  GCK(cudaStreamSynchronize(g->s));
  double ya = 0.0;
  for (int i = 0; i < m; ++i) ya += y[i] * a[i];
  lml = -0.5 * ya - a[m] - 0.5 * (double)m * std::log(2.0 * M_PI);
  return std::isfinite(lml);
}

}  // namespace

extern "C" {

int gadi_gpr_fit(const double* sizes, const double* alphas, int32_t m, const gadi_gpr_opts* opts, gadi_gpr** out) {
  try {
    if (!sizes || !alphas || !out) throw GErr(GADI_E_CONTRACT, "gpr_fit: null argument");
    *out = nullptr;
    if (m < 3) throw GErr(GADI_E_FIT, "fit: at least 3 training pairs required");  // gpr.cpp:110
    std::unique_ptr<gadi_gpr> g(new gadi_gpr());
    g->device = opts ? opts->device : 0;
    GCK(cudaSetDevice(g->device));
    g->m = m;
    std::vector<double> x(m), y(m);
    double mu = 0.0, tmin = std::numeric_limits<double>::infinity();
    for (int i = 0; i < m; ++i) {
      if (!(alphas[i] > 0.0)) throw GErr(GADI_E_FIT, "fit: alpha targets must be positive");
      if (!(sizes[i] > 0.0)) throw GErr(GADI_E_CONTRACT, "fit: sizes must be positive");
      x[i] = std::log(sizes[i]);
      mu += alphas[i];
      tmin = std::min(tmin, alphas[i]);
    }
    mu /= (double)m;
    double var = 0.0;
    for (int i = 0; i < m; ++i) {
      y[i] = alphas[i] - mu;
      var += y[i] * y[i];
    }
    var = std::max(var / (double)m, 1e-8);
    const double spacing = std::max((x[m - 1] - x[0]) / (double)(m - 1), 1e-3);
    g->mu = mu;
    g->tmin = tmin;
    GCK(cudaStreamCreateWithFlags(&g->s, cudaStreamNonBlocking));
    BCK(cublasCreate(&g->cb));
    BCK(cublasSetStream(g->cb, g->s));
    SCK(cusolverDnCreate(&g->cs));
    SCK(cusolverDnSetStream(g->cs, g->s));
    cudaEvent_t e0, e1;
    GCK(cudaEventCreate(&e0));
    GCK(cudaEventCreate(&e1));
    GCK(cudaEventRecord(e0, g->s));
    g->d_x = galloc<double>(m);
    GCK(cudaMemcpyAsync(g->d_x, x.data(), m * sizeof(double), cudaMemcpyHostToDevice, g->s));
    double* d_K = galloc<double>((size_t)m * m);
    g->d_L = galloc<double>((size_t)m * m);
    g->d_a = galloc<double>(m);
    double* d_tmp = galloc<double>(m + 1);
    int* d_info = galloc<int>(1);
    int lwork = 0;
    SCK(cusolverDnDpotrf_bufferSize(g->cs, CUBLAS_FILL_MODE_LOWER, m, d_K, m, &lwork));
    double* d_work = galloc<double>(lwork);
    std::vector<double> sfs, ells, sns;
    if (opts && opts->fixed_hypers) {
      sfs = {opts->sigma_f2};
      ells = {opts->length};
      sns = {opts->sigma_n2};
    } else {  // gpr.cpp:128-137
      sfs = {0.25 * var, 1.0 * var, 4.0 * var};
      ells = {0.5 * spacing, 1.0 * spacing, 2.0 * spacing};
      if (opts && opts->has_sigma_n2) sns = {opts->sigma_n2};
      else sns = {1e-10 * var, 1e-8 * var, 1e-6 * var};
    }
    double best = -std::numeric_limits<double>::infinity();
    for (double sf : sfs)
      for (double el : ells)
        for (double sn : sns) {
          double lml = 0.0;
          if (try_fit(g.get(), y, sf, el, sn, d_K, d_work, lwork, d_info, d_tmp, lml) && lml > best) {
            best = lml;
            g->sf2 = sf;
            g->ell = el;
            g->sn2 = sn;
            GCK(cudaMemcpyAsync(g->d_L, d_K, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToDevice, g->s));
            GCK(cudaMemcpyAsync(g->d_a, d_tmp, m * sizeof(double), cudaMemcpyDeviceToDevice, g->s));
          }
        }
    GCK(cudaEventRecord(e1, g->s));
    GCK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    g->fit_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (void* p : {(void*)d_K, (void*)d_tmp, (void*)d_info, (void*)d_work}) cudaFree(p);
    if (!std::isfinite(best)) throw GErr(GADI_E_FIT, "fit: Gram matrix not positive definite for any hyperparameter choice");
    g->lml = best;
    *out = g.release();
    return GADI_OK;
  } catch (const GErr& e) {
    gadi_host::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    gadi_host::set_last_error(e.what());
    return GADI_E_CUDA;
  }
}

int gadi_gpr_predict(gadi_gpr* g, const double* sizes, int32_t q, double* mean, double* stddev) {
  try {
    if (!g || (!sizes && q > 0) || (q > 0 && (!mean || !stddev))) throw GErr(GADI_E_CONTRACT, "gpr_predict: bad argument");
    GCK(cudaSetDevice(g->device));
    const int m = g->m;
    const int QB = 8192;  // queries per block of the triangular solve
    std::vector<double> xq(std::min(q, QB));
    double* d_xq = galloc<double>(QB);
    double* d_Ks = galloc<double>((size_t)m * QB);
    double* d_V = galloc<double>((size_t)m * QB);
    double* d_mean = galloc<double>(QB);
    double* d_sd = galloc<double>(QB);
    const double one = 1.0;
    for (int t0 = 0; t0 < q; t0 += QB) {
      const int qb = std::min(QB, q - t0);
      xq.resize(qb);
      for (int t = 0; t < qb; ++t) xq[t] = std::log(sizes[t0 + t]);
      GCK(cudaMemcpyAsync(d_xq, xq.data(), qb * sizeof(double), cudaMemcpyHostToDevice, g->s));
      const int64_t n = (int64_t)m * qb;
      k_cross<<<(unsigned)((n + 255) / 256), 256, 0, g->s>>>(g->d_x, m, d_xq, qb, g->sf2, g->ell, d_Ks);
      GCK(cudaGetLastError());
      GCK(cudaMemcpyAsync(d_V, d_Ks, n * sizeof(double), cudaMemcpyDeviceToDevice, g->s));
      // v = L^-1 k_* for every query of the block (predict_alpha, gpr.cpp:159-161)
      BCK(cublasDtrsm(g->cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, m, qb, &one,
                      g->d_L, m, d_V, m));
      k_pred_cols<<<(qb + 7) / 8, 256, 0, g->s>>>(d_Ks, d_V, g->d_a, m, qb, g->mu, g->sf2 + g->sn2, g->tmin / 10.0,
                                                   d_mean, d_sd);
      GCK(cudaGetLastError());
      GCK(cudaMemcpyAsync(mean + t0, d_mean, qb * sizeof(double), cudaMemcpyDeviceToHost, g->s));
      GCK(cudaMemcpyAsync(stddev + t0, d_sd, qb * sizeof(double), cudaMemcpyDeviceToHost, g->s));
    }
    GCK(cudaStreamSynchronize(g->s));
    for (void* p : {(void*)d_xq, (void*)d_Ks, (void*)d_V, (void*)d_mean, (void*)d_sd}) cudaFree(p);
    return GADI_OK;
  } catch (const GErr& e) {
    gadi_host::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    gadi_host::set_last_error(e.what());
    return GADI_E_CUDA;
  }
}

int gadi_gpr_params(const gadi_gpr* g, double* sigma_f2, double* length, double* sigma_n2, double* lml,
                    double* target_mean) {
  if (!g) return GADI_E_CONTRACT;
  if (sigma_f2) *sigma_f2 = g->sf2;
  if (length) *length = g->ell;
  if (sigma_n2) *sigma_n2 = g->sn2;
  if (lml) *lml = g->lml;
  if (target_mean) *target_mean = g->mu;
  return GADI_OK;
}

int gadi_gpr_destroy(gadi_gpr* g) {
  if (g) {
    cudaSetDevice(g->device);
    delete g;
  }
  return GADI_OK;
}

}  // extern "C"
