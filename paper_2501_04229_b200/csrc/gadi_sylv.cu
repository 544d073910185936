// gadi_sylv.cu — the Sylvester GADI-AB system on the device: the reference's
// second GadiSystem, SylvesterOperator (sylvester.cpp:9-120), and
// gadi_ab_solve (sylvester.cpp:122-133) driving run_gadi_ir
// (solver.cpp:57-179) over it.
//
// A X + X B = G with X m x n stored column-major (vec, dense.cpp:68-73),
// binary64 outer vectors. Per outer step:
//   residual_uf   one thread per entry folds G - A X - X B in the reference's
//                 order (A's row i, then B^T's row j), each op rounded to u_f;
//   true norm     G - (A X + X B) with the plain binary64 accumulations of
//                 apply (sylvester.cpp:20-39), then norm2_64 sequentially
//                 (exactly the reference's sum; the systems are small);
//   solve_H       (alpha I + A) Z = R column by column, solve_S
//                 (alpha I + B^T) row by row (sylvester.cpp:83-119): one
//                 thread per column / row runs BandLU's solve against the
//                 device factor (gadi_lu.cu), which prepare builds in u_r
//                 (the inner spec is ignored, as in the reference).
// Every value is the reference's bit for bit.
#include "gadi_host.cuh"

using namespace gadi_host;

struct gadi_sylv {
  int device = 0;
  cudaStream_t s = nullptr;
  int64_t m = 0, n = 0, N = 0;
  std::vector<int64_t> arp, aci, trp, tci;  // A and B^T (host, for the factors)
  std::vector<double> av, tv;
  int64_t *d_arp = nullptr, *d_aci = nullptr, *d_trp = nullptr, *d_tci = nullptr;
  double *d_av = nullptr, *d_tv = nullptr, *d_g = nullptr;
  double *x = nullptr, *sres = nullptr, *t = nullptr, *rhat = nullptr, *z = nullptr, *pz = nullptr, *w = nullptr;
  double* scal = nullptr;  // device scalars: [0] norm, [1] inf-norm bits, [2] flag, [3] norm max bits
  LuFactor *fa = nullptr, *fbt = nullptr;
  std::vector<double> history;
  int64_t launches = 0;
};

namespace {

__device__ __forceinline__ double fmax_ref(double m, double a) { return m < a ? a : m; }  // std::max(m, a)

template <int P>
__device__ __forceinline__ double rnd(double v) {
  return round_p<P>(v);
}

// residual_uf (sylvester.cpp:41-56)
template <int P>
__global__ void k_sy_resid(int64_t m, int64_t n, const int64_t* __restrict__ arp, const int64_t* __restrict__ aci,
                           const double* __restrict__ av, const int64_t* __restrict__ trp,
                           const int64_t* __restrict__ tci, const double* __restrict__ tv,
                           const double* __restrict__ g, const double* __restrict__ x, double* __restrict__ r) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m * n) return;
  const int64_t i = q % m, j = q / m;
  double acc = g[q];
  for (int64_t k = arp[i]; k < arp[i + 1]; ++k)
    acc = rnd<P>(__dsub_rn(acc, rnd<P>(__dmul_rn(av[k], x[aci[k] + j * m]))));
  for (int64_t k = trp[j]; k < trp[j + 1]; ++k)
    acc = rnd<P>(__dsub_rn(acc, rnd<P>(__dmul_rn(tv[k], x[i + tci[k] * m]))));
  r[q] = acc;
}

// G - apply(x) (sylvester.cpp:20-39, 58-63): R = (A X)_ij, then R += (X B)_ij
__global__ void k_sy_gap(int64_t m, int64_t n, const int64_t* __restrict__ arp, const int64_t* __restrict__ aci,
                         const double* __restrict__ av, const int64_t* __restrict__ trp,
                         const int64_t* __restrict__ tci, const double* __restrict__ tv,
                         const double* __restrict__ g, const double* __restrict__ x, double* __restrict__ r) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m * n) return;
  const int64_t i = q % m, j = q / m;
  double a = 0.0, b = 0.0;
  for (int64_t k = arp[i]; k < arp[i + 1]; ++k) a = __dadd_rn(a, __dmul_rn(av[k], x[aci[k] + j * m]));
  for (int64_t k = trp[j]; k < trp[j + 1]; ++k) b = __dadd_rn(b, __dmul_rn(tv[k], x[i + tci[k] * m]));
  r[q] = __dsub_rn(g[q], __dadd_rn(a, b));
}

// norm2_64 (kernels.cpp:184-194): m = max|x_i| (exact in any order), the
// terms RN(RN(x_i/m)^2) in parallel, then their sum in the reference's
// sequential order by one thread (only the additions form a chain).
__global__ void k_sy_sq(const double* __restrict__ x, int64_t N, const unsigned long long* __restrict__ mbits,
                        double* __restrict__ w) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double m = __longlong_as_double((long long)*mbits);
  const double q = __ddiv_rn(x[i], m);
  w[i] = __dmul_rn(q, q);
}

__global__ void k_sy_seqsum(const double* __restrict__ w, int64_t N, const unsigned long long* __restrict__ mbits,
                            double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double m = __longlong_as_double((long long)*mbits);
  if (m == 0.0 || !isfinite(m)) {
    *out = m;
    return;
  }
  double s = 0.0;
  int64_t i = 0;
  for (; i + 8 <= N; i += 8) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = w[i + k];
#pragma unroll
    for (int k = 0; k < 8; ++k) s = __dadd_rn(s, v[k]);
  }
  for (; i < N; ++i) s = __dadd_rn(s, w[i]);
  *out = __dmul_rn(m, __dsqrt_rn(s));
}

// inf_norm (kernels.cpp:196-200): std::max(m, |x|), NaN never wins
__global__ void k_sy_infnorm(const double* __restrict__ x, int64_t N, unsigned long long* bits) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double a = fabs(x[i]);
  if (a == a) atomicMax(bits, (unsigned long long)__double_as_longlong(a));
}

template <int P>
__global__ void k_sy_round(double* __restrict__ x, int64_t N) {  // round_vec
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) x[i] = rnd<P>(x[i]);
}

// rhat = round(ldexp(s, -e), u_r) (solver.cpp:88-91)
template <int P>
__global__ void k_sy_scale_round(const double* __restrict__ s, double* __restrict__ r, int e, int64_t N) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) r[i] = rnd<P>(e != 0 ? scalbn(s[i], -e) : s[i]);
}

// scale (kernels.cpp:166-171): round(a * x) in u_r
template <int P>
__global__ void k_sy_scale(double a, const double* __restrict__ x, double* __restrict__ z, int64_t N) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) z[i] = rnd<P>(__dmul_rn(a, x[i]));
}

// y <- ldexp(y, e); x <- axpy(1.0, y, x, u) = round(x + round(1.0 * y)) (solver.cpp:160-166)
template <int P>
__global__ void k_sy_update(const double* __restrict__ y, double* __restrict__ x, int e, int64_t N, int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double yi = e != 0 ? scalbn(y[i], e) : y[i];
  const double v = rnd<P>(__dadd_rn(x[i], rnd<P>(__dmul_rn(1.0, yi))));
  x[i] = v;
  if (!isfinite(v)) *bad = 1;
}

unsigned grid(int64_t N) { return (unsigned)((N + 255) / 256); }

template <class T>
T* dupload(const std::vector<T>& v, cudaStream_t s) {
  T* p = nullptr;
  CK(cudaMallocAsync((void**)&p, std::max<size_t>(v.size(), 1) * sizeof(T), s));
  if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return p;
}

double read_scalar(gadi_sylv* y) {
  double v = 0;
  CK(cudaMemcpyAsync(&v, y->scal, 8, cudaMemcpyDeviceToHost, y->s));
  CK(cudaStreamSynchronize(y->s));
  return v;
}

double norm2_64(gadi_sylv* y, const double* v) {
  unsigned long long* mb = (unsigned long long*)(y->scal + 3);
  CK(cudaMemsetAsync(mb, 0, 8, y->s));
  k_sy_infnorm<<<grid(y->N), 256, 0, y->s>>>(v, y->N, mb);  // std::max(m, |x_i|): NaN never wins
  k_sy_sq<<<grid(y->N), 256, 0, y->s>>>(v, y->N, mb, y->w);
  k_sy_seqsum<<<1, 32, 0, y->s>>>(y->w, y->N, mb, y->scal);
  CKL();
  y->launches += 3;
  return read_scalar(y);
}

double true_norm(gadi_sylv* y) {  // true_residual_norm (sylvester.cpp:58-63)
  k_sy_gap<<<grid(y->N), 256, 0, y->s>>>(y->m, y->n, y->d_arp, y->d_aci, y->d_av, y->d_trp, y->d_tci, y->d_tv,
                                         y->d_g, y->x, y->t);
  CKL();
  ++y->launches;
  return norm2_64(y, y->t);
}

#define SY_DISPATCH(P_, KERN, ...)                                                 \
  do {                                                                           \
    if ((P_) == GADI_HALF) KERN<P_HALF><<<grid(y->N), 256, 0, y->s>>>(__VA_ARGS__);       \
    else if ((P_) == GADI_SINGLE) KERN<P_SINGLE><<<grid(y->N), 256, 0, y->s>>>(__VA_ARGS__); \
    else KERN<P_DOUBLE><<<grid(y->N), 256, 0, y->s>>>(__VA_ARGS__);                \
    CKL();                                                                       \
    ++y->launches;                                                               \
  } while (0)

// rounded_scaled_residual (solver.cpp:86-92): s = residual_uf(x), e, rhat
int rsr(gadi_sylv* y, const gadi_config* c) {
  SY_DISPATCH(c->u_f, k_sy_resid, y->m, y->n, y->d_arp, y->d_aci, y->d_av, y->d_trp, y->d_tci, y->d_tv, y->d_g, y->x,
              y->sres);
  int e = 0;
  if (c->residual_scaling) {  // scaling_exponent (solver.cpp:48-53)
    CK(cudaMemsetAsync(y->scal + 1, 0, 8, y->s));
    k_sy_infnorm<<<grid(y->N), 256, 0, y->s>>>(y->sres, y->N, (unsigned long long*)(y->scal + 1));
    CKL();
    ++y->launches;
    double mx = 0;
    CK(cudaMemcpyAsync(&mx, y->scal + 1, 8, cudaMemcpyDeviceToHost, y->s));
    CK(cudaStreamSynchronize(y->s));
    if (mx != 0.0 && std::isfinite(mx)) e = std::ilogb(mx);
  }
  SY_DISPATCH(c->u_r, k_sy_scale_round, y->sres, y->rhat, e, y->N);
  return e;
}

void release_factors(gadi_sylv* y) {
  lu_release(y->fa, y->s);
  lu_release(y->fbt, y->s);
  y->fa = y->fbt = nullptr;
}

void validate_cfg(const gadi_config* c) {  // solver.cpp:33-40
  if (!(c->alpha > 0.0)) throw Err(GADI_E_PARAM, "alpha must be positive");
  if (!(c->omega >= 0.0 && c->omega < 2.0)) throw Err(GADI_E_PARAM, "omega must be in [0, 2)");
  if (c->xi < 0.0) throw Err(GADI_E_PARAM, "xi must be positive");
  if (c->max_outer_iters < 1) throw Err(GADI_E_PARAM, "max_outer_iters must be >= 1");
  for (int p : {c->u_r, c->u, c->u_f})
    if (p < 0 || p > 2) throw Err(GADI_E_PARAM, "unknown precision");
  const double uu = unit_roundoff(c->u), uf = unit_roundoff(c->u_f), ur = unit_roundoff(c->u_r);
  if (!(uu <= uf && uf <= ur)) throw Err(GADI_E_PARAM, "precision triple must satisfy u <= u_f <= u_r");
}

// run_gadi_ir (solver.cpp:57-179) over the SylvesterOperator
void run_sylv(gadi_sylv* y, const gadi_config* c, gadi_report* rep) {
  validate_cfg(c);
  const double xi = c->xi > 0.0 ? c->xi : gadi_default_xi(c->u);
  std::memset(rep, 0, sizeof(*rep));
  rep->status = GADI_MAX_ITERS;
  rep->final_rres = 1.0;
  y->history.assign(1, 1.0);
  const int64_t l0 = y->launches;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, y->s));
  auto finish = [&]() {
    CK(cudaEventRecord(e1, y->s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    rep->solve_ms = ms;
    rep->history_len = (int)y->history.size();
    rep->launches = y->launches - l0;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  };
  if (c->u != GADI_DOUBLE) SY_DISPATCH(c->u, k_sy_round, y->x, y->N);  // x = round_vec(x0, u)
  const double nt0 = true_norm(y);
  if (nt0 == 0.0) {
    rep->status = GADI_CONVERGED;
    rep->final_rres = 0.0;
    finish();
    return;
  }
  // prepare (sylvester.cpp:66-73): factorize alpha I + A and alpha I + B^T in u_r
  release_factors(y);
  int st = 0;
  y->fa = lu_factor_host_csr(y->device, y->s, y->m, y->arp.data(), y->aci.data(), y->av.data(), c->alpha, c->u_r, &st);
  y->launches += y->fa->launches;
  if (st == 0) {
    y->fbt = lu_factor_host_csr(y->device, y->s, y->n, y->trp.data(), y->tci.data(), y->tv.data(), c->alpha, c->u_r,
                                &st);
    y->launches += y->fbt->launches;
  }
  if (st != 0) {  // SingularInPrecision / OverflowDetected (solver.cpp:74-82)
    rep->status = st;
    finish();
    return;
  }
  int e = rsr(y, c);
  const double g0 = std::ldexp(norm2_64(y, y->rhat), e);
  const double p_rounded = hround((2.0 - c->omega) * c->alpha, c->u_r);
  double best = 1.0;
  int best_iter = 0;
  for (int k = 0;; ++k) {
    const double rres = y->history.back();
    rep->final_rres = rres;
    rep->outer_iters = k;
    const double gn = std::ldexp(norm2_64(y, y->rhat), e);
    const bool guard = gn * gn <= g0 * g0 * xi;
    const bool truem = rres * rres <= xi;
    if (guard && truem) { rep->status = GADI_CONVERGED; break; }
    if (guard) { rep->status = GADI_STALLED; break; }
    if (!std::isfinite(rres)) { rep->status = GADI_OVERFLOW_DETECTED; break; }
    if (rres > c->divergence_factor) { rep->status = GADI_DIVERGED; break; }
    if (c->stall_window > 0) {
      if (rres < best * (1.0 - 1e-3)) {
        best = rres;
        best_iter = k;
      } else if (k - best_iter >= c->stall_window) {
        rep->status = GADI_STALLED;
        break;
      }
    }
    if (k >= c->max_outer_iters) { rep->status = GADI_MAX_ITERS; break; }
    // solve_H: (alpha I + A) Z = R column by column (sylvester.cpp:83-96)
    CK(cudaMemcpyAsync(y->z, y->rhat, y->N * 8, cudaMemcpyDeviceToDevice, y->s));
    if (!lu_solve_many(y->fa, y->z, 1, y->m, y->n, y->s)) { rep->status = GADI_OVERFLOW_DETECTED; break; }
    ++y->launches;
    SY_DISPATCH(c->u_r, k_sy_scale, p_rounded, y->z, y->pz, y->N);
    // solve_S: (alpha I + B^T) row by row (sylvester.cpp:98-119)
    if (!lu_solve_many(y->fbt, y->pz, y->m, 1, y->m, y->s)) { rep->status = GADI_OVERFLOW_DETECTED; break; }
    ++y->launches;
    int* bad = (int*)(y->scal + 2);
    CK(cudaMemsetAsync(bad, 0, 4, y->s));
    SY_DISPATCH(c->u, k_sy_update, y->pz, y->x, e, y->N, bad);
    int hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, y->s));
    CK(cudaStreamSynchronize(y->s));
    if (hbad) {  // solver.cpp:168-174
      y->history.push_back(true_norm(y) / nt0);
      rep->outer_iters = k + 1;
      rep->final_rres = y->history.back();
      rep->status = GADI_OVERFLOW_DETECTED;
      break;
    }
    e = rsr(y, c);
    y->history.push_back(true_norm(y) / nt0);
  }
  finish();
}

int fail_sy(const Err& e) {
  set_last_error(e.what());
  return e.code;
}

void check_csr(int64_t N, const int64_t* rp, const int64_t* ci, const double* v, const char* what) {
  if (N < 1 || !rp || (rp[N] > 0 && (!ci || !v))) throw Err(GADI_E_CONTRACT, std::string(what) + ": bad arguments");
  if (rp[0] != 0) throw Err(GADI_E_CONTRACT, "row_ptr must start at 0");
  for (int64_t i = 0; i < N; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      if (ci[k] < 0 || ci[k] >= N) throw Err(GADI_E_CONTRACT, "column index out of range");
      if (k > rp[i] && ci[k] <= ci[k - 1])
        throw Err(GADI_E_CONTRACT, "column indices must be strictly increasing within a row");
    }
}

}  // namespace

extern "C" {

int gadi_sylv_create(int64_t m, const int64_t* a_rp, const int64_t* a_ci, const double* a_v, int64_t n,
                     const int64_t* b_rp, const int64_t* b_ci, const double* b_v, const double* G, int32_t device,
                     gadi_sylv** out) {
  try {
    if (!out || !G) throw Err(GADI_E_CONTRACT, "sylv_create: null argument");
    *out = nullptr;
    check_csr(m, a_rp, a_ci, a_v, "A");
    check_csr(n, b_rp, b_ci, b_v, "B");
    std::unique_ptr<gadi_sylv> y(new gadi_sylv);
    y->device = device;
    y->m = m;
    y->n = n;
    y->N = m * n;
    y->arp.assign(a_rp, a_rp + m + 1);
    y->aci.assign(a_ci, a_ci + a_rp[m]);
    y->av.assign(a_v, a_v + a_rp[m]);
    // B^T (sparse.cpp:104-117: counting sort by column, rows in order)
    const int64_t nb = b_rp[n];
    y->trp.assign(n + 1, 0);
    y->tci.resize(nb);
    y->tv.resize(nb);
    for (int64_t k = 0; k < nb; ++k) ++y->trp[b_ci[k] + 1];
    for (int64_t j = 0; j < n; ++j) y->trp[j + 1] += y->trp[j];
    std::vector<int64_t> next(y->trp.begin(), y->trp.end() - 1);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = b_rp[i]; k < b_rp[i + 1]; ++k) {
        const int64_t p = next[b_ci[k]]++;
        y->tci[p] = i;
        y->tv[p] = b_v[k];
      }
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&y->s, cudaStreamNonBlocking));
    y->d_arp = dupload(y->arp, y->s);
    y->d_aci = dupload(y->aci, y->s);
    y->d_av = dupload(y->av, y->s);
    y->d_trp = dupload(y->trp, y->s);
    y->d_tci = dupload(y->tci, y->s);
    y->d_tv = dupload(y->tv, y->s);
    y->d_g = dupload(std::vector<double>(G, G + y->N), y->s);
    for (double** p : {&y->x, &y->sres, &y->t, &y->rhat, &y->z, &y->pz, &y->w})
      CK(cudaMallocAsync((void**)p, y->N * 8, y->s));
    CK(cudaMallocAsync((void**)&y->scal, 32, y->s));
    CK(cudaStreamSynchronize(y->s));
    *out = y.release();
  } catch (const Err& e) {
    return fail_sy(e);
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GADI_E_CUDA;
  }
  return GADI_OK;
}

int gadi_sylv_destroy(gadi_sylv* y) {
  if (!y) return GADI_OK;
  cudaSetDevice(y->device);
  cudaStreamSynchronize(y->s);
  release_factors(y);
  for (void* p : {(void*)y->d_arp, (void*)y->d_aci, (void*)y->d_av, (void*)y->d_trp, (void*)y->d_tci,
                  (void*)y->d_tv, (void*)y->d_g, (void*)y->x, (void*)y->sres, (void*)y->t, (void*)y->rhat,
                  (void*)y->z, (void*)y->pz, (void*)y->w, (void*)y->scal})
    if (p) cudaFreeAsync(p, y->s);
  cudaStreamSynchronize(y->s);
  cudaStreamDestroy(y->s);
  delete y;
  return GADI_OK;
}

int gadi_sylv_solve(gadi_sylv* y, const gadi_config* cfg, const double* x0, double* x_out, gadi_report* rep) {
  try {
    if (!y || !cfg || !x_out || !rep) throw Err(GADI_E_CONTRACT, "sylv_solve: null argument");
    CK(cudaSetDevice(y->device));
    if (x0) {
      CK(cudaMemcpyAsync(y->x, x0, y->N * 8, cudaMemcpyHostToDevice, y->s));
    } else {  // gadi_ab_solve's x0 (sylvester.cpp:129): zeros, or ones if ones_start
      std::vector<double> v(y->N, cfg->ones_start ? 1.0 : 0.0);
      CK(cudaMemcpyAsync(y->x, v.data(), y->N * 8, cudaMemcpyHostToDevice, y->s));
      CK(cudaStreamSynchronize(y->s));
    }
    run_sylv(y, cfg, rep);
    CK(cudaMemcpyAsync(x_out, y->x, y->N * 8, cudaMemcpyDeviceToHost, y->s));
    CK(cudaStreamSynchronize(y->s));
  } catch (const Err& e) {
    return fail_sy(e);
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GADI_E_CUDA;
  }
  return GADI_OK;
}

int gadi_sylv_history(const gadi_sylv* y, double* out, int32_t cap) {
  if (!y || (!out && cap > 0)) return GADI_E_CONTRACT;
  const int k = (int)std::min<size_t>(y->history.size(), (size_t)std::max(cap, 0));
  for (int i = 0; i < k; ++i) out[i] = y->history[i];
  return k;
}

}  // extern "C"
