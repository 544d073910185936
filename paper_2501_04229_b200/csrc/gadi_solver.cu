// gadi_solver.cu — host side of the B200 GADI-IR solver and its C ABI.
//
// run_gadi_ir (solver.cpp:57-179) is restated over device-resident vectors:
// x, b, s in binary64, the inner vectors in u_r storage. Per outer step the
// host issues CG on H, the p-scaling, GMRES on S, the update and the new
// residual; the only host<->device traffic inside the loop is a few small
// status reads (one per GMRES Arnoldi step, one per outer step) — the CG
// recurrences and stop tests run on the device (gadi_kernels.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gadi_cuda.h"
#include "gadi_kernels.cuh"

using namespace gadi;

namespace {

thread_local std::string g_last_error;

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
double hround(double x, int p) {
  if (p == GADI_SINGLE) return (double)(float)x;
  if (p != GADI_HALF) return x;
  if (std::isnan(x) || std::isinf(x) || x == 0.0) return x;
  const double ax = std::fabs(x);
  if (ax >= 65520.0) return std::copysign(INFINITY, x);
  const int e = std::ilogb(ax);
  const int q = e < -14 ? -24 : e - 10;
  return std::copysign(std::ldexp(std::nearbyint(std::ldexp(ax, -q)), q), x);
}

double unit_roundoff(int p) {
  return p == GADI_HALF ? std::ldexp(1.0, -11) : p == GADI_SINGLE ? std::ldexp(1.0, -24) : std::ldexp(1.0, -53);
}

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
int ilog2(int64_t v) {
  int d = 0;
  while ((int64_t(1) << (d + 1)) <= v) ++d;
  return d;
}

Geo make_geo(int64_t N, int vec) {
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
  g.bdim = (int)std::min<int64_t>(256, nseg);
  g.nblk = (int)(nseg / g.bdim);
  return g;
}

template <int V>
struct VecTag {
  static constexpr int v = V;
};

// Elementwise launch geometry.
inline dim3 ew_grid(int64_t n) { return dim3((unsigned)((n + 255) / 256)); }

template <class T>
constexpr int prec_of() {
  return std::is_same<T, __half>::value ? GADI_HALF : std::is_same<T, float>::value ? GADI_SINGLE : GADI_DOUBLE;
}

// ---------------------------------------------------------------- the problem
struct HostCsr {
  std::vector<int64_t> rp, ci;
  std::vector<double> v;
};

// hss_split (splitting.cpp:12-20) on the host for the CSR path: union pattern
// of A and A^T, M = (A + A^T)/2, N = (A - A^T)/2 with explicit zeros, plus the
// diagonal in the pattern (shift_diagonal, sparse.cpp:180-183). Returns M/N
// values on the shared pattern and whether each row's diagonal came from M's
// own pattern (for the alpha shift).
void hss_split_host(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, HostCsr& P,
                    std::vector<double>& Mv, std::vector<double>& Nv, std::vector<uint8_t>& diag_in) {
  const int64_t nnz = rp[n];
  std::vector<int64_t> trp(n + 1, 0), tci(nnz), next(n);
  std::vector<double> tv(nnz);
  for (int64_t k = 0; k < nnz; ++k) ++trp[ci[k] + 1];
  for (int64_t j = 0; j < n; ++j) trp[j + 1] += trp[j];
  for (int64_t j = 0; j < n; ++j) next[j] = trp[j];
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t q = next[ci[k]]++;
      tci[q] = i;
      tv[q] = v[k];
    }
  P.rp.assign(n + 1, 0);
  P.ci.clear();
  Mv.clear();
  Nv.clear();
  diag_in.clear();
  P.ci.reserve(nnz + n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t a = rp[i], ae = rp[i + 1], t = trp[i], te = trp[i + 1];
    bool diag_done = false;
    while (a < ae || t < te || !diag_done) {
      const int64_t ca = a < ae ? ci[a] : INT64_MAX, ct = t < te ? tci[t] : INT64_MAX;
      int64_t col = std::min(ca, ct);
      if (!diag_done && i <= col) col = i;
      const bool hA = ca == col, hT = ct == col;
      double m = 0.0, nv = 0.0;
      if (hA && hT) {
        m = 0.5 * v[a] + 0.5 * tv[t];
        nv = 0.5 * v[a] + -0.5 * tv[t];
      } else if (hA) {
        m = 0.5 * v[a];
        nv = 0.5 * v[a];
      } else if (hT) {
        m = 0.5 * tv[t];
        nv = -0.5 * tv[t];
      }
      if (col == i) {
        diag_done = true;
        diag_in.push_back(hA || hT);
      }
      P.ci.push_back(col);
      Mv.push_back(m);
      Nv.push_back(nv);
      if (hA) ++a;
      if (hT) ++t;
    }
    P.rp[i + 1] = (int64_t)P.ci.size();
  }
}

}  // namespace

// ==================================================================== handle
struct EngineBase;

struct gadi_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  int kind = GADI_PROBLEM_STENCIL7;
  int64_t N = 0, n = 0;
  double t1 = 0, t2 = 0, t3 = 0;
  // CSR A (device) and the HSS pattern (device) + fp64 M/N values (host)
  int64_t* d_rpA = nullptr;
  int32_t* d_ciA = nullptr;
  double* d_vA = nullptr;
  int64_t nnzA = 0, nnzHS = 0;
  int64_t* d_rpHS = nullptr;
  int32_t* d_ciHS = nullptr;
  std::vector<double> Mv, Nv;
  std::vector<int64_t> diag_pos;  // position of (i,i) in the HS pattern
  std::vector<uint8_t> diag_in;
  // outer vectors (binary64)
  double *d_x = nullptr, *d_b = nullptr, *d_s = nullptr, *d_t64 = nullptr;
  // reductions / state
  DevState* st = nullptr;
  DevState* h_st = nullptr;  // pinned mirror
  double *d_part0 = nullptr, *d_part1 = nullptr;
  unsigned* d_ticket = nullptr;
  int* h_done = nullptr;  // mapped pinned flag (CG done)
  int* d_h_done = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evA = nullptr, evB = nullptr;
  std::vector<cudaEvent_t> ring;
  // prepared inner engine
  std::unique_ptr<EngineBase> eng;
  bool have_rhs = false;
  double stop_norm = 1.0;
  std::vector<double> history;
};

namespace {

template <class T>
T* dalloc(int64_t n) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<int64_t>(n, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

void read_state(gadi_handle* h) {
  CK(cudaMemcpyAsync(h->h_st, h->st, sizeof(DevState), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
}

Red red_of(gadi_handle* h) { return Red{h->d_part0, h->d_part1, h->d_ticket}; }

// ------------------------------------------------------------ outer kernels on A
struct OuterA {
  // s = b - A x in u_f; s == nullptr computes the norm only.
  static void resid(gadi_handle* h, const double* x, double* s, int uf, bool scaling) {
    CK(cudaMemsetAsync(&h->st->maxbits, 0, sizeof(unsigned long long), h->stream));
    const bool al = (h->N % 2 == 0) && is_pow2(h->N / 2) && (h->kind == GADI_PROBLEM_CSR || h->n % 2 == 0);
    const Geo g = make_geo(h->N, al ? 2 : 1);
    auto go = [&](auto op) {
      auto L = [&](auto pt, auto vt) {
        constexpr int PF = decltype(pt)::v, V = decltype(vt)::v;
        k_resid_A<decltype(op), PF, V><<<g.nblk, g.bdim, 0, h->stream>>>(op, x, h->d_b, s, scaling ? 1 : 0, g,
                                                                          red_of(h), h->st);
      };
      auto LV = [&](auto pt) {
        if (al) L(pt, VecTag<2>{});
        else L(pt, VecTag<1>{});
      };
      if (uf == GADI_HALF) LV(VecTag<P_HALF>{});
      else if (uf == GADI_SINGLE) LV(VecTag<P_SINGLE>{});
      else LV(VecTag<P_DOUBLE>{});
    };
    if (h->kind == GADI_PROBLEM_STENCIL7) {
      Stencil7<double> op{h->n, h->n * h->n, h->N, {h->t2, h->t2, h->t2, h->t1, h->t3, h->t3, h->t3}};
      go(op);
    } else {
      Csr<double> op{h->N, h->d_rpA, h->d_ciA, h->d_vA};
      go(op);
    }
    CKL();
  }
  static void apply(gadi_handle* h, const double* x, double* y) {
    auto go = [&](auto op) {
      k_apply<decltype(op), double, double, double><<<ew_grid(h->N), 256, 0, h->stream>>>(op, x, y, h->N,
                                                                                          MatvecAF());
    };
    if (h->kind == GADI_PROBLEM_STENCIL7) {
      Stencil7<double> op{h->n, h->n * h->n, h->N, {h->t2, h->t2, h->t2, h->t1, h->t3, h->t3, h->t3}};
      go(op);
    } else {
      Csr<double> op{h->N, h->d_rpA, h->d_ciA, h->d_vA};
      go(op);
    }
    CKL();
  }
};

}  // namespace

// ================================================================== engines
struct InnerOut {
  int iters = 0;
  int status = INNER_CONVERGED;
};

struct EngineBase {
  virtual ~EngineBase() = default;
  int u_r = GADI_DOUBLE, accum = 0, cprec = GADI_DOUBLE;
  size_t tsize = 8;
  gadi_inner_spec spec{};
  double alpha = 1, omega = 1;
  // inner-format device vectors (type-erased)
  void *rhat = nullptr, *z = nullptr, *pz = nullptr, *y = nullptr;
  // H/S solves on inner-format device vectors
  virtual InnerOut cg(int which, const void* rhs, void* x, double target) = 0;
  virtual InnerOut gmres(int which, const void* rhs, void* x, double target) = 0;
  virtual void scale_round(const double* s) = 0;        // rhat = round(s 2^-e)
  virtual void scale_pz(double phat) = 0;               // pz = round(phat z)
  virtual void update(double* x, int pu) = 0;           // x += 2^e y
  virtual void to_inner(const double* src, void* dst) = 0;  // round_vec to u_r
  virtual void to_double(const void* src, double* dst) = 0;
  virtual void apply(int which, const void* x, void* yv) = 0;
};

namespace {

template <class Op, class T, class C>
struct Engine final : EngineBase {
  gadi_handle* h;
  Op opH, opS;
  bool aligned;
  Geo geo;
  static constexpr int VA = 16 / sizeof(T);
  // CG / GMRES work vectors
  T *r = nullptr, *p = nullptr, *q = nullptr, *xw = nullptr, *w = nullptr, *gr = nullptr, *V = nullptr;
  C* dH = nullptr;  // CSR values (device)
  C* dS = nullptr;
  int m_restart = 30;
  std::vector<T*> owned;

  T* vec() {
    T* v = dalloc<T>(h->N);
    owned.push_back(v);
    return v;
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
    aligned = (N % VA == 0) && is_pow2(N / VA) && (h->kind == GADI_PROBLEM_CSR || h->n % VA == 0);
    geo = make_geo(N, aligned ? VA : 1);
    m_restart = std::max(1, spec.restart);
    rhat = vec();
    z = vec();
    pz = vec();
    y = vec();
    r = vec();
    p = vec();
    q = vec();
    w = vec();
    gr = vec();
    V = dalloc<T>((int64_t)(m_restart + 1) * N);
    owned.push_back(V);
    build_ops();
  }

  ~Engine() override {
    for (T* v : owned) cudaFree(v);
    if (dH) cudaFree(dH);
    if (dS) cudaFree(dS);
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
      for (int k = 0; k < 7; ++k) {
        opH.c[k] = cval(Hc[k], u_r);
        opS.c[k] = cval(Sc[k], u_r);
      }
    } else {
      const int64_t nnz = h->nnzHS;
      std::vector<C> hv(nnz), sv(nnz);
      for (int64_t k = 0; k < nnz; ++k) {
        hv[k] = cval(h->Mv[k], u_r);
        sv[k] = cval(h->Nv[k], u_r);
      }
      for (int64_t i = 0; i < h->N; ++i) {
        const int64_t k = h->diag_pos[i];
        hv[k] = cval(h->diag_in[i] ? 1.0 * h->Mv[k] + alpha : alpha, u_r);
        sv[k] = cval(h->diag_in[i] ? 1.0 * h->Nv[k] + alpha : alpha, u_r);
      }
      dH = dalloc<C>(nnz);
      dS = dalloc<C>(nnz);
      CK(cudaMemcpy(dH, hv.data(), nnz * sizeof(C), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dS, sv.data(), nnz * sizeof(C), cudaMemcpyHostToDevice));
      opH = Op{h->N, h->d_rpHS, h->d_ciHS, dH};
      opS = Op{h->N, h->d_rpHS, h->d_ciHS, dS};
    }
  }

  template <class F>
  void V2(F&& f) {
    if (aligned) f(VecTag<VA>{});
    else f(VecTag<1>{});
  }

  const Op& op(int which) const { return which == 1 ? opH : opS; }

  // ------------------------------------------------------------------ CG
  // inner_solver.cpp:47-83 on the device; the host only keeps the queue
  // filled, at most kAhead iterations ahead of the device, and stops queueing
  // once the device raises the (mapped) done flag.
  InnerOut cg(int which, const void* rhs_v, void* x_v, double target) override {
    const T* rhs = static_cast<const T*>(rhs_v);
    T* x = static_cast<T*>(x_v);
    cudaStream_t s = h->stream;
    const Red rd = red_of(h);
    const Op& o = op(which);
    *(volatile int*)h->h_done = 0;
    V2([&](auto vt) {
      constexpr int V_ = decltype(vt)::v;
      k_cg_init<T, C, V_><<<geo.nblk, geo.bdim, 0, s>>>(rhs, r, p, x, spec.max_inner_iters, target, geo, rd, h->st);
    });
    CKL();
    const int kAhead = (int)h->ring.size();
    for (int it = 0; it < spec.max_inner_iters; ++it) {
      if (it >= kAhead) {
        CK(cudaEventSynchronize(h->ring[it % kAhead]));
        if (*(volatile int*)h->h_done) break;
      }
      V2([&](auto vt) {
        constexpr int V_ = decltype(vt)::v;
        k_cg_spmv<Op, T, C, V_><<<geo.nblk, geo.bdim, 0, s>>>(o, p, q, geo, rd, h->st);
        k_cg_update<T, C, V_><<<geo.nblk, geo.bdim, 0, s>>>(x, r, p, q, geo, rd, h->st);
        k_cg_pupd<T, C, V_><<<geo.nblk, geo.bdim, 0, s>>>(r, p, geo, h->st);
      });
      CKL();
      CK(cudaEventRecord(h->ring[it % kAhead], s));
    }
    read_state(h);
    InnerOut out;
    out.iters = h->h_st->cg_iters;
    out.status = h->h_st->cg_status;
    return out;
  }

  // --------------------------------------------------------------- GMRES
  // inner_solver.cpp:85-194: vector work on the device (MGS fused with the
  // next Arnoldi dot), the (m+1) x m Hessenberg / Givens / back-solve on the
  // host in the inner format's rounding.
  InnerOut gmres(int which, const void* rhs_v, void* x_v, double target) override {
    const T* rhs = static_cast<const T*>(rhs_v);
    T* x = static_cast<T*>(x_v);
    cudaStream_t s = h->stream;
    const Red rd = red_of(h);
    const Op& o = op(which);
    const int64_t N = h->N;
    const int m = m_restart, fmt = cprec;
    auto Rf = [&](double v) { return hround(v, fmt); };
    CK(cudaMemsetAsync(x, 0, N * sizeof(T), s));
    std::vector<double> Hc((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), yv(m + 1);
    auto HC = [&](int i, int j) -> double& { return Hc[(size_t)i * m + j]; };
    int total = 0;
    InnerOut out;
    int status = -1;
    auto resid = [&]() {  // r = rhs - S x ; flags, max, ||r||_2 (binary64), norm2 in fmt
      CK(cudaMemsetAsync(&h->st->maxbits, 0, 8, s));
      CK(cudaMemsetAsync(&h->st->flags, 0, 4, s));
      V2([&](auto vt) {
        constexpr int V_ = decltype(vt)::v;
        k_gm_resid<Op, T, C, V_><<<geo.nblk, geo.bdim, 0, s>>>(o, x, rhs, gr, geo, rd, h->st);
        k_norm2<T, C, V_><<<geo.nblk, geo.bdim, 0, s>>>(gr, &h->st->red_c, geo, rd, h->st);
      });
      CKL();
      read_state(h);
    };
    while (total < spec.max_inner_iters) {
      resid();
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
      V2([&](auto vt) {
        constexpr int V_ = decltype(vt)::v;
        k_scale<T, V_><<<geo.nblk, geo.bdim, 0, s>>>(gr, V, 1.0 / beta, geo);
      });
      std::fill(Hc.begin(), Hc.end(), 0.0);
      std::fill(cs.begin(), cs.end(), 0.0);
      std::fill(sn.begin(), sn.end(), 0.0);
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      int j = 0;
      bool happy = false;
      for (; j < m && total < spec.max_inner_iters; ++j, ++total) {
        T* vj = V + (int64_t)j * N;
        V2([&](auto vt) {
          constexpr int V_ = decltype(vt)::v;
          k_gm_matvec<Op, T, C, V_><<<geo.nblk, geo.bdim, 0, s>>>(o, vj, V, w, geo, rd, h->st);
          for (int i = 0; i <= j; ++i) {
            T* vi = V + (int64_t)i * N;
            if (i < j) {
              k_gm_mgs<T, C, V_, false><<<geo.nblk, geo.bdim, 0, s>>>(w, vi, vi + N, i, geo, rd, h->st);
            } else {
              CK(cudaMemsetAsync(&h->st->maxbits, 0, 8, s));
              k_gm_mgs<T, C, V_, true><<<geo.nblk, geo.bdim, 0, s>>>(w, vi, nullptr, i, geo, rd, h->st);
            }
          }
          k_norm2<T, C, V_><<<geo.nblk, geo.bdim, 0, s>>>(w, &h->st->hcol[j + 1], geo, rd, h->st);
        });
        CKL();
        read_state(h);
        for (int i = 0; i <= j + 1; ++i) HC(i, j) = h->h_st->hcol[i];
        const double h1 = HC(j + 1, j);
        if (!std::isfinite(h1)) {
          status = INNER_OVERFLOW;
          goto done;
        }
        if (h1 != 0.0) {
          V2([&](auto vt) {
            constexpr int V_ = decltype(vt)::v;
            k_scale<T, V_><<<geo.nblk, geo.bdim, 0, s>>>(w, V + (int64_t)(j + 1) * N, 1.0 / h1, geo);
          });
        }
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
        k_gm_update<T, C, V_><<<geo.nblk, geo.bdim, 0, s>>>(x, V, N, j, geo, h->st);
      });
      CKL();
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
    if (status < 0) {
      // all_finite(x) (inner_solver.cpp:192): x was finite after its last update
      // or the loop would have returned Overflow.
      status = INNER_STAGNATED;
    }
    out.iters = total;
    out.status = status;
    return out;
  }

  // ----------------------------------------------------------- outer pieces
  void scale_round(const double* sv) override {
    const Red rd = red_of(h);
    if constexpr (sizeof(T) * 2 == 16 || true) {
      const bool al = (h->N % 2 == 0) && is_pow2(h->N / 2) && (h->kind == GADI_PROBLEM_CSR || h->n % 2 == 0);
      const Geo g = make_geo(h->N, al ? 2 : 1);
      if (al) k_scale_round<T, 2><<<g.nblk, g.bdim, 0, h->stream>>>(sv, static_cast<T*>(rhat), g, rd, h->st);
      else k_scale_round<T, 1><<<g.nblk, g.bdim, 0, h->stream>>>(sv, static_cast<T*>(rhat), g, rd, h->st);
    }
    CKL();
  }
  void scale_pz(double phat) override {
    V2([&](auto vt) {
      constexpr int V_ = decltype(vt)::v;
      k_scale<T, V_><<<geo.nblk, geo.bdim, 0, h->stream>>>(static_cast<T*>(z), static_cast<T*>(pz), phat, geo);
    });
    CKL();
  }
  void update(double* x, int pu) override {
    const bool al = (h->N % 2 == 0) && is_pow2(h->N / 2) && (h->kind == GADI_PROBLEM_CSR || h->n % 2 == 0);
    const Geo g = make_geo(h->N, al ? 2 : 1);
    auto L = [&](auto pt, auto vt) {
      constexpr int PU = decltype(pt)::v, V_ = decltype(vt)::v;
      k_update<T, PU, V_><<<g.nblk, g.bdim, 0, h->stream>>>(x, static_cast<const T*>(y), g, h->st);
    };
    auto LV = [&](auto pt) {
      if (al) L(pt, VecTag<2>{});
      else L(pt, VecTag<1>{});
    };
    if (pu == GADI_HALF) LV(VecTag<P_HALF>{});
    else if (pu == GADI_SINGLE) LV(VecTag<P_SINGLE>{});
    else LV(VecTag<P_DOUBLE>{});
    CKL();
  }
  void to_inner(const double* src, void* dst) override {
    constexpr int PT = prec_of<T>();
    k_convert<double, T, PT><<<ew_grid(h->N), 256, 0, h->stream>>>(src, static_cast<T*>(dst), h->N);
    CKL();
  }
  void to_double(const void* src, double* dst) override {
    k_convert<T, double, P_DOUBLE><<<ew_grid(h->N), 256, 0, h->stream>>>(static_cast<const T*>(src), dst, h->N);
    CKL();
  }
  void apply(int which, const void* xv, void* yv_) override {
    k_apply<Op, T, C, T><<<ew_grid(h->N), 256, 0, h->stream>>>(op(which), static_cast<const T*>(xv),
                                                               static_cast<T*>(yv_), h->N, MatvecF<C, T>());
    CKL();
  }
};

template <class T, class C>
EngineBase* make_engine_tc(gadi_handle* h, const gadi_inner_spec& sp, double a, double om, int ur, int acc) {
  if (h->kind == GADI_PROBLEM_STENCIL7) return new Engine<Stencil7<C>, T, C>(h, sp, a, om, ur, acc);
  return new Engine<Csr<C>, T, C>(h, sp, a, om, ur, acc);
}

EngineBase* make_engine(gadi_handle* h, const gadi_inner_spec& sp, double a, double om, int ur, int acc) {
  if (ur == GADI_DOUBLE) return make_engine_tc<double, double>(h, sp, a, om, ur, acc);
  if (ur == GADI_SINGLE) return make_engine_tc<float, float>(h, sp, a, om, ur, acc);
  if (acc == GADI_ACCUM_FP32) return make_engine_tc<__half, float>(h, sp, a, om, ur, acc);
  return make_engine_tc<__half, __half>(h, sp, a, om, ur, acc);
}

// ---------------------------------------------------------------- validation
void validate(const gadi_config* c) {
  // solver.cpp:33-40
  if (!(c->alpha > 0.0)) throw Err(GADI_E_PARAM, "alpha must be positive");
  if (!(c->omega >= 0.0 && c->omega < 2.0)) throw Err(GADI_E_PARAM, "omega must be in [0, 2)");
  if (c->xi < 0.0) throw Err(GADI_E_PARAM, "xi must be positive");
  if (c->max_outer_iters < 1) throw Err(GADI_E_PARAM, "max_outer_iters must be >= 1");
  for (int p : {c->u_r, c->u, c->u_f})
    if (p < 0 || p > 2) throw Err(GADI_E_PARAM, "unknown precision");
  const double uu = unit_roundoff(c->u), uf = unit_roundoff(c->u_f), ur = unit_roundoff(c->u_r);
  if (!(uu <= uf && uf <= ur)) throw Err(GADI_E_PARAM, "precision triple must satisfy u <= u_f <= u_r");
  if (c->inner.method == GADI_INNER_LU_DIRECT)
    throw Err(GADI_E_UNSUPPORTED, "inner method lu_direct has no device implementation (use cg or gmres)");
  if (c->inner.method != GADI_INNER_CG && c->inner.method != GADI_INNER_GMRES)
    throw Err(GADI_E_PARAM, "unknown inner method");
  if (c->accum != GADI_ACCUM_NATIVE && c->accum != GADI_ACCUM_FP32) throw Err(GADI_E_PARAM, "unknown accum");
}

void prepare(gadi_handle* h, double alpha, double omega, int ur, const gadi_inner_spec& sp, int accum) {
  if (!(alpha > 0.0)) throw Err(GADI_E_PARAM, "regularize: alpha must be positive");
  if (!(omega >= 0.0 && omega < 2.0)) throw Err(GADI_E_PARAM, "regularize: omega must be in [0, 2)");
  if (sp.method == GADI_INNER_LU_DIRECT)
    throw Err(GADI_E_UNSUPPORTED, "inner method lu_direct has no device implementation (use cg or gmres)");
  auto& e = h->eng;
  const bool same = e && e->u_r == ur && e->accum == accum && e->spec.restart == sp.restart;
  if (same && e->alpha == alpha && e->omega == omega) {
    e->spec = sp;
    return;
  }
  e.reset();
  CK(cudaDeviceSynchronize());
  e.reset(make_engine(h, sp, alpha, omega, ur, accum));
}

double ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// run_gadi_ir (solver.cpp:57-179) on device vectors d_b (already in h->d_b)
// and x0 (already in h->d_x, rounded to u below).
void run(gadi_handle* h, const gadi_config* cfg, gadi_report* rep) {
  validate(cfg);
  const double xi = cfg->xi > 0.0 ? cfg->xi : gadi_default_xi(cfg->u);
  std::memset(rep, 0, sizeof(*rep));
  rep->status = GADI_MAX_ITERS;
  rep->final_rres = 1.0;
  h->history.assign(1, 1.0);
  cudaStream_t s = h->stream;
  const int64_t N = h->N;
  CK(cudaEventRecord(h->ev0, s));
  float h_ms = 0, s_ms = 0;

  // x = round_vec(x0, u) (solver.cpp:65)
  {
    auto L = [&](auto pt) {
      constexpr int P = decltype(pt)::v;
      k_convert<double, double, P><<<ew_grid(N), 256, 0, s>>>(h->d_x, h->d_x, N);
    };
    if (cfg->u == GADI_HALF) L(VecTag<P_HALF>{});
    else if (cfg->u == GADI_SINGLE) L(VecTag<P_SINGLE>{});
    CKL();
  }
  // nt0 = true_residual_norm(x) (solver.cpp:67)
  OuterA::resid(h, h->d_x, nullptr, GADI_DOUBLE, false);
  read_state(h);
  const double nt0 = std::sqrt(h->h_st->res_ss);
  auto finish = [&]() {
    CK(cudaEventRecord(h->ev1, s));
    CK(cudaEventSynchronize(h->ev1));
    rep->solve_ms = ms_between(h->ev0, h->ev1);
    rep->h_ms = h_ms;
    rep->s_ms = s_ms;
    rep->history_len = (int)h->history.size();
  };
  if (nt0 == 0.0) {
    rep->status = GADI_CONVERGED;
    rep->final_rres = 0.0;
    finish();
    return;
  }
  prepare(h, cfg->alpha, cfg->omega, cfg->u_r, cfg->inner, cfg->accum);
  EngineBase* e = h->eng.get();

  // rounded_scaled_residual (solver.cpp:86-92); when u_f is binary64 the same
  // pass also yields true_residual_norm (the reference recomputes it).
  int ex = 0;
  double tnorm = 0.0;
  auto rsr = [&]() {
    OuterA::resid(h, h->d_x, h->d_s, cfg->u_f, cfg->residual_scaling != 0);
    e->scale_round(h->d_s);
    if (cfg->u_f != GADI_DOUBLE) {
      read_state(h);
      const int e_keep = h->h_st->res_e;
      const double rhat_ss = h->h_st->rhat_ss;
      OuterA::resid(h, h->d_x, nullptr, GADI_DOUBLE, false);
      read_state(h);
      tnorm = std::sqrt(h->h_st->res_ss);
      h->h_st->res_e = e_keep;
      h->h_st->rhat_ss = rhat_ss;
      // restore the scaling exponent on the device for k_update
      CK(cudaMemcpyAsync(&h->st->res_e, &h->h_st->res_e, sizeof(int), cudaMemcpyHostToDevice, s));
    } else {
      read_state(h);
      tnorm = std::sqrt(h->h_st->res_ss);
    }
    ex = h->h_st->res_e;
  };
  rsr();
  const double g0 = std::ldexp(std::sqrt(h->h_st->rhat_ss), ex);
  double stop_norm = std::ldexp(g0, -ex);
  const double p_rounded = hround((2.0 - cfg->omega) * cfg->alpha, cfg->u_r);

  double best = 1.0;
  int best_iter = 0;
  for (int k = 0;; ++k) {
    const double rres = h->history.back();
    rep->final_rres = rres;
    rep->outer_iters = k;
    const double gn = std::ldexp(std::sqrt(h->h_st->rhat_ss), ex);
    const bool guard = gn * gn <= g0 * g0 * xi;
    const bool truem = rres * rres <= xi;
    if (guard && truem) { rep->status = GADI_CONVERGED; break; }
    if (guard) { rep->status = GADI_STALLED; break; }
    if (!std::isfinite(rres)) { rep->status = GADI_OVERFLOW_DETECTED; break; }
    if (rres > cfg->divergence_factor) { rep->status = GADI_DIVERGED; break; }
    if (cfg->stall_window > 0) {
      if (rres < best * (1.0 - 1e-3)) {
        best = rres;
        best_iter = k;
      } else if (k - best_iter >= cfg->stall_window) {
        rep->status = GADI_STALLED;
        break;
      }
    }
    if (k >= cfg->max_outer_iters) { rep->status = GADI_MAX_ITERS; break; }

    const double target = cfg->inner.tol_epsilon * stop_norm;
    CK(cudaEventRecord(h->evA, s));
    const int hm = cfg->inner.method;  // solve_H uses the spec method (solver.cpp:212-216)
    InnerOut zo = hm == GADI_INNER_CG ? e->cg(1, e->rhat, e->z, target) : e->gmres(1, e->rhat, e->z, target);
    CK(cudaEventRecord(h->evB, s));
    rep->inner_iter_totals += zo.iters;
    rep->h_iters += zo.iters;
    if (zo.status == INNER_OVERFLOW) { rep->status = GADI_OVERFLOW_DETECTED; break; }
    if (zo.status == INNER_STAGNATED) ++rep->inner_stagnations;
    e->scale_pz(p_rounded);
    // solve_S: a cg request degrades to gmres (solver.cpp:217-221)
    InnerOut yo = e->gmres(2, e->pz, e->y, target);
    rep->inner_iter_totals += yo.iters;
    rep->s_iters += yo.iters;
    {
      float a = 0, b = 0;
      cudaEvent_t evC;
      CK(cudaEventCreate(&evC));
      CK(cudaEventRecord(evC, s));
      CK(cudaEventSynchronize(evC));
      cudaEventElapsedTime(&a, h->evA, h->evB);
      cudaEventElapsedTime(&b, h->evB, evC);
      cudaEventDestroy(evC);
      h_ms += a;
      s_ms += b;
    }
    if (yo.status == INNER_OVERFLOW) { rep->status = GADI_OVERFLOW_DETECTED; break; }
    if (yo.status == INNER_STAGNATED) ++rep->inner_stagnations;

    // x <- x + 2^e y in u (solver.cpp:163-166), non-finite check (:168-174)
    CK(cudaMemsetAsync(&h->st->xbad, 0, 4, s));
    e->update(h->d_x, cfg->u);
    read_state(h);
    if (h->h_st->xbad) {
      OuterA::resid(h, h->d_x, nullptr, GADI_DOUBLE, false);
      read_state(h);
      h->history.push_back(std::sqrt(h->h_st->res_ss) / nt0);
      rep->outer_iters = k + 1;
      rep->final_rres = h->history.back();
      rep->status = GADI_OVERFLOW_DETECTED;
      break;
    }
    rsr();
    stop_norm = std::ldexp(g0, -ex);
    h->history.push_back(tnorm / nt0);
  }
  finish();
}

int fail(const Err& e) {
  g_last_error = e.what();
  return e.code;
}

#define API_BEGIN try {
#define API_END                                \
  }                                            \
  catch (const Err& e) {                       \
    return fail(e);                            \
  }                                            \
  catch (const std::bad_alloc&) {              \
    g_last_error = "host allocation failed";   \
    return GADI_E_OOM;                         \
  }                                            \
  catch (const std::exception& e) {            \
    g_last_error = e.what();                   \
    return GADI_E_CUDA;                        \
  }                                            \
  return GADI_OK;

void upload_rhs(gadi_handle* h, const double* b, cudaMemcpyKind kind) {
  CK(cudaMemcpyAsync(h->d_b, b, h->N * sizeof(double), kind, h->stream));
  h->have_rhs = true;
}

}  // namespace

// ===================================================================== C ABI
extern "C" {

void gadi_config_default(gadi_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->alpha = 1.0;
  c->omega = 1.0;
  c->xi = 0.0;
  c->u_r = c->u = c->u_f = GADI_DOUBLE;
  c->inner.method = GADI_INNER_LU_DIRECT;
  c->inner.tol_epsilon = 1e-2;
  c->inner.max_inner_iters = 1000;
  c->inner.restart = 30;
  c->max_outer_iters = 20000;
  c->divergence_factor = 1e6;
  c->stall_window = 0;
  c->ones_start = 0;
  c->residual_scaling = 1;
  c->accum = GADI_ACCUM_NATIVE;
}

double gadi_default_xi(int32_t u) {
  switch (u) {
    case GADI_DOUBLE: return 1e-26;
    case GADI_SINGLE: return 1e-8;
    default: return 1e-4;
  }
}

const char* gadi_status_name(int32_t s) {
  switch (s) {
    case GADI_CONVERGED: return "Converged";
    case GADI_MAX_ITERS: return "MaxIters";
    case GADI_DIVERGED: return "Diverged";
    case GADI_OVERFLOW_DETECTED: return "OverflowDetected";
    case GADI_SINGULAR_IN_PRECISION: return "SingularInPrecision";
    default: return "Stalled";
  }
}

const char* gadi_last_error(void) { return g_last_error.c_str(); }
int32_t gadi_abi_version(void) { return GADI_ABI_VERSION; }

int gadi_cuda_create(const gadi_problem_desc* d, const gadi_device_opts* opts, gadi_handle** out) {
  API_BEGIN
  if (!d || !out) throw Err(GADI_E_CONTRACT, "gadi_cuda_create: null argument");
  *out = nullptr;
  std::unique_ptr<gadi_handle> h(new gadi_handle());
  h->device = opts ? opts->device : 0;
  CK(cudaSetDevice(h->device));
  h->kind = d->kind;
  if (d->kind == GADI_PROBLEM_STENCIL7) {
    if (d->n < 2) throw Err(GADI_E_CONTRACT, "convdiff3d: n >= 2 required");  // problems.cpp:10
    h->n = d->n;
    h->N = d->n * d->n * d->n;
    h->t1 = d->t1;
    h->t2 = d->t2;
    h->t3 = d->t3;
  } else if (d->kind == GADI_PROBLEM_CSR) {
    const int64_t n = d->n_rows;
    if (n < 1 || !d->row_ptr || !d->col_idx || !d->values) throw Err(GADI_E_CONTRACT, "csr: bad arguments");
    if (n >= (int64_t(1) << 31)) throw Err(GADI_E_UNSUPPORTED, "csr: n_rows must be < 2^31");
    const int64_t* rp = d->row_ptr;
    if (rp[0] != 0 || rp[n] != d->nnz) throw Err(GADI_E_CONTRACT, "row_ptr must start at 0 and end at nnz");
    for (int64_t i = 0; i < n; ++i) {  // sparse.cpp:19-34
      if (rp[i] > rp[i + 1]) throw Err(GADI_E_CONTRACT, "row_ptr must be non-decreasing");
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
        if (d->col_idx[k] < 0 || d->col_idx[k] >= n) throw Err(GADI_E_CONTRACT, "column index out of range");
        if (k > rp[i] && d->col_idx[k] <= d->col_idx[k - 1])
          throw Err(GADI_E_CONTRACT, "column indices must be strictly increasing within a row");
      }
    }
    h->N = n;
    h->nnzA = d->nnz;
    std::vector<int32_t> ci32(d->col_idx, d->col_idx + d->nnz);
    h->d_rpA = dalloc<int64_t>(n + 1);
    h->d_ciA = dalloc<int32_t>(d->nnz);
    h->d_vA = dalloc<double>(d->nnz);
    CK(cudaMemcpy(h->d_rpA, rp, (n + 1) * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->d_ciA, ci32.data(), d->nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->d_vA, d->values, d->nnz * 8, cudaMemcpyHostToDevice));
    HostCsr P;
    hss_split_host(n, rp, d->col_idx, d->values, P, h->Mv, h->Nv, h->diag_in);
    h->nnzHS = P.rp[n];
    h->diag_pos.resize(n);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = P.rp[i]; k < P.rp[i + 1]; ++k)
        if (P.ci[k] == i) h->diag_pos[i] = k;
    std::vector<int32_t> hci(P.ci.begin(), P.ci.end());
    h->d_rpHS = dalloc<int64_t>(n + 1);
    h->d_ciHS = dalloc<int32_t>(h->nnzHS);
    CK(cudaMemcpy(h->d_rpHS, P.rp.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->d_ciHS, hci.data(), h->nnzHS * 4, cudaMemcpyHostToDevice));
  } else {
    throw Err(GADI_E_CONTRACT, "unknown problem kind");
  }
  CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  const int64_t N = h->N;
  h->d_x = dalloc<double>(N);
  h->d_b = dalloc<double>(N);
  h->d_s = dalloc<double>(N);
  h->d_t64 = dalloc<double>(N);
  CK(cudaMemset(h->d_b, 0, N * 8));
  h->st = dalloc<DevState>(1);
  CK(cudaMemset(h->st, 0, sizeof(DevState)));
  CK(cudaHostAlloc(&h->h_st, sizeof(DevState), cudaHostAllocDefault));
  std::memset(h->h_st, 0, sizeof(DevState));
  const int64_t maxblk = std::max<int64_t>(N / 256, 1) + 8;
  h->d_part0 = dalloc<double>(maxblk);
  h->d_part1 = dalloc<double>(maxblk);
  h->d_ticket = dalloc<unsigned>(1);
  CK(cudaMemset(h->d_ticket, 0, sizeof(unsigned)));
  CK(cudaHostAlloc(&h->h_done, sizeof(int), cudaHostAllocMapped));
  *h->h_done = 0;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->d_h_done), h->h_done, 0));
  CK(cudaMemcpy(&h->st->hdone, &h->d_h_done, sizeof(int*), cudaMemcpyHostToDevice));
  CK(cudaEventCreate(&h->ev0));
  CK(cudaEventCreate(&h->ev1));
  CK(cudaEventCreate(&h->evA));
  CK(cudaEventCreate(&h->evB));
  h->ring.resize(4);
  for (auto& ev : h->ring) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  *out = h.release();
  API_END
}

int gadi_cuda_destroy(gadi_handle* h) {
  if (!h) return GADI_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->eng.reset();
  for (void* p : {(void*)h->d_rpA, (void*)h->d_ciA, (void*)h->d_vA, (void*)h->d_rpHS, (void*)h->d_ciHS,
                  (void*)h->d_x, (void*)h->d_b, (void*)h->d_s, (void*)h->d_t64, (void*)h->st,
                  (void*)h->d_part0, (void*)h->d_part1, (void*)h->d_ticket})
    if (p) cudaFree(p);
  if (h->h_st) cudaFreeHost(h->h_st);
  if (h->h_done) cudaFreeHost(h->h_done);
  for (cudaEvent_t ev : {h->ev0, h->ev1, h->evA, h->evB})
    if (ev) cudaEventDestroy(ev);
  for (auto ev : h->ring) cudaEventDestroy(ev);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return GADI_OK;
}

int gadi_cuda_dim(const gadi_handle* h, int64_t* n) {
  if (!h || !n) return GADI_E_CONTRACT;
  *n = h->N;
  return GADI_OK;
}

int gadi_cuda_set_rhs(gadi_handle* h, const double* b) {
  API_BEGIN
  if (!h || !b) throw Err(GADI_E_CONTRACT, "set_rhs: null argument");
  CK(cudaSetDevice(h->device));
  upload_rhs(h, b, cudaMemcpyHostToDevice);
  CK(cudaStreamSynchronize(h->stream));
  API_END
}

int gadi_cuda_residual_uf(gadi_handle* h, int32_t u_f, const double* x, double* s_out) {
  API_BEGIN
  if (!h || !x || !s_out) throw Err(GADI_E_CONTRACT, "residual_uf: null argument");
  if (u_f < 0 || u_f > 2) throw Err(GADI_E_PARAM, "unknown precision");
  CK(cudaSetDevice(h->device));
  CK(cudaMemcpyAsync(h->d_t64, x, h->N * 8, cudaMemcpyHostToDevice, h->stream));
  OuterA::resid(h, h->d_t64, h->d_s, u_f, false);
  CK(cudaMemcpyAsync(s_out, h->d_s, h->N * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  API_END
}

int gadi_cuda_true_residual_norm(gadi_handle* h, const double* x, double* norm_out) {
  API_BEGIN
  if (!h || !x || !norm_out) throw Err(GADI_E_CONTRACT, "true_residual_norm: null argument");
  CK(cudaSetDevice(h->device));
  CK(cudaMemcpyAsync(h->d_t64, x, h->N * 8, cudaMemcpyHostToDevice, h->stream));
  OuterA::resid(h, h->d_t64, nullptr, GADI_DOUBLE, false);
  read_state(h);
  *norm_out = std::sqrt(h->h_st->res_ss);
  API_END
}

int gadi_cuda_prepare(gadi_handle* h, double alpha, double omega, int32_t u_r, const gadi_inner_spec* spec,
                      int32_t accum) {
  API_BEGIN
  if (!h || !spec) throw Err(GADI_E_CONTRACT, "prepare: null argument");
  if (u_r < 0 || u_r > 2) throw Err(GADI_E_PARAM, "unknown precision");
  CK(cudaSetDevice(h->device));
  prepare(h, alpha, omega, u_r, *spec, accum);
  API_END
}

int gadi_cuda_set_inner_stop_norm(gadi_handle* h, double stop_norm) {
  if (!h) return GADI_E_CONTRACT;
  h->stop_norm = stop_norm;
  return GADI_OK;
}

static int inner_call(gadi_handle* h, int which, const double* rhs, double* x_out, int32_t* iters,
                      int32_t* status) {
  API_BEGIN
  if (!h || !rhs || !x_out) throw Err(GADI_E_CONTRACT, "solve: null argument");
  if (!h->eng) throw Err(GADI_E_STATE, "solve_H/solve_S before prepare");
  CK(cudaSetDevice(h->device));
  EngineBase* e = h->eng.get();
  CK(cudaMemcpyAsync(h->d_t64, rhs, h->N * 8, cudaMemcpyHostToDevice, h->stream));
  e->to_inner(h->d_t64, e->rhat);
  const double target = e->spec.tol_epsilon * h->stop_norm;
  InnerOut o;
  if (which == 1 && e->spec.method == GADI_INNER_CG) o = e->cg(1, e->rhat, e->z, target);
  else o = e->gmres(which, e->rhat, e->z, target);
  e->to_double(e->z, h->d_t64);
  CK(cudaMemcpyAsync(x_out, h->d_t64, h->N * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (iters) *iters = o.iters;
  if (status) *status = o.status;
  API_END
}

int gadi_cuda_solve_H(gadi_handle* h, const double* rhs, double* x_out, int32_t* iters, int32_t* status) {
  return inner_call(h, 1, rhs, x_out, iters, status);
}
int gadi_cuda_solve_S(gadi_handle* h, const double* rhs, double* x_out, int32_t* iters, int32_t* status) {
  return inner_call(h, 2, rhs, x_out, iters, status);
}

int gadi_cuda_solve(gadi_handle* h, const gadi_config* cfg, const double* b, const double* x0, double* x_out,
                    gadi_report* rep) {
  API_BEGIN
  if (!h || !cfg || !b || !x_out || !rep) throw Err(GADI_E_CONTRACT, "solve: null argument");
  CK(cudaSetDevice(h->device));
  validate(cfg);
  // timed from the host copy of b to the host copy of x (e2e)
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, h->stream));
  upload_rhs(h, b, cudaMemcpyHostToDevice);
  double h2d = (double)h->N * 8;
  if (x0) {
    CK(cudaMemcpyAsync(h->d_x, x0, h->N * 8, cudaMemcpyHostToDevice, h->stream));
    h2d += (double)h->N * 8;
  } else {
    k_fill<<<ew_grid(h->N), 256, 0, h->stream>>>(h->d_x, cfg->ones_start ? 1.0 : 0.0, h->N);
    CKL();
  }
  run(h, cfg, rep);
  CK(cudaMemcpyAsync(x_out, h->d_x, h->N * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaEventRecord(e1, h->stream));
  CK(cudaEventSynchronize(e1));
  rep->solve_ms = ms_between(e0, e1);
  rep->h2d_bytes = h2d;
  rep->d2h_bytes = (double)h->N * 8;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  API_END
}

int gadi_cuda_solve_device(gadi_handle* h, const gadi_config* cfg, const double* d_b, const double* d_x0,
                           double* d_x, gadi_report* rep) {
  API_BEGIN
  if (!h || !cfg || !d_b || !d_x || !rep) throw Err(GADI_E_CONTRACT, "solve_device: null argument");
  CK(cudaSetDevice(h->device));
  validate(cfg);
  upload_rhs(h, d_b, cudaMemcpyDeviceToDevice);
  if (d_x0) {
    CK(cudaMemcpyAsync(h->d_x, d_x0, h->N * 8, cudaMemcpyDeviceToDevice, h->stream));
  } else {
    k_fill<<<ew_grid(h->N), 256, 0, h->stream>>>(h->d_x, cfg->ones_start ? 1.0 : 0.0, h->N);
    CKL();
  }
  run(h, cfg, rep);
  CK(cudaMemcpyAsync(d_x, h->d_x, h->N * 8, cudaMemcpyDeviceToDevice, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  API_END
}

int gadi_cuda_history(const gadi_handle* h, double* out, int32_t cap) {
  if (!h || (!out && cap > 0)) return GADI_E_CONTRACT;
  const int n = (int)std::min<size_t>(h->history.size(), (size_t)std::max(cap, 0));
  for (int i = 0; i < n; ++i) out[i] = h->history[i];
  return n;
}

int gadi_cuda_apply(gadi_handle* h, int32_t which, const double* x, double* y) {
  API_BEGIN
  if (!h || !x || !y) throw Err(GADI_E_CONTRACT, "apply: null argument");
  CK(cudaSetDevice(h->device));
  CK(cudaMemcpyAsync(h->d_t64, x, h->N * 8, cudaMemcpyHostToDevice, h->stream));
  if (which == 0) {
    OuterA::apply(h, h->d_t64, h->d_s);
    CK(cudaMemcpyAsync(y, h->d_s, h->N * 8, cudaMemcpyDeviceToHost, h->stream));
  } else {
    if (!h->eng) throw Err(GADI_E_STATE, "apply H/S before prepare");
    EngineBase* e = h->eng.get();
    e->to_inner(h->d_t64, e->rhat);
    e->apply(which, e->rhat, e->z);
    e->to_double(e->z, h->d_s);
    CK(cudaMemcpyAsync(y, h->d_s, h->N * 8, cudaMemcpyDeviceToHost, h->stream));
  }
  CK(cudaStreamSynchronize(h->stream));
  API_END
}

static int reduce_test(int32_t device, int32_t p, const double* x, const double* y, int64_t n, double* out,
                       bool norm) {
  API_BEGIN
  if (!x || !out || n < 0) throw Err(GADI_E_CONTRACT, "dot: bad argument");
  if (p < 0 || p > 2) throw Err(GADI_E_PARAM, "unknown precision");
  CK(cudaSetDevice(device));
  if (n == 0) {
    *out = 0.0;
    return GADI_OK;
  }
  std::vector<double> xs(x, x + n), ys;
  double m = 0.0;
  if (norm) {  // norm2 = m * sqrt(pairwise(round(round(x/m)^2))) (kernels.cpp:71-82)
    for (double v : xs)
      if (m < std::fabs(v)) m = std::fabs(v);
    if (m == 0.0 || !std::isfinite(m)) {
      *out = m;
      return GADI_OK;
    }
    for (double& v : xs) v = hround(v / m, p);
    ys = xs;
  } else {
    ys.assign(y, y + n);
  }
  double *dx = dalloc<double>(n), *dy = dalloc<double>(n), *dout = dalloc<double>(1);
  const Geo g = make_geo(n, 1);
  double *p0 = dalloc<double>(g.nblk + 1), *p1 = dalloc<double>(g.nblk + 1);
  unsigned* tk = dalloc<unsigned>(1);
  CK(cudaMemset(tk, 0, 4));
  CK(cudaMemcpy(dx, xs.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dy, ys.data(), n * 8, cudaMemcpyHostToDevice));
  Red rd{p0, p1, tk};
  if (p == GADI_HALF) k_dot_d<__half><<<g.nblk, g.bdim>>>(dx, dy, g, rd, dout);
  else if (p == GADI_SINGLE) k_dot_d<float><<<g.nblk, g.bdim>>>(dx, dy, g, rd, dout);
  else k_dot_d<double><<<g.nblk, g.bdim>>>(dx, dy, g, rd, dout);
  CKL();
  double r = 0;
  CK(cudaMemcpy(&r, dout, 8, cudaMemcpyDeviceToHost));
  for (void* q : {(void*)dx, (void*)dy, (void*)dout, (void*)p0, (void*)p1, (void*)tk}) cudaFree(q);
  *out = norm ? hround(m * hround(std::sqrt(r), p), p) : r;
  API_END
}

int gadi_cuda_dot(int32_t device, int32_t p, const double* x, const double* y, int64_t n, double* out) {
  if (!y) return GADI_E_CONTRACT;
  return reduce_test(device, p, x, y, n, out, false);
}
int gadi_cuda_norm2(int32_t device, int32_t p, const double* x, int64_t n, double* out) {
  return reduce_test(device, p, x, nullptr, n, out, true);
}

int gadi_cuda_make_rhs(gadi_handle* h, uint64_t seed, double lo, double hi, double* d_xtrue, double* d_b) {
  API_BEGIN
  if (!h || !d_xtrue || !d_b) throw Err(GADI_E_CONTRACT, "make_rhs: null argument");
  CK(cudaSetDevice(h->device));
  k_uniform<<<ew_grid(h->N), 256, 0, h->stream>>>(d_xtrue, seed, lo, hi, h->N);
  CKL();
  OuterA::apply(h, d_xtrue, d_b);
  CK(cudaStreamSynchronize(h->stream));
  API_END
}

}  // extern "C"
