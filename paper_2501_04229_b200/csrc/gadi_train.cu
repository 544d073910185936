// gadi_train.cu — GPR training-set generation on the device: alpha_bisection
// and generate_training_set (gpr.cpp:15-68) over the reference's convdiff
// family (build_convdiff3d, problems.cpp:8-43: r = 1/(2n+2), b = A * ones).
//
// Every probe is one full GADI-IR solve with u_r = u = u_f = fmt. The
// reference runs the budget x sizes probes one after another; they are
// independent, so here a pool of host threads runs them concurrently, each
// thread on its own handle and stream (handles are one per host thread,
// gadi_cuda.h), and small-N solves -- launch- and sync-latency bound -- fill
// the device together. The choice is made afterwards in the reference's probe
// order (strictly fewer outer iterations wins, so ties keep the smaller
// alpha), and every probe's solve is the device's bitwise-reference solve, so
// the result is the reference's.
#include <atomic>
#include <climits>
#include <mutex>
#include <thread>

#include "gadi_host.cuh"

using namespace gadi_host;

namespace {

struct Probe {
  int64_t size_param;
  double alpha;
  int status = -1, outer = 0;
};

// The convdiff family member of size parameter n (ConvDiff3DSpec, problems.hpp:16-22).
gadi_problem_desc convdiff_desc(int64_t n) {
  gadi_problem_desc d;
  std::memset(&d, 0, sizeof(d));
  d.kind = GADI_PROBLEM_STENCIL7;
  d.n = n;
  const double r = 1.0 / (2.0 * (double)n + 2.0);
  d.t1 = 6.0;
  d.t2 = -1.0 - r;
  d.t3 = -1.0 + r;
  return d;
}

void check(int rc) {
  if (rc < 0) throw Err(rc, gadi_last_error());
}

// Runs every probe; one handle per worker and size parameter.
void run_probes(std::vector<Probe>& probes, int fmt, const gadi_dichotomy* st, int device, int workers) {
  std::atomic<size_t> next{0};
  std::mutex mu;
  int first_rc = GADI_OK;
  std::string first_msg;
  auto worker = [&]() {
    gadi_handle* h = nullptr;
    int64_t hn = -1;
    double *d_b = nullptr, *d_x = nullptr, *d_xt = nullptr;
    auto drop = [&]() {
      if (h) gadi_cuda_destroy(h);
      for (double* p : {d_b, d_x, d_xt})
        if (p) cudaFree(p);
      h = nullptr;
      d_b = d_x = d_xt = nullptr;
    };
    try {
      CK(cudaSetDevice(device));
      for (;;) {
        const size_t k = next.fetch_add(1);
        if (k >= probes.size()) break;
        Probe& p = probes[k];
        if (p.size_param != hn) {
          drop();
          const gadi_problem_desc d = convdiff_desc(p.size_param);
          gadi_device_opts o{device};
          check(gadi_cuda_create(&d, &o, &h));
          int64_t N = 0;
          gadi_cuda_dim(h, &N);
          d_b = dalloc<double>(N);
          d_x = dalloc<double>(N);
          d_xt = dalloc<double>(N);
          check(gadi_cuda_make_rhs(h, 0, 1.0, 1.0, d_xt, d_b));  // x_exact = ones, b = A x_exact
          hn = p.size_param;
        }
        // gpr.cpp:30-38
        gadi_config cfg;
        gadi_config_default(&cfg);
        cfg.alpha = p.alpha;
        cfg.omega = 1.0;
        cfg.xi = st->train_xi;
        cfg.u_r = cfg.u = cfg.u_f = fmt;
        cfg.inner = st->inner;
        cfg.max_outer_iters = st->max_outer;
        gadi_report rep;
        check(gadi_cuda_solve_device(h, &cfg, d_b, nullptr, d_x, &rep));
        p.status = rep.status;
        p.outer = rep.outer_iters;
      }
    } catch (const Err& e) {
      std::lock_guard<std::mutex> g(mu);
      if (first_rc == GADI_OK) {
        first_rc = e.code;
        first_msg = e.what();
      }
      next = probes.size();
    }
    drop();
  };
  std::vector<std::thread> th;
  for (int w = 0; w < workers; ++w) th.emplace_back(worker);
  for (auto& t : th) t.join();
  if (first_rc != GADI_OK) throw Err(first_rc, first_msg);
}

void check_settings(const gadi_dichotomy* st, int fmt) {
  if (!st) throw Err(GADI_E_CONTRACT, "dichotomy settings: null");
  if (fmt < 0 || fmt > 2) throw Err(GADI_E_PARAM, "unknown precision");
}

// alpha_bisection's grid (gpr.cpp:17-29): budget log-spaced probes.
void add_grid(std::vector<Probe>& probes, int64_t sp, double lo, double hi, int budget) {
  if (!(lo > 0.0) || !(hi > lo)) throw Err(GADI_E_PARAM, "alpha_bisection: need 0 < alpha_lo < alpha_hi");
  if (budget < 3) throw Err(GADI_E_PARAM, "alpha_bisection: budget >= 3 required");
  const double ratio = hi / lo;
  for (int i = 0; i < budget; ++i)
    probes.push_back({sp, lo * std::pow(ratio, (double)i / (double)(budget - 1))});
}

// The reference's choice over one size's probes, in probe order (gpr.cpp:39-49).
void choose(const Probe* p, int budget, double lo, double hi, double* alpha, int32_t* iters) {
  double best_alpha = 0.0;
  long long best = LLONG_MAX;
  for (int i = 0; i < budget; ++i)
    if (p[i].status == GADI_CONVERGED && (long long)p[i].outer < best) {
      best = p[i].outer;
      best_alpha = p[i].alpha;
    }
  if (best_alpha == 0.0)
    throw Err(GADI_E_NO_CONVERGENT_ALPHA, "no alpha in [" + std::to_string(lo) + ", " + std::to_string(hi) +
                                              "] converged at size " + std::to_string(p[0].size_param));
  *alpha = best_alpha;
  *iters = (int32_t)best;
}

int pool_size(size_t tasks) {
  const char* e = std::getenv("GADI_TRAIN_WORKERS");
  const int w = e ? std::atoi(e) : 16;
  return (int)std::max<size_t>(1, std::min<size_t>(tasks, (size_t)std::max(w, 1)));
}

}  // namespace

extern "C" {

void gadi_dichotomy_default(gadi_dichotomy* st) {
  // DichotomySettings, gpr.hpp:37-44 (InnerSolverSpec{} inner: lu_direct)
  std::memset(st, 0, sizeof(*st));
  st->alpha_lo = 1e-2;
  st->alpha_hi = 1e2;
  st->budget = 21;
  st->train_xi = 1e-8;
  st->max_outer = 1500;
  st->inner.method = GADI_INNER_LU_DIRECT;
  st->inner.tol_epsilon = 1e-2;
  st->inner.max_inner_iters = 1000;
  st->inner.restart = 30;
}

int gadi_alpha_bisection(int64_t size_param, int32_t fmt, double alpha_lo, double alpha_hi, int32_t budget,
                         const gadi_dichotomy* st, int32_t device, double* alpha, int32_t* iters) {
  try {
    check_settings(st, fmt);
    if (!alpha || !iters) throw Err(GADI_E_CONTRACT, "alpha_bisection: null output");
    if (size_param < 2) throw Err(GADI_E_CONTRACT, "convdiff3d: n >= 2 required");
    std::vector<Probe> probes;
    add_grid(probes, size_param, alpha_lo, alpha_hi, budget);
    run_probes(probes, fmt, st, device, pool_size(probes.size()));
    choose(probes.data(), budget, alpha_lo, alpha_hi, alpha, iters);
  } catch (const Err& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GADI_E_CUDA;
  }
  return GADI_OK;
}

int gadi_generate_training_set(const int64_t* size_params, int32_t count, int32_t fmt, const gadi_dichotomy* st,
                               int32_t device, int64_t* size_n, double* alpha, int32_t* iters) {
  try {
    check_settings(st, fmt);
    if (count < 0 || (count > 0 && (!size_params || !size_n || !alpha || !iters)))
      throw Err(GADI_E_CONTRACT, "generate_training_set: bad arguments");
    for (int32_t s = 0; s < count; ++s)
      if (size_params[s] < 2) throw Err(GADI_E_CONTRACT, "convdiff3d: n >= 2 required");
    // all sizes' probes in one pool (gpr.cpp:56-63 runs them size by size)
    std::vector<Probe> probes;
    for (int32_t s = 0; s < count; ++s) add_grid(probes, size_params[s], st->alpha_lo, st->alpha_hi, st->budget);
    run_probes(probes, fmt, st, device, pool_size(probes.size()));
    struct Pair {
      int64_t n;
      double a;
      int32_t it;
    };
    std::vector<Pair> pairs(count);
    for (int32_t s = 0; s < count; ++s) {
      pairs[s].n = size_params[s] * size_params[s] * size_params[s];  // builder(sp).A.n_rows()
      choose(probes.data() + (size_t)s * st->budget, st->budget, st->alpha_lo, st->alpha_hi, &pairs[s].a,
             &pairs[s].it);
    }
    std::stable_sort(pairs.begin(), pairs.end(), [](const Pair& a, const Pair& b) { return a.n < b.n; });
    for (size_t i = 1; i < pairs.size(); ++i)
      if (pairs[i].n == pairs[i - 1].n) throw Err(GADI_E_PARAM, "generate_training_set: duplicate sizes");
    for (int32_t s = 0; s < count; ++s) {
      size_n[s] = pairs[s].n;
      alpha[s] = pairs[s].a;
      iters[s] = pairs[s].it;
    }
  } catch (const Err& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GADI_E_CUDA;
  }
  return GADI_OK;
}

}  // extern "C"
