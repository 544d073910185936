// The reference's plugin boundary driven by the B200 library: a
// gadi::GadiSystem (solver.hpp:74-89) whose six virtuals call the C ABI in
// include/gadi_cuda.h, so the REFERENCE's own run_gadi_ir (solver.cpp:57-179)
// runs its outer loop over device-resident operators and inner solvers.
//
// This is the binding a maintainer of the reference would add (INTEGRATION.md
// walks through it). It is built against the reference headers into
// oracle/_ref/ by oracle/Makefile.ref and exercised by
// tests/test_gpu_integration.py; it is test/integration code, not product.
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

#include "gadi/errors.hpp"
#include "gadi/solver.hpp"
#include "gadi_cuda.h"

namespace gadi {
namespace cuda {

// Error codes back to the reference's exception types (errors.hpp:9-45).
inline void check(int rc) {
  if (rc >= 0) return;
  const std::string msg = gadi_last_error();
  switch (rc) {
    case GADI_E_PARAM: throw ParameterError(msg);
    case GADI_E_CONTRACT: throw ContractViolation(msg);
    case GADI_E_UNSUPPORTED: throw ParameterError("unsupported on the device: " + msg);
    case GADI_E_SINGULAR: throw SingularInPrecision(msg);  // prepare, band_lu.cpp:106-108
    case GADI_E_OVERFLOW: throw OverflowDetected(msg);     // prepare, band_lu.cpp:132-134
    default: throw std::runtime_error("gadi_cuda error " + std::to_string(rc) + ": " + msg);
  }
}

class CudaGadiSystem final : public GadiSystem {
 public:
  explicit CudaGadiSystem(const gadi_problem_desc& d, const Vector& b, int device = 0) {
    gadi_device_opts o{device};
    check(gadi_cuda_create(&d, &o, &h_));
    int64_t n = 0;
    gadi_cuda_dim(h_, &n);
    n_ = n;
    check(gadi_cuda_set_rhs(h_, b.data()));
  }
  ~CudaGadiSystem() override { gadi_cuda_destroy(h_); }

  index_t dim() const override { return n_; }

  Vector residual_uf(const Vector& x, RoundingStats&) const override {
    Vector s(n_);
    check(gadi_cuda_residual_uf(h_, static_cast<int32_t>(u_f_), x.data(), s.data()));
    return s;
  }
  double true_residual_norm(const Vector& x) const override {
    double r = 0.0;
    check(gadi_cuda_true_residual_norm(h_, x.data(), &r));
    return r;
  }
  void prepare(double alpha, double omega, Precision u_r, const InnerSolverSpec& spec, RoundingStats&) override {
    gadi_inner_spec s{static_cast<int32_t>(spec.method), spec.tol_epsilon, spec.max_inner_iters, spec.restart};
    check(gadi_cuda_prepare(h_, alpha, omega, static_cast<int32_t>(u_r), &s, accum_));
  }
  void set_inner_stop_norm(double s) override { check(gadi_cuda_set_inner_stop_norm(h_, s)); }
  InnerResult solve_H(const Vector& rhat, RoundingStats&) override { return inner(rhat, true); }
  InnerResult solve_S(const Vector& pz, RoundingStats&) override { return inner(pz, false); }

  void set_u_f(Precision p) { u_f_ = p; }

 private:
  InnerResult inner(const Vector& rhs, bool h) {
    InnerResult r;
    r.x.resize(n_);
    int32_t it = 0, st = 0;
    check(h ? gadi_cuda_solve_H(h_, rhs.data(), r.x.data(), &it, &st)
            : gadi_cuda_solve_S(h_, rhs.data(), r.x.data(), &it, &st));
    r.iters = it;
    r.status = static_cast<InnerStatus>(st);
    return r;
  }
  gadi_handle* h_ = nullptr;
  index_t n_ = 0;
  Precision u_f_ = Precision::Double;
  int32_t accum_ = GADI_ACCUM_NATIVE;
};

}  // namespace cuda
}  // namespace gadi

extern "C" {

// The reference's run_gadi_ir over CudaGadiSystem on the convdiff stencil
// (t1, t2, t3 as in problems.hpp:16-22). Returns 0 or a gadi_error.
int refcuda_solve_stencil(int64_t n, double t1, double t2, double t3, const double* b, const gadi_config* c,
                          double* x, double* hist, int cap, gadi_report* rep) {
  using namespace gadi;
  try {
    gadi_problem_desc d{};
    d.kind = GADI_PROBLEM_STENCIL7;
    d.n = n;
    d.t1 = t1;
    d.t2 = t2;
    d.t3 = t3;
    const index_t N = n * n * n;
    Vector bv(b, b + N);
    cuda::CudaGadiSystem sys(d, bv);
    GadiConfig cfg;
    cfg.alpha = c->alpha;
    cfg.omega = c->omega;
    cfg.xi = c->xi;
    cfg.u_r = static_cast<Precision>(c->u_r);
    cfg.u = static_cast<Precision>(c->u);
    cfg.u_f = static_cast<Precision>(c->u_f);
    cfg.inner.method = static_cast<InnerMethod>(c->inner.method);
    cfg.inner.tol_epsilon = c->inner.tol_epsilon;
    cfg.inner.max_inner_iters = c->inner.max_inner_iters;
    cfg.inner.restart = c->inner.restart;
    cfg.max_outer_iters = c->max_outer_iters;
    cfg.divergence_factor = c->divergence_factor;
    cfg.stall_window = c->stall_window;
    cfg.ones_start = c->ones_start != 0;
    cfg.residual_scaling = c->residual_scaling != 0;
    sys.set_u_f(cfg.u_f);
    Vector x0(N, cfg.ones_start ? 1.0 : 0.0);
    GadiResult res = run_gadi_ir(sys, cfg, x0);
    std::memcpy(x, res.x.data(), N * sizeof(double));
    std::memset(rep, 0, sizeof(*rep));
    rep->status = static_cast<int>(res.report.status);
    rep->outer_iters = res.report.outer_iters;
    rep->final_rres = res.report.final_rres;
    rep->inner_iter_totals = res.report.inner_iter_totals;
    rep->inner_stagnations = res.report.inner_stagnations;
    rep->history_len = static_cast<int>(res.report.rel_residual_history.size());
    for (int i = 0; i < rep->history_len && i < cap; ++i) hist[i] = res.report.rel_residual_history[i];
    return 0;
  } catch (const ParameterError&) {
    return GADI_E_PARAM;
  } catch (const ContractViolation&) {
    return GADI_E_CONTRACT;
  } catch (...) {
    return -99;
  }
}

}  // extern "C"
