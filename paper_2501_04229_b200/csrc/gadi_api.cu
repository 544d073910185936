// gadi_api.cu — run_gadi_ir on the device and the C ABI (include/gadi_cuda.h).
#include <thread>

#include "gadi_host.cuh"

using namespace gadi_host;

namespace gadi_host {
void set_last_error(const std::string& m) { g_last_error = m; }
}  // namespace gadi_host

namespace {

// hss_split on the device (splitting.cpp:12-20; gadi_csr.cuh): A^T by column
// counts + scan + scatter + per-row sort, then the per-row union of A, A^T and
// the diagonal with M = (A+A^T)/2, N = (A-A^T)/2 in binary64; plus the SELL
// image of A (binary64, 2 rows per lane) for the outer residual.
void device_split(gadi_handle* h) {
  cudaStream_t s = h->stream;
  const int64_t N = h->N, nnz = h->nnzA;
  const dim3 gN = ew_grid(N), gZ = ew_grid(nnz);
  int* cnt = dalloc<int>(N + 1);
  CK(cudaMemsetAsync(cnt, 0, (N + 1) * sizeof(int), s));
  k_count_cols<<<gZ, 256, 0, s>>>(h->d_ciA, nnz, cnt);
  int64_t* c64 = dalloc<int64_t>(N + 1);
  k_i32_to_i64<<<ew_grid(N + 1), 256, 0, s>>>(cnt, c64, N + 1);
  CKL();
  int64_t* trp = dalloc<int64_t>(N + 1);
  scan_i64(s, c64, trp, N + 1);
  unsigned long long* next = dalloc<unsigned long long>(N);
  CK(cudaMemcpyAsync(next, trp, N * 8, cudaMemcpyDeviceToDevice, s));
  int32_t* tci = dalloc<int32_t>(nnz);
  double* tv = dalloc<double>(nnz);
  k_scatter_t<<<gN, 256, 0, s>>>(N, h->d_rpA, h->d_ciA, h->d_vA, next, tci, tv);
  k_sort_rows<<<gN, 256, 0, s>>>(N, trp, tci, tv);
  // union pattern: count, scan, fill
  k_union<false><<<gN, 256, 0, s>>>(N, h->d_rpA, h->d_ciA, h->d_vA, trp, tci, tv, c64, nullptr, nullptr, nullptr,
                                    nullptr, nullptr, nullptr);
  CKL();
  CK(cudaMemsetAsync(c64 + N, 0, 8, s));
  h->d_urp = dalloc<int64_t>(N + 1);
  scan_i64(s, c64, h->d_urp, N + 1);
  CK(cudaMemcpy(&h->nnzHS, h->d_urp + N, 8, cudaMemcpyDeviceToHost));
  h->d_uci = dalloc<int32_t>(h->nnzHS);
  h->d_mv = dalloc<double>(h->nnzHS);
  h->d_nv = dalloc<double>(h->nnzHS);
  h->d_dpos = dalloc<int64_t>(N);
  h->d_din = dalloc<uint8_t>(N);
  k_union<true><<<gN, 256, 0, s>>>(N, h->d_rpA, h->d_ciA, h->d_vA, trp, tci, tv, nullptr, h->d_urp, h->d_uci,
                                   h->d_mv, h->d_nv, h->d_dpos, h->d_din);
  CKL();
  CK(cudaStreamSynchronize(s));
  for (void* p : {(void*)cnt, (void*)c64, (void*)trp, (void*)next, (void*)tci, (void*)tv}) cudaFree(p);
  h->launches += 7;
}

// SELL image of A for the binary64 residual (2 rows per lane: 16-byte loads)
void build_sell_A(gadi_handle* h) {
  build_sell_layout(h->stream, h->N, ilog2(64), h->d_rpA, h->d_ciA, h->sellA, h->max_band < 32768);
  h->sellA.val = fill_sell_values<double, P_DOUBLE>(h->stream, h->N, h->sellA, h->d_rpA, h->d_vA, nullptr, nullptr,
                                                    0.0);
}

// A CSR row block (sharded solves): the split ran on the window [lo, hi)^2
// around the block; keep rows [a, b) of A and of the union pattern, columns
// renumbered relative to row a (the block's first row: negative columns and
// columns >= b - a address the ghost entries of the shard vectors).
void crop_rows(gadi_handle* h, int64_t a, int64_t b) {
  cudaStream_t s = h->stream;
  const int64_t m = b - a;
  auto crop = [&](int64_t*& rp, int32_t*& ci, std::vector<double**> vals, int64_t& nnz, int64_t* first) {
    int64_t pa = 0, pb = 0;
    CK(cudaMemcpy(&pa, rp + a, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&pb, rp + b, 8, cudaMemcpyDeviceToHost));
    int64_t* nrp = dalloc<int64_t>(m + 1);
    k_sub_i64<<<ew_grid(m + 1), 256, 0, s>>>(rp + a, nrp, m + 1, pa);
    int32_t* nci = dalloc<int32_t>(pb - pa);
    k_sub_i32<<<ew_grid(pb - pa), 256, 0, s>>>(ci + pa, nci, pb - pa, (int32_t)a);
    CKL();
    for (double** v : vals) {
      double* nv = dalloc<double>(pb - pa);
      CK(cudaMemcpyAsync(nv, *v + pa, (pb - pa) * 8, cudaMemcpyDeviceToDevice, s));
      CK(cudaStreamSynchronize(s));
      cudaFree(*v);
      *v = nv;
    }
    CK(cudaStreamSynchronize(s));
    cudaFree(rp);
    cudaFree(ci);
    rp = nrp;
    ci = nci;
    nnz = pb - pa;
    *first = pa;
  };
  int64_t pa = 0, ua = 0;
  crop(h->d_rpA, h->d_ciA, {&h->d_vA}, h->nnzA, &pa);
  crop(h->d_urp, h->d_uci, {&h->d_mv, &h->d_nv}, h->nnzHS, &ua);
  int64_t* ndp = dalloc<int64_t>(m);
  k_sub_i64<<<ew_grid(m), 256, 0, s>>>(h->d_dpos + a, ndp, m, ua);
  uint8_t* ndi = dalloc<uint8_t>(m);
  CK(cudaMemcpyAsync(ndi, h->d_din + a, m, cudaMemcpyDeviceToDevice, s));
  CKL();
  CK(cudaStreamSynchronize(s));
  cudaFree(h->d_dpos);
  cudaFree(h->d_din);
  h->d_dpos = ndp;
  h->d_din = ndi;
  h->N = m;
}

EngineBase* make_engine(gadi_handle* h, const gadi_inner_spec& sp, double a, double om, int ur, int acc) {
  const bool st = h->stencil();
  if (ur == GADI_DOUBLE) return (st ? make_engine_st_d64 : make_engine_csr_d64)(h, sp, a, om, ur, acc);
  if (ur == GADI_SINGLE) return (st ? make_engine_st_f32 : make_engine_csr_f32)(h, sp, a, om, ur, acc);
  if (acc == GADI_ACCUM_FP32) return (st ? make_engine_st_h32 : make_engine_csr_h32)(h, sp, a, om, ur, acc);
  return (st ? make_engine_st_h16 : make_engine_csr_h16)(h, sp, a, om, ur, acc);
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
  if (c->inner.method != GADI_INNER_LU_DIRECT && c->inner.method != GADI_INNER_CG &&
      c->inner.method != GADI_INNER_GMRES)
    throw Err(GADI_E_PARAM, "unknown inner method");
  if (c->accum != GADI_ACCUM_NATIVE && c->accum != GADI_ACCUM_FP32) throw Err(GADI_E_PARAM, "unknown accum");
}

// prepare threw SingularInPrecision / OverflowDetected (the LuDirect
// factorizations, inner_solver.cpp:27-34 -> band_lu.cpp:106-108,132-134);
// run_gadi_ir turns it into the solve status (solver.cpp:74-82).
struct PrepareStatus {
  int status;
};

// Factor H then S in u_r when the method is LuDirect (solver.cpp:204-207).
void lu_factors(gadi_handle* h, EngineBase* e) {
  for (int which : {1, 2}) {
    if (e->lu[which]) continue;
    int st = 0;
    e->lu[which] = lu_factor_build(h, which, e->alpha, e->u_r, &st);
    h->launches += e->lu[which]->launches;
    if (st != 0) {
      lu_release(e->lu[which], h->stream);
      e->lu[which] = nullptr;
      throw PrepareStatus{st};
    }
  }
}

void prepare(gadi_handle* h, double alpha, double omega, int ur, const gadi_inner_spec& sp, int accum) {
  if (!(alpha > 0.0)) throw Err(GADI_E_PARAM, "regularize: alpha must be positive");
  if (!(omega >= 0.0 && omega < 2.0)) throw Err(GADI_E_PARAM, "regularize: omega must be in [0, 2)");
  if (sp.method != GADI_INNER_LU_DIRECT && sp.method != GADI_INNER_CG && sp.method != GADI_INNER_GMRES)
    throw Err(GADI_E_PARAM, "unknown inner method");
  if (sp.method == GADI_INNER_LU_DIRECT && h->sharded())
    throw Err(GADI_E_UNSUPPORTED, "lu_direct: not on a shard (the band LU is one device)");
  if (accum != GADI_ACCUM_NATIVE && accum != GADI_ACCUM_FP32) throw Err(GADI_E_PARAM, "unknown accum");
  if (sp.restart > 64) throw Err(GADI_E_UNSUPPORTED, "gmres restart > 64");
  auto& e = h->eng;
  const bool same = e && e->u_r == ur && e->accum == accum && std::max(1, e->spec.restart) == std::max(1, sp.restart);
  if (!(same && e->alpha == alpha && e->omega == omega)) {
    if (same && e->set_alpha(alpha, omega)) {
      for (LuFactor*& f : e->lu) {  // factors of the previous alpha
        lu_release(f, h->stream);
        f = nullptr;
      }
    } else {
      e.reset();
      CK(cudaStreamSynchronize(h->stream));
      e.reset(make_engine(h, sp, alpha, omega, ur, accum));
    }
  }
  e->spec = sp;
  if (sp.method == GADI_INNER_LU_DIRECT) lu_factors(h, e.get());
}

// solve_H / solve_S through LuDirect (solver.cpp:226-231)
InnerOut lu_solve(gadi_handle* h, EngineBase* e, int which, const void* rhs, void* x) {
  const int64_t l0 = e->lu[which]->launches;
  InnerOut o = lu_inner_solve(e->lu[which], rhs, x, h->stream);
  h->launches += e->lu[which]->launches - l0;
  return o;
}

double ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// run_gadi_ir (solver.cpp:57-179) on the device vectors h->d_b and h->d_x
// (x0, rounded to u below).
void run(gadi_handle* h, const gadi_config* cfg, gadi_report* rep) {
  validate(cfg);
  const double xi = cfg->xi > 0.0 ? cfg->xi : gadi_default_xi(cfg->u);
  const int64_t launches0 = h->launches;
  std::memset(rep, 0, sizeof(*rep));
  rep->status = GADI_MAX_ITERS;
  rep->final_rres = 1.0;
  h->history.assign(1, 1.0);
  cudaStream_t s = h->stream;
  const int64_t N = h->N;
  CK(cudaEventRecord(h->ev0, s));
  double h_ms = 0, s_ms = 0;

  // x = round_vec(x0, u) (solver.cpp:65)
  {
    auto L = [&](auto pt) {
      constexpr int P = decltype(pt)::v;
      k_convert<double, double, P><<<ew_grid(N), 256, 0, s>>>(h->d_x, h->d_x, N);
      ++h->launches;
    };
    if (cfg->u == GADI_HALF) L(VecTag<P_HALF>{});
    else if (cfg->u == GADI_SINGLE) L(VecTag<P_SINGLE>{});
    CKL();
  }
  // nt0 = true_residual_norm(x) (solver.cpp:67)
  h->ns = 0;
  OuterA::resid_sync(h, h->d_x, nullptr, GADI_DOUBLE, false);
  const double nt0 = res_norm(h);
  auto finish = [&]() {
    CK(cudaEventRecord(h->ev1, s));
    CK(cudaEventSynchronize(h->ev1));
    rep->solve_ms = ms_between(h->ev0, h->ev1);
    rep->h_ms = h_ms;
    rep->s_ms = s_ms;
    rep->outer_ms = rep->solve_ms - h_ms - s_ms;
    rep->history_len = (int)h->history.size();
    rep->launches = h->launches - launches0;
  };
  if (nt0 == 0.0) {
    rep->status = GADI_CONVERGED;
    rep->final_rres = 0.0;
    finish();
    return;
  }
  try {
    prepare(h, cfg->alpha, cfg->omega, cfg->u_r, cfg->inner, cfg->accum);
  } catch (const PrepareStatus& ps) {  // solver.cpp:74-82
    rep->status = ps.status;
    finish();
    return;
  }
  EngineBase* e = h->eng.get();
  const bool lu = cfg->inner.method == GADI_INNER_LU_DIRECT;

  // rounded_scaled_residual (solver.cpp:86-92); when u_f is binary64 the same
  // pass also yields true_residual_norm (the reference recomputes it).
  int ex = 0;
  double tnorm = 0.0, rhat_n = 0.0;  // ||b - A x||_2 and ||rhat||_2 (in the scaled frame), binary64
  bool rhat_ss_at0 = false;          // st->rhat_ss = sum of rhat^2 unscaled (ns_r = 0): what k_cg_init would reduce
  // spec: when u_f is binary64, first try the single pass that also rounds
  // rhat with the previous step's exponent (accepted iff the exponent is
  // unchanged -- the usual case; else the two-pass route below reruns).
  const bool trace = std::getenv("GADI_TRACE") != nullptr;
  cudaEvent_t trU = nullptr, trR = nullptr, trR0 = nullptr, trK = nullptr, trX = nullptr;
  double tr_gap = 0.0, tr_upd = 0.0, tr_res = 0.0, tr_kern = 0.0, tr_wake = 0.0;
  if (trace) {
    CK(cudaEventCreate(&trU));
    CK(cudaEventCreate(&trR));
    CK(cudaEventCreate(&trR0));
    CK(cudaEventCreate(&trK));
    CK(cudaEventCreate(&trX));
  }
  const bool can_spec = cfg->u_f == GADI_DOUBLE && !std::getenv("GADI_NO_SPEC");
  auto rsr = [&](bool spec) {
    const bool sc = cfg->residual_scaling != 0;
    if (spec && can_spec && e->resid_spec(h->d_x, ex, sc)) {
      const int ns_r = sc ? 0 : h->ns;
      if (trace) CK(cudaEventRecord(trK, s));
      read_state(h);
      if (trace) CK(cudaEventRecord(trX, s));
      if (res_norm_ok(h) && h->h_st->res_e == ex) {
        rhat_n = std::ldexp(std::sqrt(h->h_st->rhat_ss), ns_r);
        tnorm = res_norm(h);
        rhat_ss_at0 = ns_r == 0;
        return;
      }
    }
    OuterA::resid_sync(h, h->d_x, h->d_s, cfg->u_f, sc);
    const int ns_r = sc ? 0 : h->ns;
    e->scale_round(h->d_s, ns_r);
    read_state(h);
    ex = h->h_st->res_e;
    rhat_n = std::ldexp(std::sqrt(h->h_st->rhat_ss), ns_r);
    rhat_ss_at0 = ns_r == 0;
    if (cfg->u_f != GADI_DOUBLE) {
      OuterA::resid_sync(h, h->d_x, nullptr, GADI_DOUBLE, false);
      tnorm = res_norm(h);
      // keep the scaling exponent of the u_f residual on the device for k_update
      h->h_st->res_e = ex;
      CK(cudaMemcpyAsync(&h->st->res_e, &h->h_st->res_e, sizeof(int), cudaMemcpyHostToDevice, s));
    } else {
      tnorm = res_norm(h);
    }
  };
  rsr(false);
  const double g0 = std::ldexp(rhat_n, ex);
  double stop_norm = std::ldexp(g0, -ex);
  const double p_rounded = hround((2.0 - cfg->omega) * cfg->alpha, cfg->u_r);

  double best = 1.0;
  int best_iter = 0;
  for (int k = 0;; ++k) {
    const double rres = h->history.back();
    rep->final_rres = rres;
    rep->outer_iters = k;
    const double gn = std::ldexp(rhat_n, ex);
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
    // solve_H uses the spec method (solver.cpp:212-216)
    // rhat's binary64 sum of squares is on the device from the pass that produced it (rsr)
    e->rhs_ss_known = !lu && cfg->inner.method == GADI_INNER_CG && rhat_ss_at0;
    InnerOut zo = lu                                  ? lu_solve(h, e, 1, e->rhat, e->z)
                  : cfg->inner.method == GADI_INNER_CG ? e->cg(1, e->rhat, e->z, target)
                                                       : e->gmres(1, e->rhat, e->z, target);
    e->rhs_ss_known = false;
    CK(cudaEventRecord(h->evB, s));
    rep->inner_iter_totals += zo.iters;
    rep->h_iters += zo.iters;
    if (zo.status == INNER_OVERFLOW) { rep->status = GADI_OVERFLOW_DETECTED; break; }
    if (zo.status == INNER_STAGNATED) ++rep->inner_stagnations;
    if (lu) e->scale_pz(p_rounded);
    else e->defer_pz(p_rounded);  // formed inside the GMRES zero-start residual pass
    // solve_S: a cg request degrades to gmres (solver.cpp:217-221)
    InnerOut yo = lu ? lu_solve(h, e, 2, e->pz, e->y) : e->gmres(2, e->pz, e->y, target);
    CK(cudaEventRecord(h->evC, s));
    rep->inner_iter_totals += yo.iters;
    rep->s_iters += yo.iters;
    if (yo.status == INNER_OVERFLOW) { rep->status = GADI_OVERFLOW_DETECTED; break; }
    if (yo.status == INNER_STAGNATED) ++rep->inner_stagnations;

    // x <- x + 2^e y in u (solver.cpp:163-166), non-finite check (:168-174)
    CK(cudaMemsetAsync(&h->st->xbad, 0, 4, s));
    e->update(h->d_x, cfg->u);
    if (trace) CK(cudaEventRecord(trU, s));
    rsr(true);  // syncs: also closes the H/S timing events
    h_ms += ms_between(h->evA, h->evB);
    s_ms += ms_between(h->evB, h->evC);
    if (trace) {  // GADI_TRACE: where the outer part of a step goes (measurement only)
      CK(cudaEventRecord(trR, s));
      CK(cudaEventSynchronize(trR));
      if (k > 0) tr_gap += ms_between(trR0, h->evA);
      tr_upd += ms_between(h->evC, trU);
      tr_res += ms_between(trU, trR);
      if (cudaEventQuery(trK) == cudaSuccess && k > 2) {
        tr_kern += ms_between(trU, trK);
        tr_wake += ms_between(trK, trX);
      }
      std::swap(trR, trR0);
    }
    if (h->h_st->xbad) {
      OuterA::resid_sync(h, h->d_x, nullptr, GADI_DOUBLE, false);
      h->history.push_back(res_norm(h) / nt0);
      rep->outer_iters = k + 1;
      rep->final_rres = h->history.back();
      rep->status = GADI_OVERFLOW_DETECTED;
      break;
    }
    stop_norm = std::ldexp(g0, -ex);
    h->history.push_back(tnorm / nt0);
  }
  if (trace) {
    std::fprintf(stderr, "[gadi trace] outer steps %d: update %.3f ms, residual pass + sync %.3f ms, host gap before the next step %.3f ms; from step 3 on: residual kernel %.3f ms, copy + host wake-up %.3f ms (totals)\n",
                 rep->outer_iters, tr_upd, tr_res, tr_gap, tr_kern, tr_wake);
    cudaEventDestroy(trK);
    cudaEventDestroy(trX);
    cudaEventDestroy(trU);
    cudaEventDestroy(trR);
    cudaEventDestroy(trR0);
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

// One device's part of a problem: the whole problem (grp == nullptr) or the
// z-slab `rank` of a sharded stencil solve over grp (gadi_dist.cuh).
static gadi_handle* create_impl(const gadi_problem_desc* d, const gadi_device_opts* opts, gadi_group* grp,
                                int rank) {
  if (!d) throw Err(GADI_E_CONTRACT, "gadi_cuda_create: null argument");
  std::unique_ptr<gadi_handle> h(new gadi_handle());
  h->device = opts ? opts->device : 0;
  CK(cudaSetDevice(h->device));
  h->kind = d->kind;
  // sharded CSR / band problems: rank's row block [r0, r1) of N/world rows;
  // the split runs on the window [lo, hi) = the block +- the band
  int64_t r0 = 0, r1 = 0, lo = 0, hi = 0;
  if (grp) {
    const int w = grp->world;
    if (w < 1 || w > GADI_MAX_RANKS || (w & (w - 1)) != 0)
      throw Err(GADI_E_PARAM, "sharded solves: world must be a power of two <= 64");
    if (rank < 0 || rank >= w) throw Err(GADI_E_PARAM, "sharded solves: rank out of range");
    if (d->kind == GADI_PROBLEM_STENCIL7 && d->n % w != 0)
      throw Err(GADI_E_PARAM, "sharded solves: world must divide n");
    if (d->kind != GADI_PROBLEM_STENCIL7 && (d->n_rows < w || d->n_rows % w != 0))
      throw Err(GADI_E_PARAM, "sharded solves: world must divide n_rows");
    if (grp->nccl_rank >= 0 && grp->nccl_rank != rank)
      throw Err(GADI_E_PARAM, "sharded solves: an NCCL group holds this process's rank only");
    h->world = w;
    h->rank = rank;
    if (d->kind != GADI_PROBLEM_STENCIL7) {
      const int64_t m = d->n_rows / w;
      r0 = rank * m;
      r1 = r0 + m;
    }
  }
  auto set_window = [&](int64_t N, int64_t band) {
    if (band > r1 - r0) throw Err(GADI_E_UNSUPPORTED, "sharded solves: the band exceeds a row block (fewer ranks)");
    lo = std::max<int64_t>(0, r0 - band);
    hi = std::min<int64_t>(N, r1 + band);
  };
  if (d->kind == GADI_PROBLEM_STENCIL7) {
    if (d->n < 2) throw Err(GADI_E_CONTRACT, "convdiff3d: n >= 2 required");  // problems.cpp:10
    h->n = d->n;
    h->N = d->n * d->n * d->n;
    h->t1 = d->t1;
    h->t2 = d->t2;
    h->t3 = d->t3;
    h->i0 = 0;
    h->i1 = d->n;
    if (grp) {
      const int64_t np = d->n / grp->world;
      h->world = grp->world;
      h->rank = rank;
      h->i0 = rank * np;
      h->i1 = h->i0 + np;
      h->N = d->n * d->n * np;
      h->gh = d->n * d->n;
      if (grp->local)
        h->comm.reset(new LocalComm(grp->local.get(), rank));
      else if (grp->ipc)
        h->comm.reset(new IpcComm(grp->ipc.get(), (size_t)h->gh * 8));
      else
        h->comm.reset(new NcclComm(grp->world, rank, grp->id));
    }
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
    h->max_band = 0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
        h->max_band = std::max<int64_t>(h->max_band, std::llabs(d->col_idx[k] - i));
    std::vector<int64_t> rpw;
    std::vector<int32_t> ci32;
    std::vector<double> vw;
    if (grp) {  // the window [lo, hi)^2 around this rank's row block, columns shifted by -lo
      set_window(n, h->max_band);
      rpw.push_back(0);
      for (int64_t i = lo; i < hi; ++i) {
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
          if (d->col_idx[k] >= lo && d->col_idx[k] < hi) {
            ci32.push_back((int32_t)(d->col_idx[k] - lo));
            vw.push_back(d->values[k]);
          }
        rpw.push_back((int64_t)ci32.size());
      }
    } else {
      rpw.assign(rp, rp + n + 1);
      ci32.assign(d->col_idx, d->col_idx + d->nnz);
      vw.assign(d->values, d->values + d->nnz);
    }
    h->N = (int64_t)rpw.size() - 1;
    h->nnzA = (int64_t)ci32.size();
    h->d_rpA = dalloc<int64_t>(h->N + 1);
    h->d_ciA = dalloc<int32_t>(h->nnzA);
    h->d_vA = dalloc<double>(h->nnzA);
    CK(cudaMemcpy(h->d_rpA, rpw.data(), (h->N + 1) * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->d_ciA, ci32.data(), h->nnzA * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->d_vA, vw.data(), h->nnzA * 8, cudaMemcpyHostToDevice));
  } else if (d->kind == GADI_PROBLEM_BAND) {
    // BASELINE configs[3] generated on the device (bit for bit orc_band_csr)
    const int64_t n = d->n_rows;
    if (n < 2 || d->k_off < 1 || d->k_off > 31 || d->band < d->k_off || n - 1 < d->k_off)
      throw Err(GADI_E_CONTRACT, "band: need 1 <= k_off <= 31, band >= k_off, n_rows > k_off");
    if (n >= (int64_t(1) << 31)) throw Err(GADI_E_UNSUPPORTED, "band: n_rows must be < 2^31");
    h->max_band = d->band;
    if (grp) set_window(n, d->band);
    else hi = n;
    const int64_t rows = hi - lo, gnnz = rows * (int64_t)(d->k_off + 1);
    h->d_rpA = dalloc<int64_t>(rows + 1);
    h->d_ciA = dalloc<int32_t>(gnnz);
    h->d_vA = dalloc<double>(gnnz);
    k_iota_scaled<<<ew_grid(rows + 1), 256>>>(h->d_rpA, rows + 1, d->k_off + 1);
    k_band_gen<<<ew_grid(rows), 256>>>(n, d->k_off, d->band, d->seed, h->d_ciA, h->d_vA, lo, rows);
    CKL();
    CK(cudaDeviceSynchronize());
    h->N = rows;
    h->nnzA = gnnz;
    if (grp) {  // rows [lo, hi) restricted to the columns [lo, hi), shifted by -lo
      int64_t* cnt = dalloc<int64_t>(rows + 1);
      CK(cudaMemset(cnt + rows, 0, 8));
      k_window_count<<<ew_grid(rows), 256>>>(h->d_rpA, h->d_ciA, rows, lo, hi, cnt);
      CKL();
      int64_t* nrp = dalloc<int64_t>(rows + 1);
      scan_i64(nullptr, cnt, nrp, rows + 1);
      CK(cudaMemcpy(&h->nnzA, nrp + rows, 8, cudaMemcpyDeviceToHost));
      int32_t* nci = dalloc<int32_t>(h->nnzA);
      double* nv = dalloc<double>(h->nnzA);
      k_window_fill<<<ew_grid(rows), 256>>>(h->d_rpA, h->d_ciA, h->d_vA, rows, lo, hi, nrp, nci, nv);
      CKL();
      CK(cudaDeviceSynchronize());
      for (void* p : {(void*)cnt, (void*)h->d_rpA, (void*)h->d_ciA, (void*)h->d_vA}) cudaFree(p);
      h->d_rpA = nrp;
      h->d_ciA = nci;
      h->d_vA = nv;
    }
  } else {
    throw Err(GADI_E_CONTRACT, "unknown problem kind");
  }
  CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  if (!h->stencil()) {
    device_split(h.get());
    if (grp) {
      crop_rows(h.get(), r0 - lo, r1 - lo);
      h->row0 = r0;
      h->gh = (h->max_band + 7) & ~int64_t(7);  // >= the band; a multiple of 8 keeps 16-byte windows aligned
      if (h->gh > h->N) throw Err(GADI_E_UNSUPPORTED, "sharded solves: the band exceeds a row block (fewer ranks)");
      if (grp->local)
        h->comm.reset(new LocalComm(grp->local.get(), rank));
      else if (grp->ipc)
        h->comm.reset(new IpcComm(grp->ipc.get(), (size_t)h->gh * 8));
      else
        h->comm.reset(new NcclComm(grp->world, rank, grp->id));
    }
    build_sell_A(h.get());
  }
  const int64_t N = h->N;
  h->d_x = hvec<double>(h.get());
  h->d_b = hvec<double>(h.get());
  h->d_s = hvec<double>(h.get());
  h->d_t64 = hvec<double>(h.get());
  h->st = dalloc<DevState>(1);
  CK(cudaMemset(h->st, 0, sizeof(DevState)));
  if (h->sharded()) {
    const int one = 1;
    CK(cudaMemcpy(&h->st->dist, &one, sizeof(int), cudaMemcpyHostToDevice));
  }
  CK(cudaHostAlloc(&h->h_st, sizeof(DevState), cudaHostAllocDefault));
  std::memset(h->h_st, 0, sizeof(DevState));
  const int64_t maxblk = std::max<int64_t>(N / 64, 1) + 8;
  h->d_part0 = dalloc<double>(maxblk);
  h->d_part1 = dalloc<double>(maxblk);
  h->d_partm = dalloc<double>(4 * maxblk);
  h->partm_stride = maxblk;
  h->d_ticket = dalloc<unsigned>(1);
  CK(cudaMemset(h->d_ticket, 0, sizeof(unsigned)));
  CK(cudaHostAlloc(&h->h_done, sizeof(int), cudaHostAllocMapped));
  *h->h_done = 0;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->d_h_done), h->h_done, 0));
  CK(cudaMemcpy(&h->st->hdone, &h->d_h_done, sizeof(int*), cudaMemcpyHostToDevice));
  for (cudaEvent_t* ev : {&h->ev0, &h->ev1, &h->evA, &h->evB, &h->evC}) CK(cudaEventCreate(ev));
  h->ring.resize(4);
  for (auto& ev : h->ring) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  return h.release();
}

int gadi_cuda_create(const gadi_problem_desc* d, const gadi_device_opts* opts, gadi_handle** out) {
  API_BEGIN
  if (!d || !out) throw Err(GADI_E_CONTRACT, "gadi_cuda_create: null argument");
  *out = nullptr;
  *out = create_impl(d, opts, nullptr, 0);
  API_END
}

int gadi_cuda_destroy(gadi_handle* h) {
  if (!h) return GADI_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->eng.reset();
  for (auto& p : h->ex)
    for (void* q : {(void*)p.rp, (void*)p.ci, (void*)p.v, (void*)p.dpos, (void*)p.din})
      if (q) cudaFree(q);
  for (void* p : {(void*)h->d_rpA, (void*)h->d_ciA, (void*)h->d_vA, (void*)h->d_urp, (void*)h->d_uci,
                  (void*)h->d_mv, (void*)h->d_nv, (void*)h->d_dpos, (void*)h->d_din, (void*)h->st,
                  (void*)h->d_part0, (void*)h->d_part1, (void*)h->d_partm, (void*)h->d_ticket})
    if (p) cudaFree(p);
  for (void* p : h->raw) cudaFree(p);  // d_x, d_b, d_s, d_t64 (hvec)
  h->comm.reset();
  h->sellA.release();
  if (h->h_st) cudaFreeHost(h->h_st);
  if (h->h_done) cudaFreeHost(h->h_done);
  for (cudaEvent_t ev : {h->ev0, h->ev1, h->evA, h->evB, h->evC})
    if (ev) cudaEventDestroy(ev);
  for (auto ev : h->ring) cudaEventDestroy(ev);
  if (h->stream) {
    cudaStreamSynchronize(h->stream);
    cudaStreamDestroy(h->stream);
  }
  try {
    engine_pool_trim(h->device);  // unused work-vector memory back to the device (other live handles keep theirs)
  } catch (...) {
  }
  delete h;
  return GADI_OK;
}

// explicit_splitting(A, M, N) (splitting.cpp:22-35): shapes, the M + N = A
// check on the entries of add(1.0, M, 1.0, N) (A's entry there, 0 where A has
// none, within one ulp of |a|), then M and N go to the device on
// shift_diagonal's pattern (their own plus the diagonal, sparse.cpp:180-183);
// the alpha shift itself happens on the device when prepare fills the operator
// images (k_sell_fill / k_band_csr). HSS drops an explicit split again.
int gadi_cuda_set_split(gadi_handle* h, int32_t kind, const gadi_csr_desc* M, const gadi_csr_desc* Nn) {
  API_BEGIN
  if (!h) throw Err(GADI_E_CONTRACT, "set_split: null handle");
  if (kind != GADI_SPLIT_HSS && kind != GADI_SPLIT_EXPLICIT) throw Err(GADI_E_PARAM, "set_split: unknown split kind");
  if (h->sharded()) throw Err(GADI_E_UNSUPPORTED, "set_split: not on a shard");
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->stream));
  h->eng.reset();  // operators of the previous split
  auto drop = [&]() {
    for (auto& p : h->ex) {
      for (void* q : {(void*)p.rp, (void*)p.ci, (void*)p.v, (void*)p.dpos, (void*)p.din})
        if (q) cudaFree(q);
      p = gadi_handle::SplitPart{};
    }
    h->explicit_split = false;
  };
  drop();
  if (kind == GADI_SPLIT_HSS) return GADI_OK;
  if (h->stencil() || h->kind == GADI_PROBLEM_BAND)
    throw Err(GADI_E_UNSUPPORTED, "set_split: explicit splittings need a GADI_PROBLEM_CSR handle");
  if (!M || !Nn) throw Err(GADI_E_CONTRACT, "explicit_splitting: null argument");
  const int64_t n = h->N;
  for (const gadi_csr_desc* m : {M, Nn}) {
    if (m->n_rows != n || m->n_cols != n) throw Err(GADI_E_CONTRACT, "explicit_splitting: shape mismatch");
    if (!m->row_ptr || (m->nnz > 0 && (!m->col_idx || !m->values)) || m->row_ptr[0] != 0 || m->row_ptr[n] != m->nnz)
      throw Err(GADI_E_CONTRACT, "explicit_splitting: bad CSR arrays");
    for (int64_t i = 0; i < n; ++i) {  // the SparseMatrix invariants, sparse.cpp:19-34
      if (m->row_ptr[i] > m->row_ptr[i + 1]) throw Err(GADI_E_CONTRACT, "row_ptr must be non-decreasing");
      for (int64_t k = m->row_ptr[i]; k < m->row_ptr[i + 1]; ++k) {
        if (m->col_idx[k] < 0 || m->col_idx[k] >= n) throw Err(GADI_E_CONTRACT, "column index out of range");
        if (k > m->row_ptr[i] && m->col_idx[k] <= m->col_idx[k - 1])
          throw Err(GADI_E_CONTRACT, "column indices must be strictly increasing within a row");
      }
    }
  }
  // A back from the device (this is setup; the handle keeps no host copy)
  std::vector<int64_t> arp(n + 1);
  std::vector<int32_t> aci(h->nnzA);
  std::vector<double> av(h->nnzA);
  CK(cudaMemcpy(arp.data(), h->d_rpA, (n + 1) * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(aci.data(), h->d_ciA, h->nnzA * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(av.data(), h->d_vA, h->nnzA * 8, cudaMemcpyDeviceToHost));
  int64_t band = h->max_band;
  for (int64_t i = 0; i < n; ++i) {
    int64_t m = M->row_ptr[i], me = M->row_ptr[i + 1], q = Nn->row_ptr[i], qe = Nn->row_ptr[i + 1];
    int64_t a = arp[i];
    const int64_t ae = arp[i + 1];
    while (m < me || q < qe) {
      const int64_t cm = m < me ? M->col_idx[m] : INT64_MAX, cn = q < qe ? Nn->col_idx[q] : INT64_MAX;
      const int64_t col = std::min(cm, cn);
      double sum;
      if (cm == col && cn == col) sum = 1.0 * M->values[m] + 1.0 * Nn->values[q];
      else if (cm == col) sum = 1.0 * M->values[m];
      else sum = 1.0 * Nn->values[q];
      if (cm == col) ++m;
      if (cn == col) ++q;
      while (a < ae && aci[a] < col) ++a;
      const double aa = (a < ae && aci[a] == col) ? av[a] : 0.0;
      if (std::fabs(sum - aa) > std::fabs(aa) * 2.220446049250313e-16)
        throw Err(GADI_E_CONTRACT, "explicit_splitting: M + N != A");
      band = std::max<int64_t>(band, std::llabs(col - i));
    }
  }
  for (int w = 0; w < 2; ++w) {
    const gadi_csr_desc* m = w == 0 ? M : Nn;
    std::vector<int64_t> rp(n + 1, 0), dpos(n);
    std::vector<int32_t> ci;
    std::vector<double> v;
    std::vector<uint8_t> din(n);
    ci.reserve(m->nnz + n);
    v.reserve(m->nnz + n);
    for (int64_t i = 0; i < n; ++i) {
      bool done = false;
      for (int64_t k = m->row_ptr[i]; k < m->row_ptr[i + 1] || !done;) {
        const int64_t col = k < m->row_ptr[i + 1] ? m->col_idx[k] : INT64_MAX;
        if (!done && i <= col) {
          dpos[i] = (int64_t)ci.size();
          din[i] = col == i;
          ci.push_back((int32_t)i);
          v.push_back(col == i ? m->values[k] : 0.0);
          if (col == i) ++k;
          done = true;
        } else {
          ci.push_back((int32_t)col);
          v.push_back(m->values[k]);
          ++k;
        }
      }
      rp[i + 1] = (int64_t)ci.size();
    }
    auto& p = h->ex[w];
    p.nnz = (int64_t)ci.size();
    p.rp = dalloc<int64_t>(n + 1);
    p.ci = dalloc<int32_t>(p.nnz);
    p.v = dalloc<double>(p.nnz);
    p.dpos = dalloc<int64_t>(n);
    p.din = dalloc<uint8_t>(n);
    CK(cudaMemcpy(p.rp, rp.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(p.ci, ci.data(), p.nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(p.v, v.data(), p.nnz * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(p.dpos, dpos.data(), n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(p.din, din.data(), n, cudaMemcpyHostToDevice));
  }
  h->ex_band = band;
  h->explicit_split = true;
  API_END
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
  CK(cudaMemcpyAsync(h->d_b, b, h->N * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  API_END
}

int gadi_cuda_residual_uf(gadi_handle* h, int32_t u_f, const double* x, double* s_out) {
  API_BEGIN
  if (h && h->sharded()) throw Err(GADI_E_UNSUPPORTED, "gadi_cuda_residual_uf: not on a shard (use the sharded solve)");
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
  if (h && h->sharded()) throw Err(GADI_E_UNSUPPORTED, "gadi_cuda_true_residual_norm: not on a shard (use the sharded solve)");
  if (!h || !x || !norm_out) throw Err(GADI_E_CONTRACT, "true_residual_norm: null argument");
  CK(cudaSetDevice(h->device));
  CK(cudaMemcpyAsync(h->d_t64, x, h->N * 8, cudaMemcpyHostToDevice, h->stream));
  OuterA::resid_sync(h, h->d_t64, nullptr, GADI_DOUBLE, false);
  *norm_out = res_norm(h);
  API_END
}

int gadi_cuda_prepare(gadi_handle* h, double alpha, double omega, int32_t u_r, const gadi_inner_spec* spec,
                      int32_t accum) {
  API_BEGIN
  if (h && h->sharded()) throw Err(GADI_E_UNSUPPORTED, "gadi_cuda_prepare: not on a shard (use the sharded solve)");
  if (!h || !spec) throw Err(GADI_E_CONTRACT, "prepare: null argument");
  if (u_r < 0 || u_r > 2) throw Err(GADI_E_PARAM, "unknown precision");
  CK(cudaSetDevice(h->device));
  try {
    prepare(h, alpha, omega, u_r, *spec, accum);
  } catch (const PrepareStatus& ps) {  // the exceptions prepare throws (inner_solver.cpp:27-34)
    if (ps.status == GADI_SINGULAR_IN_PRECISION)
      throw Err(GADI_E_SINGULAR, "SingularInPrecision: pivot below the normal range of u_r");
    throw Err(GADI_E_OVERFLOW, "OverflowDetected: non-finite entry produced during banded elimination");
  }
  API_END
}

int gadi_cuda_reset(gadi_handle* h) {
  API_BEGIN
  if (!h) throw Err(GADI_E_CONTRACT, "reset: null handle");
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->stream));
  h->eng.reset();
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
  if (e->spec.method == GADI_INNER_LU_DIRECT) o = lu_solve(h, e, which, e->rhat, e->z);
  else if (which == 1 && e->spec.method == GADI_INNER_CG) o = e->cg(1, e->rhat, e->z, target);
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
  // e2e: timed from the host copy of b to the host copy of x
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, h->stream));
  CK(cudaMemcpyAsync(h->d_b, b, h->N * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  double h2d = (double)h->N * 8;
  if (x0) {
    CK(cudaMemcpyAsync(h->d_x, x0, h->N * 8, cudaMemcpyHostToDevice, h->stream));
    h2d += (double)h->N * 8;
  } else {
    k_fill<<<ew_grid(h->N), 256, 0, h->stream>>>(h->d_x, cfg->ones_start ? 1.0 : 0.0, h->N);
    CKL();
    ++h->launches;
  }
  const int64_t l0 = h->launches;
  run(h, cfg, rep);
  CK(cudaMemcpyAsync(x_out, h->d_x, h->N * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaEventRecord(e1, h->stream));
  CK(cudaEventSynchronize(e1));
  rep->e2e_ms = ms_between(e0, e1);
  rep->h2d_bytes = h2d;
  rep->d2h_bytes = (double)h->N * 8;
  rep->launches = h->launches - l0 + (x0 ? 0 : 1);
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
  CK(cudaMemcpyAsync(h->d_b, d_b, h->N * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  if (d_x0) {
    CK(cudaMemcpyAsync(h->d_x, d_x0, h->N * 8, cudaMemcpyDeviceToDevice, h->stream));
  } else {
    k_fill<<<ew_grid(h->N), 256, 0, h->stream>>>(h->d_x, cfg->ones_start ? 1.0 : 0.0, h->N);
    CKL();
    ++h->launches;
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
  if (h && h->sharded()) throw Err(GADI_E_UNSUPPORTED, "gadi_cuda_apply: not on a shard (use the sharded solve)");
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

int64_t gadi_cuda_launch_count(const gadi_handle* h) { return h ? h->launches : 0; }

int gadi_cuda_nnz(const gadi_handle* h, int64_t* nnz_a, int64_t* nnz_hs) {
  if (!h || !nnz_a || !nnz_hs) return GADI_E_CONTRACT;
  *nnz_a = h->nnzA;
  *nnz_hs = h->nnzHS;
  return GADI_OK;
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
  if (p == GADI_HALF) k_dot_d<__half><<<g.nblk, g.threads()>>>(dx, dy, g, rd, dout);
  else if (p == GADI_SINGLE) k_dot_d<float><<<g.nblk, g.threads()>>>(dx, dy, g, rd, dout);
  else k_dot_d<double><<<g.nblk, g.threads()>>>(dx, dy, g, rd, dout);
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
  // x_true by global row (a shard draws its slab of the same sequence), then
  // b = A x_true with the neighbours' x_true planes (a collective on shards)
  k_uniform<<<ew_grid(h->N), 256, 0, h->stream>>>(h->d_t64, seed, lo, hi, h->N, h->e_off());
  CKL();
  ++h->launches;
  halo(h, h->d_t64);
  OuterA::apply(h, h->d_t64, d_b);
  CK(cudaMemcpyAsync(d_xtrue, h->d_t64, h->N * 8, cudaMemcpyDeviceToDevice, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  API_END
}

// ------------------------------------------------------------ sharded solves
int gadi_group_local(int32_t world, gadi_group** out) {
  API_BEGIN
  if (!out) throw Err(GADI_E_CONTRACT, "group: null argument");
  if (world < 1 || world > GADI_MAX_RANKS || (world & (world - 1)) != 0)
    throw Err(GADI_E_PARAM, "group: world must be a power of two <= 64");
  gadi_group* g = new gadi_group();
  g->world = world;
  g->local.reset(new LocalGroup(world));
  *out = g;
  API_END
}

int gadi_nccl_unique_id(uint8_t* out128) {
  API_BEGIN
  if (!out128) throw Err(GADI_E_CONTRACT, "nccl id: null argument");
  NcclApi& a = NcclApi::get();
  if (a.get_unique_id(out128) != 0) throw Err(GADI_E_NCCL, "ncclGetUniqueId failed");
  API_END
}

int gadi_group_nccl(int32_t world, int32_t rank, const uint8_t* id128, gadi_group** out) {
  API_BEGIN
  if (!out || !id128) throw Err(GADI_E_CONTRACT, "group: null argument");
  if (world < 1 || world > GADI_MAX_RANKS || (world & (world - 1)) != 0)
    throw Err(GADI_E_PARAM, "group: world must be a power of two <= 64");
  if (rank < 0 || rank >= world) throw Err(GADI_E_PARAM, "group: rank out of range");
  NcclApi::get();  // fails loudly without libnccl
  gadi_group* g = new gadi_group();
  g->world = world;
  g->nccl_rank = rank;
  std::memcpy(g->id.b, id128, sizeof(g->id.b));
  *out = g;
  API_END
}

int gadi_group_ipc(int32_t world, int32_t rank, const char* name, gadi_group** out) {
  API_BEGIN
  if (!out || !name || name[0] != '/') throw Err(GADI_E_CONTRACT, "ipc group: need a shared-memory name starting with '/'");
  if (world < 1 || world > GADI_MAX_RANKS || (world & (world - 1)) != 0)
    throw Err(GADI_E_PARAM, "group: world must be a power of two <= 64");
  if (rank < 0 || rank >= world) throw Err(GADI_E_PARAM, "group: rank out of range");
  std::unique_ptr<gadi_group> g(new gadi_group());
  g->world = world;
  g->nccl_rank = rank;
  g->ipc.reset(new IpcGroup(world, rank, name));
  *out = g.release();
  API_END
}

int gadi_group_destroy(gadi_group* g) {
  delete g;
  return GADI_OK;
}

int gadi_cuda_create_shard(const gadi_problem_desc* d, const gadi_device_opts* opts, gadi_group* g, int32_t rank,
                           gadi_handle** out) {
  API_BEGIN
  if (!d || !g || !out) throw Err(GADI_E_CONTRACT, "create_shard: null argument");
  *out = nullptr;
  *out = create_impl(d, opts, g, rank);
  API_END
}

int gadi_cuda_shard_range(const gadi_handle* h, int64_t* first_row, int64_t* n_rows) {
  if (!h || !first_row || !n_rows) return GADI_E_CONTRACT;
  *first_row = h->e_off();
  *n_rows = h->N;
  return GADI_OK;
}

int gadi_cuda_solve_group(gadi_handle* const* hs, int32_t world, const gadi_config* cfg, const double* const* d_b,
                          const double* const* d_x0, double* const* d_x, gadi_report* reps) {
  API_BEGIN
  if (!hs || !cfg || !d_b || !d_x || !reps || world < 1) throw Err(GADI_E_CONTRACT, "solve_group: null argument");
  LocalGroup* lg = nullptr;
  for (int r = 0; r < world; ++r) {
    auto* lc = hs[r] ? dynamic_cast<LocalComm*>(hs[r]->comm.get()) : nullptr;
    if (!lc || lc->rank != r || lc->world != world || (lg && lc->g != lg))
      throw Err(GADI_E_CONTRACT, "solve_group: handles must be ranks 0..world-1 of one local group");
    lg = lc->g;
  }
  std::vector<int> rc(world, GADI_OK);
  std::vector<std::string> msg(world);
  std::vector<std::thread> th;
  for (int r = 0; r < world; ++r)
    th.emplace_back([&, r] {
      rc[r] = gadi_cuda_solve_device(hs[r], cfg, d_b[r], d_x0 ? d_x0[r] : nullptr, d_x[r], &reps[r]);
      if (rc[r] != GADI_OK) {
        msg[r] = gadi_last_error();
        lg->abort();  // release the ranks waiting at a collective
      }
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < world; ++r)
    if (rc[r] != GADI_OK && msg[r].find("aborted by another rank") == std::string::npos)
      throw Err(rc[r], "rank " + std::to_string(r) + ": " + msg[r]);
  for (int r = 0; r < world; ++r)
    if (rc[r] != GADI_OK) throw Err(rc[r], msg[r]);
  API_END
}

}  // extern "C"
