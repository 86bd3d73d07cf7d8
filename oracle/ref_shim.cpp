// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (checker / CPU baseline).
//
// extern "C" wrapper around the UNMODIFIED reference library
// (/root/reference/proj/core).  oracle/Makefile compiles this file together
// with the reference's own translation units (src/tiles.cpp,
// src/threadpool.cpp) straight from /root/reference with the reference's
// Release flags (-O3 -DNDEBUG -std=gnu++20, baseline x86-64 ISA: no FMA, no
// contraction) into oracle/_ref/libdrotref.so.  No reference source is
// copied into this repository; this file only calls the reference's public
// API:
//   drot::solve<T>             solver.hpp:372-540
//   drot::init_state / drot_step / detail::state_report   solver.hpp:143,361,312
//   drot::FusedEngine<T>       fused.hpp:107-202 (fused_pass :127,
//                              fused_pass_skip_cost :140, unfused_pass :359)
//   drot::check_problem        problem.hpp:122-136
//   drot::residual_report      problem.hpp:174-225
//   drot::gen_gaussian_problem probgen.hpp:131-170
//   drot::CounterRng           rng.hpp:30-106
//   drot::lp_exact             reference.hpp:537-552
//   drot::sinkhorn_solve       reference.hpp:165-288
#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "drot/drot.hpp"
#include "oracle.h"

namespace {

thread_local std::string g_last_error;

int errc_ret(const drot::Error& e) {
  g_last_error = e.what();
  return 1 + static_cast<int>(e.code());
}

drot::DrotConfig to_cfg(const orc_config* c) {
  drot::DrotConfig cfg;
  if (!c) return cfg;
  cfg.rho0 = c->rho0;
  if (c->has_rho_override) cfg.rho_override = c->rho_override;
  cfg.tol_primal = c->tol_primal;
  cfg.tol_dual = c->tol_dual;
  cfg.tol_gap = c->tol_gap;
  cfg.relative_tolerances = c->relative_tolerances != 0;
  cfg.max_iters = c->max_iters;
  cfg.check_every = c->check_every;
  cfg.engine = c->engine == 0 ? drot::EngineKind::reference
                              : drot::EngineKind::fused;
  cfg.skip_cost = c->skip_cost != 0;
  cfg.deterministic = c->deterministic != 0;
  cfg.workers = static_cast<std::size_t>(c->workers);
  cfg.block_rows = static_cast<std::size_t>(c->block_rows);
  cfg.work_size = static_cast<std::size_t>(c->work_size);
  cfg.record_trace = c->record_trace != 0;
  cfg.trace_every = c->trace_every;
  return cfg;
}

template <class T>
drot::Matrix<T> to_matrix(const T* src, int64_t m, int64_t n) {
  drot::Matrix<T> a(static_cast<std::size_t>(m), static_cast<std::size_t>(n));
  if (m * n) std::memcpy(a.data(), src, sizeof(T) * m * n);
  return a;
}

template <class T>
drot::TransportProblem<T> to_problem(const T* C, int64_t m, int64_t n,
                                     const T* p, const T* q) {
  drot::TransportProblem<T> pr;
  pr.cost = to_matrix(C, m, n);
  pr.p.assign(p, p + m);
  pr.q.assign(q, q + n);
  return pr;
}

void put_report(orc_report* out, const drot::ResidualReport& r) {
  if (!out) return;
  out->r_primal = r.r_primal;
  out->r_dual = r.r_dual;
  out->gap = r.gap;
  out->objective = r.objective;
}

template <class T>
int sinkhorn_impl(const T* C, int64_t m, int64_t n, const T* p, const T* q, T eta, double tol,
                  int64_t max_iters, int64_t check_every, T* plan, T* mu, T* nu,
                  orc_report* rep, orc_trace_row* trace, int64_t trace_cap,
                  int64_t* trace_len, int64_t* iters, int32_t* status, double* wall) {
  try {
    auto pr = to_problem(C, m, n, p, q);
    auto res = drot::sinkhorn_solve<T>(pr, eta, tol, max_iters, check_every);
    if (plan) std::memcpy(plan, res.plan.x.data(), sizeof(T) * m * n);
    if (mu) std::memcpy(mu, res.cert.mu.data(), sizeof(T) * m);
    if (nu) std::memcpy(nu, res.cert.nu.data(), sizeof(T) * n);
    put_report(rep, res.report);
    if (trace_len) *trace_len = static_cast<int64_t>(res.trace.rows.size());
    if (trace) {
      const int64_t cnt =
          std::min<int64_t>(trace_cap, static_cast<int64_t>(res.trace.rows.size()));
      for (int64_t k = 0; k < cnt; ++k) {
        const auto& r = res.trace.rows[k];
        trace[k] = orc_trace_row{r.iter,      r.r_primal,
                                 r.r_dual,    r.gap,
                                 r.objective, r.ergodic_objective,
                                 r.fixed_point_residual};
      }
    }
    if (iters) *iters = res.trace.iterations;
    if (status) *status = static_cast<int32_t>(res.status);
    if (wall) *wall = res.trace.wall_time_s;
    return 0;
  } catch (const drot::Error& e) {
    return errc_ret(e);
  }
}

template <class T>
int solve_impl(const T* C, int64_t m, int64_t n, const T* p, const T* q,
               const orc_config* c, const T* x0, T* plan, T* mu, T* nu,
               orc_report* rep, orc_trace_row* trace, int64_t trace_cap,
               int64_t* trace_len, int64_t* iters, int32_t* status,
               double* wall) {
  try {
    auto pr = to_problem(C, m, n, p, q);
    auto cfg = to_cfg(c);
    drot::Matrix<T> x0m;
    if (x0) x0m = to_matrix(x0, m, n);
    auto res = drot::solve<T>(pr, cfg, x0 ? &x0m : nullptr);
    if (plan) std::memcpy(plan, res.plan.x.data(), sizeof(T) * m * n);
    if (mu) std::memcpy(mu, res.cert.mu.data(), sizeof(T) * m);
    if (nu) std::memcpy(nu, res.cert.nu.data(), sizeof(T) * n);
    put_report(rep, res.report);
    if (trace_len) *trace_len = static_cast<int64_t>(res.trace.rows.size());
    if (trace) {
      const int64_t cnt =
          std::min<int64_t>(trace_cap, static_cast<int64_t>(res.trace.rows.size()));
      for (int64_t k = 0; k < cnt; ++k) {
        const auto& r = res.trace.rows[k];
        trace[k] = orc_trace_row{r.iter,      r.r_primal,
                                 r.r_dual,    r.gap,
                                 r.objective, r.ergodic_objective,
                                 r.fixed_point_residual};
      }
    }
    if (iters) *iters = res.trace.iterations;
    if (status) *status = static_cast<int32_t>(res.status);
    if (wall) *wall = res.trace.wall_time_s;
    return 0;
  } catch (const drot::Error& e) {
    return errc_ret(e);
  }
}

template <class T>
int pass_impl(T* xy, const T* C, int64_t m, int64_t n, const T* phi,
              const T* varphi, T rho, int64_t bs, int64_t ws, int64_t workers,
              int32_t kind, int32_t fold, int32_t* folded_inout, int32_t parity,
              int32_t want_dual, int32_t want_dx, int32_t deterministic,
              T* row_sums, T* col_sums, orc_pass_out* out,
              orc_counters* counters) {
  try {
    drot::FusedEngine<T> eng(drot::plan_tiles(
        static_cast<std::size_t>(m), static_cast<std::size_t>(n),
        static_cast<std::size_t>(bs), static_cast<std::size_t>(ws),
        static_cast<std::size_t>(workers)));
    auto cost = to_matrix(C, m, n);
    drot::PassOptions opts;
    opts.parity = parity;
    opts.want_dual = want_dual != 0;
    opts.want_dx = want_dx != 0;
    opts.deterministic = deterministic != 0;
    drot::MemoryCounters mc;
    if (counters) {
      mc.passes = counters->passes;
      mc.xy_elems_read = counters->xy_elems_read;
      mc.xy_elems_written = counters->xy_elems_written;
      mc.cost_elems_read = counters->cost_elems_read;
      opts.counters = &mc;
    }
    std::span<const T> ph(phi, static_cast<std::size_t>(m));
    std::span<const T> vph(varphi, static_cast<std::size_t>(n));
    drot::FusedPassOutput<T> o;
    if (kind == ORC_PASS_SKIP_COST) {
      drot::FusedArray<T> arr{to_matrix(xy, m, n), *folded_inout != 0};
      o = eng.fused_pass_skip_cost(arr, cost, ph, vph, rho, fold != 0, opts);
      *folded_inout = arr.cost_folded ? 1 : 0;
      std::memcpy(xy, arr.values.data(), sizeof(T) * m * n);
    } else {
      auto a = to_matrix(xy, m, n);
      if (kind == ORC_PASS_UNFUSED)
        o = eng.unfused_pass(a, cost, ph, vph, rho, opts);
      else
        o = eng.fused_pass(a, cost, ph, vph, rho, opts);
      std::memcpy(xy, a.data(), sizeof(T) * m * n);
    }
    if (row_sums) std::memcpy(row_sums, o.row_sums.data(), sizeof(T) * m);
    if (col_sums) std::memcpy(col_sums, o.col_sums.data(), sizeof(T) * n);
    if (out) {
      out->cost_dot = o.cost_dot;
      out->max_abs = o.max_abs;
      out->dual_sq = o.dual_sq;
      out->dx_sq = o.dx_sq;
      out->prev_cost_dot = o.prev_cost_dot;
      out->cost_valid = o.cost_valid;
      out->nonfinite = o.nonfinite;
      out->dual_valid = o.dual_valid;
      out->dx_valid = o.dx_valid;
      out->prev_cost_valid = o.prev_cost_valid;
    }
    if (counters) {
      counters->passes = mc.passes;
      counters->xy_elems_read = mc.xy_elems_read;
      counters->xy_elems_written = mc.xy_elems_written;
      counters->cost_elems_read = mc.cost_elems_read;
    }
    return 0;
  } catch (const drot::Error& e) {
    return errc_ret(e);
  }
}

// init_state + k x drot_step, then the state arrays and state_report.
template <class T>
int steps_impl(const T* C, int64_t m, int64_t n, const T* p, const T* q,
               const orc_config* c, int64_t k, T* xy, int32_t* folded,
               T* phi, T* varphi, T* a, T* b, T* alpha, T* r, T* s, T* beta,
               orc_report* rep) {
  try {
    auto pr = to_problem(C, m, n, p, q);
    auto cfg = to_cfg(c);
    auto st = drot::init_state(pr, cfg);
    for (int64_t it = 0; it < k; ++it) drot::drot_step(st, pr, cfg);
    const T rho = static_cast<T>(cfg.resolved_rho(pr.m(), pr.n()));
    if (xy) std::memcpy(xy, st.xy.values.data(), sizeof(T) * m * n);
    if (folded) *folded = st.xy.cost_folded ? 1 : 0;
    if (phi) std::memcpy(phi, st.row_shift.data(), sizeof(T) * m);
    if (varphi) std::memcpy(varphi, st.col_shift.data(), sizeof(T) * n);
    if (a) std::memcpy(a, st.y_row_defect.data(), sizeof(T) * m);
    if (b) std::memcpy(b, st.y_col_defect.data(), sizeof(T) * n);
    if (alpha) *alpha = st.y_mass_gap;
    if (r) std::memcpy(r, st.row_residual.data(), sizeof(T) * m);
    if (s) std::memcpy(s, st.col_residual.data(), sizeof(T) * n);
    if (beta) *beta = st.x_mass_gap;
    put_report(rep, drot::detail::state_report(st, pr, rho));
    return 0;
  } catch (const drot::Error& e) {
    return errc_ret(e);
  }
}

// Per-iteration wall time of the reference solve loop: solve(max_iters=w)
// and solve(max_iters=w+k) (best of two calls each) with unreachable tolerances (every other field of
// cfg, record_trace included, as given); the difference / k removes
// validation, init, the w warm-up iterations and the final report.
template <class T>
int time_iters_impl(const T* C, int64_t m, int64_t n, const T* p, const T* q,
                    const orc_config* c, int64_t k, int64_t w, double* sec_per_iter,
                    double* sec_total) {
  try {
    auto pr = to_problem(C, m, n, p, q);
    auto cfg = to_cfg(c);
    cfg.tol_primal = cfg.tol_dual = cfg.tol_gap = -1.0;
    using clk = std::chrono::steady_clock;
    auto timed = [&](int64_t iters) {  // best of two calls
      cfg.max_iters = static_cast<decltype(cfg.max_iters)>(iters);
      double best = 1e300;
      for (int rep = 0; rep < 2; ++rep) {
        const auto t0 = clk::now();
        (void)drot::solve<T>(pr, cfg);
        best = std::min(best, std::chrono::duration<double>(clk::now() - t0).count());
      }
      return best;
    };
    cfg.max_iters = static_cast<decltype(cfg.max_iters)>(w);
    (void)drot::solve<T>(pr, cfg);  // warm: first-touch of the solver's buffers
    const double a = timed(w);
    const double b = timed(w + k);
    if (sec_per_iter) *sec_per_iter = (b - a) / static_cast<double>(k);
    if (sec_total) *sec_total = 2.0 * (a + b);
    return 0;
  } catch (const drot::Error& e) {
    return errc_ret(e);
  }
}

// Median-free single timing of k FusedEngine passes (plain or skip-C).
template <class T>
int time_pass_impl(T* xy, const T* C, int64_t m, int64_t n, const T* phi,
                   const T* varphi, T rho, int64_t workers, int32_t skip,
                   int64_t k, double* sec_per_pass) {
  try {
    drot::FusedEngine<T> eng(drot::plan_tiles(
        static_cast<std::size_t>(m), static_cast<std::size_t>(n), 64, 4,
        static_cast<std::size_t>(workers)));
    auto cost = to_matrix(C, m, n);
    drot::FusedArray<T> arr{to_matrix(xy, m, n), false};
    std::span<const T> ph(phi, static_cast<std::size_t>(m));
    std::span<const T> vph(varphi, static_cast<std::size_t>(n));
    drot::PassOptions opts;
    opts.want_dual = true;
    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    for (int64_t it = 0; it < k; ++it) {
      opts.parity = static_cast<int>(it & 1);
      if (skip)
        (void)eng.fused_pass_skip_cost(arr, cost, ph, vph, rho,
                                       !arr.cost_folded, opts);
      else
        (void)eng.fused_pass(arr.values, cost, ph, vph, rho, opts);
    }
    auto t1 = clk::now();
    *sec_per_pass =
        std::chrono::duration<double>(t1 - t0).count() / static_cast<double>(k);
    return 0;
  } catch (const drot::Error& e) {
    return errc_ret(e);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_last_error.c_str(); }

int64_t ref_hardware_workers(void) {
  return static_cast<int64_t>(drot::ThreadPool::hardware_workers());
}

void ref_default_config(orc_config* c) {
  drot::DrotConfig d;
  c->rho0 = d.rho0;
  c->has_rho_override = 0;
  c->relative_tolerances = d.relative_tolerances;
  c->rho_override = 0;
  c->tol_primal = d.tol_primal;
  c->tol_dual = d.tol_dual;
  c->tol_gap = d.tol_gap;
  c->max_iters = d.max_iters;
  c->check_every = d.check_every;
  c->engine = d.engine == drot::EngineKind::reference ? 0 : 1;
  c->skip_cost = d.skip_cost;
  c->deterministic = d.deterministic;
  c->record_trace = d.record_trace;
  c->workers = static_cast<int64_t>(d.workers);
  c->block_rows = static_cast<int64_t>(d.block_rows);
  c->work_size = static_cast<int64_t>(d.work_size);
  c->trace_every = d.trace_every;
}

#define DROT_REF_INSTANTIATE(T, SFX)                                          \
  int ref_solve_##SFX(const T* C, int64_t m, int64_t n, const T* p,           \
                      const T* q, const orc_config* c, const T* x0, T* plan,  \
                      T* mu, T* nu, orc_report* rep, orc_trace_row* trace,    \
                      int64_t trace_cap, int64_t* trace_len, int64_t* iters,  \
                      int32_t* status, double* wall) {                        \
    return solve_impl<T>(C, m, n, p, q, c, x0, plan, mu, nu, rep, trace,      \
                         trace_cap, trace_len, iters, status, wall);          \
  }                                                                           \
  int ref_pass_##SFX(T* xy, const T* C, int64_t m, int64_t n, const T* phi,   \
                     const T* varphi, T rho, int64_t bs, int64_t ws,          \
                     int64_t workers, int32_t kind, int32_t fold,             \
                     int32_t* folded_inout, int32_t parity,                   \
                     int32_t want_dual, int32_t want_dx,                      \
                     int32_t deterministic, T* row_sums, T* col_sums,         \
                     orc_pass_out* out, orc_counters* counters) {             \
    return pass_impl<T>(xy, C, m, n, phi, varphi, rho, bs, ws, workers, kind, \
                        fold, folded_inout, parity, want_dual, want_dx,       \
                        deterministic, row_sums, col_sums, out, counters);    \
  }                                                                           \
  int ref_steps_##SFX(const T* C, int64_t m, int64_t n, const T* p,           \
                      const T* q, const orc_config* c, int64_t k, T* xy,      \
                      int32_t* folded, T* phi, T* varphi, T* a, T* b,         \
                      T* alpha, T* r, T* s, T* beta, orc_report* rep) {       \
    return steps_impl<T>(C, m, n, p, q, c, k, xy, folded, phi, varphi, a, b,  \
                         alpha, r, s, beta, rep);                             \
  }                                                                           \
  int ref_time_iters_##SFX(const T* C, int64_t m, int64_t n, const T* p,      \
                           const T* q, const orc_config* c, int64_t k,        \
                           int64_t w, double* sec_per_iter,                   \
                           double* sec_total) {                               \
    return time_iters_impl<T>(C, m, n, p, q, c, k, w, sec_per_iter, sec_total); \
  }                                                                           \
  int ref_time_pass_##SFX(T* xy, const T* C, int64_t m, int64_t n,            \
                          const T* phi, const T* varphi, T rho,               \
                          int64_t workers, int32_t skip, int64_t k,           \
                          double* sec_per_pass) {                             \
    return time_pass_impl<T>(xy, C, m, n, phi, varphi, rho, workers, skip, k, \
                             sec_per_pass);                                   \
  }                                                                           \
  int ref_check_problem_##SFX(const T* C, int64_t m, int64_t n, const T* p,   \
                              const T* q) {                                   \
    try {                                                                     \
      drot::check_problem(to_problem(C, m, n, p, q));                         \
      return 0;                                                               \
    } catch (const drot::Error& e) {                                          \
      return errc_ret(e);                                                     \
    }                                                                         \
  }                                                                           \
  int ref_sinkhorn_##SFX(const T* C, int64_t m, int64_t n, const T* p,        \
                         const T* q, T eta, double tol, int64_t max_iters,    \
                         int64_t check_every, T* plan, T* mu, T* nu,          \
                         orc_report* rep, orc_trace_row* trace,               \
                         int64_t trace_cap, int64_t* trace_len,               \
                         int64_t* iters, int32_t* status, double* wall) {     \
    return sinkhorn_impl<T>(C, m, n, p, q, eta, tol, max_iters, check_every,  \
                            plan, mu, nu, rep, trace, trace_cap, trace_len,   \
                            iters, status, wall);                             \
  }                                                                           \
  int ref_residual_report_##SFX(const T* C, int64_t m, int64_t n,             \
                                const T* p, const T* q, const T* plan,        \
                                const T* mu, const T* nu, orc_report* rep) {  \
    try {                                                                     \
      auto pr = to_problem(C, m, n, p, q);                                    \
      drot::TransportPlan<T> pl{to_matrix(plan, m, n)};                       \
      drot::DualCertificate<T> cert;                                          \
      cert.mu.assign(mu, mu + m);                                             \
      cert.nu.assign(nu, nu + n);                                             \
      put_report(rep, drot::residual_report(pr, pl, cert));                   \
      return 0;                                                               \
    } catch (const drot::Error& e) {                                          \
      return errc_ret(e);                                                     \
    }                                                                         \
  }

DROT_REF_INSTANTIATE(float, f32)
DROT_REF_INSTANTIATE(double, f64)

int ref_gen_gaussian(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                     int32_t dirichlet, double* C, double* p, double* q) {
  try {
    drot::GaussianSpec spec;
    spec.m = static_cast<std::size_t>(m);
    spec.n = static_cast<std::size_t>(n);
    spec.sigma_t = sigma_t;
    spec.seed = seed;
    spec.dirichlet_marginals = dirichlet != 0;
    auto pr = drot::gen_gaussian_problem(spec);
    std::memcpy(C, pr.cost.data(), sizeof(double) * m * n);
    std::memcpy(p, pr.p.data(), sizeof(double) * m);
    std::memcpy(q, pr.q.data(), sizeof(double) * n);
    return 0;
  } catch (const drot::Error& e) {
    return errc_ret(e);
  }
}

// drot_tests::random_matrix (tests/support/oracles.hpp:128-135) is test code
// of the reference and not part of its library; it is the one-liner
// lo + (hi-lo)*CounterRng(seed).next_unit() in storage order, expressed here
// through the library's CounterRng.
void ref_random_unit(uint64_t seed, int64_t count, double lo, double hi,
                     double* out) {
  drot::CounterRng rng(seed);
  for (int64_t k = 0; k < count; ++k) out[k] = lo + (hi - lo) * rng.next_unit();
}

void ref_rng_u64(uint64_t key, int64_t count, uint64_t* out) {
  drot::CounterRng rng(key);
  for (int64_t k = 0; k < count; ++k) out[k] = rng.next_u64();
}

uint64_t ref_derive_key(uint64_t key, uint64_t stream) {
  return drot::CounterRng::derive_key(key, stream);
}

int ref_lp_exact(const double* C, int64_t m, int64_t n, const double* p,
                 const double* q, double* objective, double* plan) {
  try {
    auto pr = to_problem(C, m, n, p, q);
    auto sol = drot::lp_exact(pr);
    if (objective) *objective = sol.objective;
    if (plan) std::memcpy(plan, sol.plan.data(), sizeof(double) * m * n);
    return 0;
  } catch (const drot::Error& e) {
    return errc_ret(e);
  }
}

}  // extern "C"
