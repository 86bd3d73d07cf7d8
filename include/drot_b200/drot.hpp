// drot_b200/drot.hpp -- source-compatible drop-in for the reference's
// umbrella header drot/drot.hpp (proj/core/include/drot/drot.hpp:17-27),
// restricted to the solve path.  Code written against
//   drot::solve<T>, drot::drot_step<T>, drot::init_state<T>,
//   drot::FusedEngine<T>, drot::check_problem, drot::DrotConfig, ...
// compiles unchanged against this header (swap the include path, link
// libdrotb200.so) and runs on a B200.  Every call goes through the C ABI of
// include/drotb.h; the types below mirror the reference's field for field
// (cited per type).  Header-only; C++17.
#ifndef DROT_B200_DROT_HPP_
#define DROT_B200_DROT_HPP_

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../drotb.h"

namespace drot {

// ---- errors.hpp:24-88 ---------------------------------------------------
enum class Errc {
  negative_cost, marginal_not_simplex, empty_dimension, non_finite_entry,
  shape_mismatch, non_positive_rho, invalid_initial_plan, non_finite_iterate,
  zero_marginal, too_large, degenerate_cost, dimension_mismatch,
  fold_state_mismatch, bad_magic, version_unsupported, size_mismatch,
  ragged_csv, empty_image, k_too_large, io_error, bad_config,
};

inline const char* errc_name(Errc c) { return drotb_errc_name(static_cast<int32_t>(c)); }

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  Errc code() const { return code_; }

 private:
  Errc code_;
};

// Raised for CUDA / NCCL failures (no reference counterpart).
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

[[noreturn]] inline void fail(Errc code, const std::string& what) {
  throw Error(code, std::string(errc_name(code)) + ": " + what);
}

namespace detail {
inline void check(int rc) {
  if (rc == 0) return;
  if (rc >= 1 && rc < DROTB_ERR_CUDA)
    throw Error(static_cast<Errc>(rc - 1), drotb_last_error());
  throw DeviceError(drotb_last_error());
}
template <class T>
constexpr bool is_f32 = std::is_same_v<T, float>;
}  // namespace detail

// ---- matrix.hpp:30-86: dense column-major storage -------------------------
template <class T>
class Matrix {
 public:
  Matrix() = default;
  Matrix(std::size_t rows, std::size_t cols, T fill = T(0))
      : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
  static Matrix from_rows(std::initializer_list<std::initializer_list<T>> rows) {
    const std::size_t m = rows.size(), n = m ? rows.begin()->size() : 0;
    Matrix out(m, n);
    std::size_t i = 0;
    for (const auto& row : rows) {
      if (row.size() != n) fail(Errc::shape_mismatch, "ragged initializer");
      std::size_t j = 0;
      for (T v : row) out(i, j++) = v;
      ++i;
    }
    return out;
  }
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  std::size_t size() const { return data_.size(); }
  T& operator()(std::size_t i, std::size_t j) { return data_[j * rows_ + i]; }
  const T& operator()(std::size_t i, std::size_t j) const { return data_[j * rows_ + i]; }
  T* data() { return data_.data(); }
  const T* data() const { return data_.data(); }
  T* col(std::size_t j) { return data_.data() + j * rows_; }
  const T* col(std::size_t j) const { return data_.data() + j * rows_; }
  bool same_shape(const Matrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<T> data_;
};

// ---- problem.hpp:31-92 ------------------------------------------------------
template <class T>
struct TransportProblem {
  Matrix<T> cost;
  std::vector<T> p, q;
  std::size_t m() const { return cost.rows(); }
  std::size_t n() const { return cost.cols(); }
};
template <class T>
struct TransportPlan {
  Matrix<T> x;
};
template <class T>
struct DualCertificate {
  std::vector<T> mu, nu;
  T rho = T(1);
};
struct ResidualReport {
  double r_primal = 0, r_dual = 0, gap = 0, objective = 0;
};
inline constexpr double kResidualNotApplicable = -1.0;
enum class SolveStatus { converged, max_iters, numerical_failure };
inline const char* to_string(SolveStatus s) {
  switch (s) {
    case SolveStatus::converged: return "converged";
    case SolveStatus::max_iters: return "max_iters";
    case SolveStatus::numerical_failure: return "numerical_failure";
  }
  return "unknown";
}
struct TraceRow {
  std::int64_t iter = 0;
  double r_primal = 0, r_dual = 0, gap = 0, objective = 0, ergodic_objective = 0,
         fixed_point_residual = 0;
};
struct SolveTrace {
  std::vector<TraceRow> rows;
  SolveStatus termination = SolveStatus::max_iters;
  std::int64_t iterations = 0;
  double wall_time_s = 0;
};

// ---- solver.hpp:37-123 ------------------------------------------------------
enum class EngineKind { reference, fused };
enum class Precision { f32, f64 };
// B200 extension (include/drotb.h): reduction order of the device kernels.
enum class Order { reference = DROTB_ORDER_REFERENCE, fast = DROTB_ORDER_FAST };

inline double rho0_warmup_preset(std::size_t m) {
  return 1.0 / std::log(static_cast<double>(m < 3 ? 3 : m));
}

struct DrotConfig {
  double rho0 = 2.0;
  std::optional<double> rho_override;
  double tol_primal = 1e-4, tol_dual = 1e-4, tol_gap = 1e-4;
  bool relative_tolerances = false;
  std::int64_t max_iters = 100000;
  std::int64_t check_every = 1;
  EngineKind engine = EngineKind::fused;
  bool skip_cost = true;
  bool deterministic = true;
  std::size_t workers = 0;       // CPU knob, accepted and ignored
  std::size_t block_rows = 64;
  std::size_t work_size = 4;
  bool record_trace = true;
  std::int64_t trace_every = 1;
  Precision precision = Precision::f64;
  // B200 extensions
  int device = -1;
  Order order = Order::fast;
  bool use_graphs = true;

  double resolved_rho(std::size_t m, std::size_t n) const {
    const double rho = rho_override ? *rho_override : rho0 / static_cast<double>(m + n);
    if (!(rho > 0) || !std::isfinite(rho))
      fail(Errc::non_positive_rho, "resolved rho must be positive");
    return rho;
  }

  drotb_config to_c() const {
    drotb_config c;
    drotb_config_default(&c);
    c.rho0 = rho0;
    c.has_rho_override = rho_override ? 1 : 0;
    c.rho_override = rho_override ? *rho_override : 0.0;
    c.relative_tolerances = relative_tolerances;
    c.tol_primal = tol_primal;
    c.tol_dual = tol_dual;
    c.tol_gap = tol_gap;
    c.max_iters = max_iters;
    c.check_every = check_every;
    c.engine = engine == EngineKind::reference ? DROTB_ENGINE_REFERENCE : DROTB_ENGINE_FUSED;
    c.skip_cost = skip_cost;
    c.deterministic = deterministic;
    c.record_trace = record_trace;
    c.workers = static_cast<int64_t>(workers);
    c.block_rows = static_cast<int64_t>(block_rows);
    c.work_size = static_cast<int64_t>(work_size);
    c.trace_every = trace_every;
    c.precision = precision == Precision::f32 ? 0 : 1;
    c.device = device;
    c.order = static_cast<int32_t>(order);
    c.use_graphs = use_graphs;
    return c;
  }
};

// fused.hpp:34-81
struct MemoryCounters {
  std::uint64_t passes = 0, xy_elems_read = 0, xy_elems_written = 0, cost_elems_read = 0;
};
template <class T>
struct FusedPassOutput {
  std::vector<T> row_sums, col_sums;
  T cost_dot = T(0);
  bool cost_valid = false;
  T max_abs = T(0);
  bool nonfinite = false;
  T dual_sq = T(0);
  bool dual_valid = false;
  T dx_sq = T(0);
  bool dx_valid = false;
  T prev_cost_dot = T(0);
  bool prev_cost_valid = false;
  T total_mass() const {
    T acc = T(0);
    for (T v : row_sums) acc += v;
    return acc;
  }
};
template <class T>
struct FusedArray {
  Matrix<T> values;
  bool cost_folded = false;
};
struct PassOptions {
  int parity = 0;
  bool want_dual = false;
  bool want_dx = false;
  bool deterministic = true;
  MemoryCounters* counters = nullptr;
};

template <class T>
struct DrotState {
  FusedArray<T> xy;
  std::vector<T> row_shift, col_shift;
  std::vector<T> y_row_defect, y_col_defect;
  T y_mass_gap = T(0);
  std::vector<T> row_residual, col_residual;
  T x_mass_gap = T(0);
  std::int64_t iter = 0;
};

template <class T>
struct SolveResult {
  TransportPlan<T> plan;
  DualCertificate<T> cert;
  ResidualReport report;
  SolveTrace trace;
  SolveStatus status = SolveStatus::max_iters;
};

// ---- tiles.hpp:22-49 ----------------------------------------------------------
struct TilePlan {
  std::size_t rows = 0, cols = 0, block_rows = 64, work_size = 4, workers = 1;
  std::size_t grid_rows = 0, grid_cols = 0;
  std::size_t tile_cols() const { return work_size * block_rows; }
};
inline TilePlan plan_tiles(std::size_t m, std::size_t n, std::size_t bs, std::size_t ws,
                           std::size_t workers) {
  TilePlan p;
  p.rows = m;
  p.cols = n;
  p.block_rows = bs ? bs : 1;
  p.work_size = ws ? ws : 1;
  p.workers = workers ? workers : 1;
  p.grid_rows = (m + p.block_rows - 1) / p.block_rows;
  p.grid_cols = (n + p.tile_cols() - 1) / p.tile_cols();
  return p;
}

// ---- problem.hpp:122-136 --------------------------------------------------------
template <class T>
void check_problem(const TransportProblem<T>& pr) {
  if (pr.m() == 0 || pr.n() == 0) fail(Errc::empty_dimension, "cost matrix has an empty dimension");
  if (pr.p.size() != pr.m() || pr.q.size() != pr.n())
    fail(Errc::shape_mismatch, "marginal lengths do not match the cost matrix");
  const auto m = static_cast<int64_t>(pr.m()), n = static_cast<int64_t>(pr.n());
  if constexpr (detail::is_f32<T>)
    detail::check(drotb_check_problem_f32(pr.cost.data(), m, n, pr.p.data(), pr.q.data()));
  else
    detail::check(drotb_check_problem_f64(pr.cost.data(), m, n, pr.p.data(), pr.q.data()));
}

// ---- problem.hpp:155-225 (evaluated on the B200) --------------------------------
template <class T>
ResidualReport residual_report(const TransportProblem<T>& pr, const TransportPlan<T>& plan,
                               const DualCertificate<T>& cert) {
  if (plan.x.rows() != pr.m() || plan.x.cols() != pr.n())
    fail(Errc::shape_mismatch, "residual_report: plan vs cost");
  if (cert.mu.size() != pr.m() || cert.nu.size() != pr.n())
    fail(Errc::shape_mismatch, "residual_report: dual lengths");
  const auto m = static_cast<int64_t>(pr.m()), n = static_cast<int64_t>(pr.n());
  drotb_report r{};
  // exact = 1: the reference's summation order, bitwise equal report
  if constexpr (detail::is_f32<T>)
    detail::check(drotb_residual_report_f32(pr.cost.data(), m, n, pr.p.data(), pr.q.data(),
                                            plan.x.data(), cert.mu.data(), cert.nu.data(), 1, &r));
  else
    detail::check(drotb_residual_report_f64(pr.cost.data(), m, n, pr.p.data(), pr.q.data(),
                                            plan.x.data(), cert.mu.data(), cert.nu.data(), 1, &r));
  return ResidualReport{r.r_primal, r.r_dual, r.gap, r.objective};
}

template <class T>
double objective(const TransportProblem<T>& pr, const TransportPlan<T>& plan) {
  DualCertificate<T> zero;
  zero.mu.assign(pr.m(), T(0));
  zero.nu.assign(pr.n(), T(0));
  return residual_report(pr, plan, zero).objective;
}

// ---- reference.hpp:165-288: the Sinkhorn baseline on the B200 -----------------------
template <class T>
SolveResult<T> sinkhorn_solve(const TransportProblem<T>& pr, T eta, double tol,
                              std::int64_t max_iters, std::int64_t check_every = 10) {
  const std::size_t m = pr.m(), n = pr.n();
  if (m == 0 || n == 0) fail(Errc::empty_dimension, "cost matrix has an empty dimension");
  SolveResult<T> res;
  res.plan.x = Matrix<T>(m, n);
  res.cert.mu.assign(m, T(0));
  res.cert.nu.assign(n, T(0));
  res.cert.rho = eta;
  const std::int64_t ce = check_every < 1 ? 1 : check_every;
  const std::int64_t cap = (max_iters > 0 ? max_iters : 0) / ce + 2;
  std::vector<drotb_trace_row> tr(static_cast<std::size_t>(cap));
  drotb_report r{};
  int64_t tlen = 0, iters = 0;
  int32_t status = 0;
  double wall = 0;
  const auto mi = static_cast<int64_t>(m), ni = static_cast<int64_t>(n);
  if constexpr (detail::is_f32<T>)
    detail::check(drotb_sinkhorn_f32(pr.cost.data(), mi, ni, pr.p.data(), pr.q.data(), eta, tol,
                                     max_iters, ce, 0, res.plan.x.data(), res.cert.mu.data(),
                                     res.cert.nu.data(), &r, tr.data(), cap, &tlen, &iters,
                                     &status, &wall));
  else
    detail::check(drotb_sinkhorn_f64(pr.cost.data(), mi, ni, pr.p.data(), pr.q.data(), eta, tol,
                                     max_iters, ce, 0, res.plan.x.data(), res.cert.mu.data(),
                                     res.cert.nu.data(), &r, tr.data(), cap, &tlen, &iters,
                                     &status, &wall));
  res.report = ResidualReport{r.r_primal, r.r_dual, r.gap, r.objective};
  res.status = static_cast<SolveStatus>(status);
  res.trace.termination = res.status;
  res.trace.iterations = iters;
  res.trace.wall_time_s = wall;
  for (int64_t k = 0; k < tlen && k < cap; ++k)
    res.trace.rows.push_back(TraceRow{tr[k].iter, tr[k].r_primal, tr[k].r_dual, tr[k].gap,
                                      tr[k].objective, tr[k].ergodic_objective,
                                      tr[k].fixed_point_residual});
  return res;
}

// ---- solver.hpp:143-186 / 361-370 / 372-540 -------------------------------------
template <class T>
DrotState<T> init_state(const TransportProblem<T>& pr, const DrotConfig& cfg,
                        const Matrix<T>* x0 = nullptr) {
  const std::size_t m = pr.m(), n = pr.n();
  if (x0 && (x0->rows() != m || x0->cols() != n)) fail(Errc::shape_mismatch, "initial plan shape");
  DrotState<T> st;
  st.xy.values = Matrix<T>(m, n);
  st.row_shift.assign(m, T(0));
  st.col_shift.assign(n, T(0));
  st.y_row_defect.assign(m, T(0));
  st.y_col_defect.assign(n, T(0));
  st.row_residual.assign(m, T(0));
  st.col_residual.assign(n, T(0));
  int32_t folded = 0;
  const drotb_config c = cfg.to_c();
  const auto mi = static_cast<int64_t>(m), ni = static_cast<int64_t>(n);
  if constexpr (detail::is_f32<T>)
    detail::check(drotb_init_state_f32(
        st.xy.values.data(), &folded, st.row_shift.data(), st.col_shift.data(),
        st.y_row_defect.data(), st.y_col_defect.data(), &st.y_mass_gap, st.row_residual.data(),
        st.col_residual.data(), &st.x_mass_gap, &st.iter, pr.cost.data(), mi, ni, pr.p.data(),
        pr.q.data(), x0 ? x0->data() : nullptr, &c));
  else
    detail::check(drotb_init_state_f64(
        st.xy.values.data(), &folded, st.row_shift.data(), st.col_shift.data(),
        st.y_row_defect.data(), st.y_col_defect.data(), &st.y_mass_gap, st.row_residual.data(),
        st.col_residual.data(), &st.x_mass_gap, &st.iter, pr.cost.data(), mi, ni, pr.p.data(),
        pr.q.data(), x0 ? x0->data() : nullptr, &c));
  st.xy.cost_folded = folded != 0;
  return st;
}

template <class T>
void drot_step(DrotState<T>& st, const TransportProblem<T>& pr, const DrotConfig& cfg) {
  int32_t folded = st.xy.cost_folded ? 1 : 0;
  const drotb_config c = cfg.to_c();
  const auto mi = static_cast<int64_t>(pr.m()), ni = static_cast<int64_t>(pr.n());
  int rc;
  if constexpr (detail::is_f32<T>)
    rc = drotb_step_f32(st.xy.values.data(), &folded, st.row_shift.data(), st.col_shift.data(),
                        st.y_row_defect.data(), st.y_col_defect.data(), &st.y_mass_gap,
                        st.row_residual.data(), st.col_residual.data(), &st.x_mass_gap,
                        &st.iter, pr.cost.data(), mi, ni, pr.p.data(), pr.q.data(), &c);
  else
    rc = drotb_step_f64(st.xy.values.data(), &folded, st.row_shift.data(), st.col_shift.data(),
                        st.y_row_defect.data(), st.y_col_defect.data(), &st.y_mass_gap,
                        st.row_residual.data(), st.col_residual.data(), &st.x_mass_gap,
                        &st.iter, pr.cost.data(), mi, ni, pr.p.data(), pr.q.data(), &c);
  st.xy.cost_folded = folded != 0;
  detail::check(rc);
}

template <class T>
SolveResult<T> solve(const TransportProblem<T>& pr, const DrotConfig& cfg,
                     const Matrix<T>* x0 = nullptr) {
  const std::size_t m = pr.m(), n = pr.n();
  if (m == 0 || n == 0) fail(Errc::empty_dimension, "cost matrix has an empty dimension");
  if (pr.p.size() != m || pr.q.size() != n)
    fail(Errc::shape_mismatch, "marginal lengths do not match the cost matrix");
  if (x0 && (x0->rows() != m || x0->cols() != n)) fail(Errc::shape_mismatch, "initial plan shape");
  SolveResult<T> res;
  res.plan.x = Matrix<T>(m, n);
  res.cert.mu.assign(m, T(0));
  res.cert.nu.assign(n, T(0));
  std::int64_t cap = 0;
  if (cfg.record_trace) {
    const std::int64_t te = cfg.trace_every > 0 ? cfg.trace_every : 1;
    cap = (cfg.max_iters > 0 ? cfg.max_iters : 0) / te + 1;
  }
  std::vector<drotb_trace_row> rows(static_cast<std::size_t>(cap ? cap : 1));
  drotb_report rep{};
  std::int64_t tlen = 0, iters = 0;
  int32_t status = 0;
  double wall = 0;
  const drotb_config c = cfg.to_c();
  const auto mi = static_cast<int64_t>(m), ni = static_cast<int64_t>(n);
  if constexpr (detail::is_f32<T>)
    detail::check(drotb_solve_f32(pr.cost.data(), mi, ni, pr.p.data(), pr.q.data(), &c,
                                  x0 ? x0->data() : nullptr, res.plan.x.data(),
                                  res.cert.mu.data(), res.cert.nu.data(), &res.cert.rho, &rep,
                                  rows.data(), cap, &tlen, &iters, &status, &wall));
  else
    detail::check(drotb_solve_f64(pr.cost.data(), mi, ni, pr.p.data(), pr.q.data(), &c,
                                  x0 ? x0->data() : nullptr, res.plan.x.data(),
                                  res.cert.mu.data(), res.cert.nu.data(), &res.cert.rho, &rep,
                                  rows.data(), cap, &tlen, &iters, &status, &wall));
  res.report = ResidualReport{rep.r_primal, rep.r_dual, rep.gap, rep.objective};
  res.status = static_cast<SolveStatus>(status);
  res.trace.termination = res.status;
  res.trace.iterations = iters;
  res.trace.wall_time_s = wall;
  const std::int64_t cnt = tlen < cap ? tlen : cap;
  res.trace.rows.reserve(static_cast<std::size_t>(cnt));
  for (std::int64_t k = 0; k < cnt; ++k) {
    const auto& r = rows[static_cast<std::size_t>(k)];
    res.trace.rows.push_back(TraceRow{r.iter, r.r_primal, r.r_dual, r.gap, r.objective,
                                      r.ergodic_objective, r.fixed_point_residual});
  }
  return res;
}

template <class T>
DualCertificate<T> recover_duals(const DrotState<T>& st, T rho) {
  DualCertificate<T> cert;
  cert.rho = rho;
  for (T v : st.row_shift) cert.mu.push_back(v / rho);
  for (T v : st.col_shift) cert.nu.push_back(v / rho);
  return cert;
}

// ---- fused.hpp:107-202: the engine on the device ----------------------------------
template <class T>
class FusedEngine {
 public:
  explicit FusedEngine(TilePlan plan, int device = -1) : plan_(plan) {
    drotb_engine* e = nullptr;
    detail::check(drotb_engine_create(&e, static_cast<int64_t>(plan.rows),
                                      static_cast<int64_t>(plan.cols),
                                      static_cast<int64_t>(plan.block_rows),
                                      static_cast<int64_t>(plan.work_size),
                                      detail::is_f32<T> ? 0 : 1, device));
    eng_.reset(e);
  }
  const TilePlan& plan() const { return plan_; }

  FusedPassOutput<T> fused_pass(Matrix<T>& xy, const Matrix<T>& cost,
                                const std::vector<T>& row_shift,
                                const std::vector<T>& col_shift, T rho,
                                const PassOptions& opts = {}) {
    return run(xy, cost, row_shift, col_shift, rho, DROTB_PASS_FUSED, 0, nullptr, opts);
  }
  FusedPassOutput<T> fused_pass_skip_cost(FusedArray<T>& xy, const Matrix<T>& cost,
                                          const std::vector<T>& row_shift,
                                          const std::vector<T>& col_shift, T rho, bool fold,
                                          PassOptions opts = {}) {
    int32_t folded = xy.cost_folded ? 1 : 0;
    auto out = run(xy.values, cost, row_shift, col_shift, rho, DROTB_PASS_SKIP_COST,
                   fold ? 1 : 0, &folded, opts);
    xy.cost_folded = folded != 0;
    return out;
  }
  FusedPassOutput<T> unfused_pass(Matrix<T>& xy, const Matrix<T>& cost,
                                  const std::vector<T>& row_shift,
                                  const std::vector<T>& col_shift, T rho,
                                  const PassOptions& opts = {}) {
    return run(xy, cost, row_shift, col_shift, rho, DROTB_PASS_UNFUSED, 0, nullptr, opts);
  }

 private:
  struct Del {
    void operator()(drotb_engine* e) const { drotb_engine_destroy(e); }
  };
  FusedPassOutput<T> run(Matrix<T>& xy, const Matrix<T>& cost, const std::vector<T>& rs,
                         const std::vector<T>& cs, T rho, int32_t kind, int32_t fold,
                         int32_t* folded, const PassOptions& opts) {
    if (xy.rows() != plan_.rows || xy.cols() != plan_.cols)
      fail(Errc::shape_mismatch, "fused pass: array vs tile plan");
    if (!xy.same_shape(cost)) fail(Errc::shape_mismatch, "fused pass: cost");
    if (rs.size() != plan_.rows || cs.size() != plan_.cols)
      fail(Errc::shape_mismatch, "fused pass: shift vectors");
    FusedPassOutput<T> o;
    o.row_sums.assign(plan_.rows, T(0));
    o.col_sums.assign(plan_.cols, T(0));
    drotb_pass_out po{};
    drotb_counters ctr{};
    if (opts.counters) {
      ctr.passes = opts.counters->passes;
      ctr.xy_elems_read = opts.counters->xy_elems_read;
      ctr.xy_elems_written = opts.counters->xy_elems_written;
      ctr.cost_elems_read = opts.counters->cost_elems_read;
    }
    int32_t dummy = 0;
    if constexpr (detail::is_f32<T>)
      detail::check(drotb_engine_pass_f32(eng_.get(), xy.data(), cost.data(), rs.data(),
                                          cs.data(), rho, kind, fold, folded ? folded : &dummy,
                                          opts.parity, opts.want_dual, opts.want_dx,
                                          opts.deterministic, o.row_sums.data(),
                                          o.col_sums.data(), &po, &ctr));
    else
      detail::check(drotb_engine_pass_f64(eng_.get(), xy.data(), cost.data(), rs.data(),
                                          cs.data(), rho, kind, fold, folded ? folded : &dummy,
                                          opts.parity, opts.want_dual, opts.want_dx,
                                          opts.deterministic, o.row_sums.data(),
                                          o.col_sums.data(), &po, &ctr));
    if (opts.counters) {
      opts.counters->passes = ctr.passes;
      opts.counters->xy_elems_read = ctr.xy_elems_read;
      opts.counters->xy_elems_written = ctr.xy_elems_written;
      opts.counters->cost_elems_read = ctr.cost_elems_read;
    }
    o.cost_dot = static_cast<T>(po.cost_dot);
    o.cost_valid = po.cost_valid;
    o.max_abs = static_cast<T>(po.max_abs);
    o.nonfinite = po.nonfinite;
    o.dual_sq = static_cast<T>(po.dual_sq);
    o.dual_valid = po.dual_valid;
    o.dx_sq = static_cast<T>(po.dx_sq);
    o.dx_valid = po.dx_valid;
    o.prev_cost_dot = static_cast<T>(po.prev_cost_dot);
    o.prev_cost_valid = po.prev_cost_valid;
    return o;
  }
  TilePlan plan_;
  std::unique_ptr<drotb_engine, Del> eng_;
};

}  // namespace drot

#endif  // DROT_B200_DROT_HPP_
