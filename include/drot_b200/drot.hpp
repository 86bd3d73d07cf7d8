// drot_b200/drot.hpp -- source-compatible drop-in for the reference's
// umbrella header drot/drot.hpp (proj/core/include/drot/drot.hpp:17-27),
// restricted to the solve path.  Code written against
//   drot::solve<T>, drot::drot_step<T>, drot::init_state<T>,
//   drot::FusedEngine<T>, drot::check_problem, drot::DrotConfig, ...
// compiles unchanged against this header (swap the include path, link
// libdrotb200.so) and runs on a B200.  Every array-sized computation goes
// through the C ABI of include/drotb.h; the types below mirror the
// reference's field for field (cited per type).  The small host helpers
// (Matrix, vec_*, row_sums / col_sums, ErgodicMean, ThreadPool) are the
// reference's value-type utilities, kept so that client code written against
// them compiles; the solver never calls them.  Header-only; C++20 (std::span,
// as the reference).
#ifndef DROT_B200_DROT_HPP_
#define DROT_B200_DROT_HPP_

#if __cplusplus < 202002L
#error "drot_b200/drot.hpp mirrors the reference's C++20 API (std::span): build with -std=c++20"
#endif

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <initializer_list>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
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
  std::span<T> flat() { return std::span<T>(data_); }
  std::span<const T> flat() const { return std::span<const T>(data_); }
  bool same_shape(const Matrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }
  template <class U>
  Matrix<U> cast() const {  // element-wise static_cast, storage order
    Matrix<U> out(rows_, cols_);
    std::transform(data_.begin(), data_.end(), out.data(),
                   [](T v) { return static_cast<U>(v); });
    return out;
  }

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<T> data_;
};

template <class T>
void require_same_shape(const Matrix<T>& a, const Matrix<T>& b, const char* where) {
  if (!a.same_shape(b)) fail(Errc::shape_mismatch, where);
}

// ---- matrix.hpp:93-158: host vector helpers, ascending-index order ---------
template <class T>
T vec_sum(std::span<const T> x) {
  T s = T(0);
  for (std::size_t k = 0; k < x.size(); ++k) s += x[k];
  return s;
}
template <class T>
T vec_dot(std::span<const T> x, std::span<const T> y) {
  T s = T(0);
  for (std::size_t k = 0; k < x.size(); ++k) s += x[k] * y[k];
  return s;
}
template <class T>
T vec_norm_sq(std::span<const T> x) {
  T s = T(0);
  for (std::size_t k = 0; k < x.size(); ++k) s += x[k] * x[k];
  return s;
}
template <class T>
bool all_finite(std::span<const T> x) {
  return std::all_of(x.begin(), x.end(),
                     [](T v) { return std::isfinite(static_cast<double>(v)); });
}
template <class T>
std::vector<T> row_sums(const Matrix<T>& x) {  // X e, column by column
  std::vector<T> u(x.rows(), T(0));
  for (std::size_t j = 0; j < x.cols(); ++j)
    for (std::size_t i = 0; i < x.rows(); ++i) u[i] += x(i, j);
  return u;
}
template <class T>
std::vector<T> col_sums(const Matrix<T>& x) {  // X' f, one chain per column
  std::vector<T> v(x.cols(), T(0));
  for (std::size_t j = 0; j < x.cols(); ++j) {
    T s = T(0);
    for (std::size_t i = 0; i < x.rows(); ++i) s += x(i, j);
    v[j] = s;
  }
  return v;
}
template <class T>
T frobenius_dot(const Matrix<T>& a, const Matrix<T>& b) {
  return vec_dot(std::span<const T>(a.flat()), std::span<const T>(b.flat()));
}
template <class T>
T frobenius_norm_sq(const Matrix<T>& a) {
  return vec_norm_sq(std::span<const T>(a.flat()));
}
template <class T>
double frobenius_distance(const Matrix<T>& a, const Matrix<T>& b) {
  double s = 0;
  for (std::size_t k = 0; k < a.size(); ++k) {
    const double d = static_cast<double>(a.data()[k]) - static_cast<double>(b.data()[k]);
    s += d * d;
  }
  return std::sqrt(s);
}

// ---- rng.hpp:30-106: the counter-based generator behind every synthetic
// input (SplitMix64 finalizer over key + k * golden gamma).  The host and
// device generators (csrc/probgen.cpp / probgen.cu) restate the same stream.
class CounterRng {
 public:
  explicit CounterRng(std::uint64_t key) : key_(key) {}
  static std::uint64_t mix(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  static std::uint64_t derive_key(std::uint64_t key, std::uint64_t stream) {
    return mix(key ^ mix(stream + kGamma));
  }
  CounterRng substream(std::uint64_t stream) const { return CounterRng(derive_key(key_, stream)); }
  std::uint64_t next_u64() { return mix(key_ + (ctr_ += kGamma)); }
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_unit_open() { return (static_cast<double>(next_u64() >> 11) + 0.5) * 0x1.0p-53; }
  void next_gaussian_pair(double& z0, double& z1) {  // Marsaglia polar
    while (true) {
      const double a = 2.0 * next_unit() - 1.0;
      const double b = 2.0 * next_unit() - 1.0;
      const double s = a * a + b * b;
      if (!(s > 0.0 && s < 1.0)) continue;
      const double r = std::sqrt(-2.0 * std::log(s) / s);
      z0 = a * r;
      z1 = b * r;
      return;
    }
  }
  double next_gaussian() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    double z0 = 0;
    next_gaussian_pair(z0, spare_);
    spare_ok_ = true;
    return z0;
  }
  std::uint64_t next_below(std::uint64_t bound) {  // rejection, bias-free
    const std::uint64_t floor_ = (0 - bound) % bound;
    std::uint64_t r = next_u64();
    while (r < floor_) r = next_u64();
    return r % bound;
  }

 private:
  static constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ull;
  std::uint64_t key_;
  std::uint64_t ctr_ = 0;
  double spare_ = 0;
  bool spare_ok_ = false;
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

// ---- threadpool.hpp:19-52 ---------------------------------------------------
// The reference's CPU worker pool.  On the B200 the CUDA grid does this
// work, so the pool only keeps the API: run() executes the tasks in order on
// the calling thread (worker index 0); FusedEngine accepts a pool and ignores
// it.
class ThreadPool {
 public:
  explicit ThreadPool(std::size_t workers) : workers_(workers ? workers : 1) {}
  ThreadPool(const ThreadPool&) = delete;
  ThreadPool& operator=(const ThreadPool&) = delete;
  std::size_t workers() const { return workers_; }
  void run(std::size_t n_tasks, const std::function<void(std::size_t, std::size_t)>& fn) {
    for (std::size_t t = 0; t < n_tasks; ++t) fn(t, 0);
  }
  static std::size_t hardware_workers() {
    const unsigned hc = std::thread::hardware_concurrency();
    return hc ? static_cast<std::size_t>(hc) : 1;
  }

 private:
  std::size_t workers_;
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
  std::size_t resolved_workers() const {
    return workers == 0 ? ThreadPool::hardware_workers() : workers;
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

// solver.hpp:127-139: running mean of the per-iterate objectives (the solve
// keeps its own copy of this recursion on the device, csrc/gate.cuh)
class ErgodicMean {
 public:
  void update(double value) {
    count_ += 1;
    mean_ += (value - mean_) / static_cast<double>(count_);
  }
  double mean() const { return mean_; }
  std::int64_t count() const { return count_; }

 private:
  double mean_ = 0;
  std::int64_t count_ = 0;
};

// ---- tiles.hpp:22-49, tiles.cpp:20-47 -----------------------------------------
// The tile list is the reference's reduction order (tile-column-major); the
// device kernels reproduce it from (block_rows, work_size) in order=reference.
struct TileRange {
  std::size_t r0 = 0, r1 = 0;
  std::size_t c0 = 0, c1 = 0;
  std::size_t grid_r = 0, grid_c = 0;
  std::size_t rows() const { return r1 - r0; }
  std::size_t cols() const { return c1 - c0; }
  std::size_t size() const { return rows() * cols(); }
};
struct TilePlan {
  std::size_t rows = 0, cols = 0, block_rows = 64, work_size = 4, workers = 1;
  std::size_t grid_rows = 0, grid_cols = 0;
  std::vector<TileRange> tiles;
  std::size_t tile_cols() const { return work_size * block_rows; }
};
inline TilePlan plan_tiles(std::size_t m, std::size_t n, std::size_t bs, std::size_t ws,
                           std::size_t workers) {
  TilePlan p;
  p.rows = m;
  p.cols = n;
  p.block_rows = std::max<std::size_t>(bs, 1);
  p.work_size = std::max<std::size_t>(ws, 1);
  p.workers = std::max<std::size_t>(workers, 1);
  const std::size_t tc = p.tile_cols();
  p.grid_rows = (m + p.block_rows - 1) / p.block_rows;
  p.grid_cols = (n + tc - 1) / tc;
  p.tiles.resize(p.grid_rows * p.grid_cols);
  std::size_t k = 0;
  for (std::size_t gc = 0; gc < p.grid_cols; ++gc)
    for (std::size_t gr = 0; gr < p.grid_rows; ++gr, ++k) {
      TileRange& t = p.tiles[k];
      t.grid_r = gr;
      t.grid_c = gc;
      t.r0 = gr * p.block_rows;
      t.r1 = std::min(m, t.r0 + p.block_rows);
      t.c0 = gc * tc;
      t.c1 = std::min(n, t.c0 + tc);
    }
  return p;
}

// ---- problem.hpp:96-154 ---------------------------------------------------------
struct ValidateOptions {
  bool renormalize = false;    // rescale marginals to sum exactly to one
  double simplex_tol = 1e-12;  // allowed |sum - 1|
};

// The matrix scan runs on the device (K0, first offending entry in flat
// order); the marginals are checked with the reference's sequential double sum.
template <class T>
void check_problem(const TransportProblem<T>& pr, double simplex_tol = 1e-12) {
  if (pr.m() == 0 || pr.n() == 0) fail(Errc::empty_dimension, "cost matrix has an empty dimension");
  if (pr.p.size() != pr.m() || pr.q.size() != pr.n())
    fail(Errc::shape_mismatch, "marginal lengths do not match the cost matrix");
  const auto m = static_cast<int64_t>(pr.m()), n = static_cast<int64_t>(pr.n());
  if constexpr (detail::is_f32<T>)
    detail::check(drotb_check_problem_tol_f32(pr.cost.data(), m, n, pr.p.data(), pr.q.data(),
                                              simplex_tol));
  else
    detail::check(drotb_check_problem_tol_f64(pr.cost.data(), m, n, pr.p.data(), pr.q.data(),
                                              simplex_tol));
}

// Marginals are divided by their double sum (then cast back to T) only under
// renormalize; the result is then checked like check_problem.
template <class T>
TransportProblem<T> validate_problem(TransportProblem<T> pr, const ValidateOptions& opts = {}) {
  if (opts.renormalize) {
    for (std::vector<T>* marg : {&pr.p, &pr.q}) {
      double total = 0;
      for (T e : *marg) total += static_cast<double>(e);
      if (!(total > 0)) continue;
      for (T& e : *marg) e = static_cast<T>(static_cast<double>(e) / total);
    }
  }
  check_problem(pr, opts.simplex_tol);
  return pr;
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
  const std::int64_t cap =
      std::min<std::int64_t>((max_iters > 0 ? max_iters : 0) / ce + 2, std::int64_t(1) << 23);
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

// ---- probgen.hpp:40-51, 131-180: the synthetic Gaussian instance ------------------
// Bit-identical to the reference generator (same CounterRng substreams);
// on_degenerate = resample is not supported (a degenerate draw fails).
struct GaussianSpec {
  std::size_t m = 0, n = 0;
  double sigma_t = 5.0;
  std::uint64_t seed = 0;
  enum class OnDegenerate { error, resample };
  OnDegenerate on_degenerate = OnDegenerate::error;
  bool dirichlet_marginals = false;
};

inline TransportProblem<double> gen_gaussian_problem(const GaussianSpec& spec) {
  if (spec.m == 0 || spec.n == 0) fail(Errc::empty_dimension, "gen_gaussian_problem");
  TransportProblem<double> pr;
  pr.cost = Matrix<double>(spec.m, spec.n);
  pr.p.assign(spec.m, 0.0);
  pr.q.assign(spec.n, 0.0);
  detail::check(drotb_gen_gaussian(static_cast<int64_t>(spec.m), static_cast<int64_t>(spec.n),
                                   spec.sigma_t, spec.seed, spec.dirichlet_marginals ? 1 : 0,
                                   pr.cost.data(), pr.p.data(), pr.q.data()));
  return pr;
}

template <class T>
TransportProblem<T> gen_gaussian_problem_as(const GaussianSpec& spec) {
  TransportProblem<double> d = gen_gaussian_problem(spec);
  TransportProblem<T> out;
  out.cost = d.cost.template cast<T>();
  out.p.assign(d.p.begin(), d.p.end());
  out.q.assign(d.q.begin(), d.q.end());
  return out;
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
  if (cfg.record_trace) {  // the device trace holds at most 2^23 rows (as the other front ends)
    const std::int64_t te = cfg.trace_every > 0 ? cfg.trace_every : 1;
    cap = std::min<std::int64_t>((cfg.max_iters > 0 ? cfg.max_iters : 0) / te + 1,
                                 std::int64_t(1) << 23);
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

// solver.hpp:204-217: the plan iterate of a state, unfolded (and clamped)
// when the array holds X - rho C; evaluated on the device (K6).
template <class T>
TransportPlan<T> materialize_plan(const DrotState<T>& st, const Matrix<T>& cost, T rho) {
  const Matrix<T>& xy = st.xy.values;
  if (st.xy.cost_folded) require_same_shape(xy, cost, "materialize_plan: array vs cost");
  TransportPlan<T> plan{Matrix<T>(xy.rows(), xy.cols())};
  if (xy.size() == 0) return plan;
  const auto m = static_cast<int64_t>(xy.rows()), n = static_cast<int64_t>(xy.cols());
  const int32_t f = st.xy.cost_folded ? 1 : 0;
  if constexpr (detail::is_f32<T>)
    detail::check(drotb_materialize_plan_f32(xy.data(), f, cost.data(), m, n, rho, plan.x.data()));
  else
    detail::check(drotb_materialize_plan_f64(xy.data(), f, cost.data(), m, n, rho, plan.x.data()));
  return plan;
}

// solver.hpp:219-230: Y_k = X_k + phi e' + f varphi' (tests / diagnostics).
template <class T>
Matrix<T> materialize_y(const DrotState<T>& st, const Matrix<T>& cost, T rho) {
  const Matrix<T>& xy = st.xy.values;
  if (st.xy.cost_folded) require_same_shape(xy, cost, "materialize_y: array vs cost");
  if (st.row_shift.size() != xy.rows() || st.col_shift.size() != xy.cols())
    fail(Errc::shape_mismatch, "materialize_y: shift lengths");
  Matrix<T> y(xy.rows(), xy.cols());
  if (xy.size() == 0) return y;
  const auto m = static_cast<int64_t>(xy.rows()), n = static_cast<int64_t>(xy.cols());
  const int32_t f = st.xy.cost_folded ? 1 : 0;
  if constexpr (detail::is_f32<T>)
    detail::check(drotb_materialize_y_f32(xy.data(), f, cost.data(), st.row_shift.data(),
                                          st.col_shift.data(), m, n, rho, y.data()));
  else
    detail::check(drotb_materialize_y_f64(xy.data(), f, cost.data(), st.row_shift.data(),
                                          st.col_shift.data(), m, n, rho, y.data()));
  return y;
}

// ---- fused.hpp:107-202: the engine on the device ----------------------------------
template <class T>
class FusedEngine {
 public:
  // The pool is accepted for source compatibility (fused.hpp:110-113) and
  // kept for pool(); the passes run on `device` (-1: the current device).
  explicit FusedEngine(TilePlan plan, std::shared_ptr<ThreadPool> pool = nullptr,
                       int device = -1)
      : plan_(std::move(plan)),
        pool_(pool ? std::move(pool) : std::make_shared<ThreadPool>(plan_.workers)) {
    drotb_engine* e = nullptr;
    detail::check(drotb_engine_create(&e, static_cast<int64_t>(plan_.rows),
                                      static_cast<int64_t>(plan_.cols),
                                      static_cast<int64_t>(plan_.block_rows),
                                      static_cast<int64_t>(plan_.work_size),
                                      detail::is_f32<T> ? 0 : 1, device));
    eng_.reset(e);
  }
  const TilePlan& plan() const { return plan_; }
  ThreadPool& pool() { return *pool_; }

  FusedPassOutput<T> fused_pass(Matrix<T>& xy, const Matrix<T>& cost,
                                std::span<const T> row_shift,
                                std::span<const T> col_shift, T rho,
                                const PassOptions& opts = {}) {
    return run(xy, cost, row_shift, col_shift, rho, DROTB_PASS_FUSED, 0, nullptr, opts);
  }
  FusedPassOutput<T> fused_pass_skip_cost(FusedArray<T>& xy, const Matrix<T>& cost,
                                          std::span<const T> row_shift,
                                          std::span<const T> col_shift, T rho, bool fold,
                                          PassOptions opts = {}) {
    if (fold == xy.cost_folded)
      fail(Errc::fold_state_mismatch,
           fold ? "array already stores X - rho C" : "array does not store X - rho C");
    opts.parity = fold ? 0 : 1;
    int32_t folded = xy.cost_folded ? 1 : 0;
    auto out = run(xy.values, cost, row_shift, col_shift, rho, DROTB_PASS_SKIP_COST,
                   fold ? 1 : 0, &folded, opts);
    xy.cost_folded = folded != 0;
    return out;
  }
  FusedPassOutput<T> unfused_pass(Matrix<T>& xy, const Matrix<T>& cost,
                                  std::span<const T> row_shift,
                                  std::span<const T> col_shift, T rho,
                                  const PassOptions& opts = {}) {
    return run(xy, cost, row_shift, col_shift, rho, DROTB_PASS_UNFUSED, 0, nullptr, opts);
  }

 private:
  struct Del {
    void operator()(drotb_engine* e) const { drotb_engine_destroy(e); }
  };
  FusedPassOutput<T> run(Matrix<T>& xy, const Matrix<T>& cost, std::span<const T> rs,
                         std::span<const T> cs, T rho, int32_t kind, int32_t fold,
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
  std::shared_ptr<ThreadPool> pool_;
  std::unique_ptr<drotb_engine, Del> eng_;
};

}  // namespace drot

#endif  // DROT_B200_DROT_HPP_
