// Reference-style client of the API surface around the solve path, compiled
// unchanged-style against the drop-in headers (-I include/drot_b200, C++20)
// and run on the B200: validation (problem.hpp:96-154), materialize_plan /
// materialize_y (solver.hpp:204-230), ErgodicMean (:127-139), the engine's
// pool constructor (fused.hpp:110-113), tile plans (tiles.cpp:20-47), the
// Gaussian generator (probgen.hpp:131-180).  Build: tests/cpp/Makefile.
#include <cmath>
#include <limits>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "doctest.h"
#include "drot/fused.hpp"
#include "drot/probgen.hpp"
#include "drot/problem.hpp"
#include "drot/solver.hpp"
#include "drot/tiles.hpp"

using drot::Errc;
using drot::Matrix;
using drot::TransportProblem;

namespace {

TransportProblem<double> two_by_two() {
  TransportProblem<double> pr;
  pr.cost = Matrix<double>::from_rows({{0, 1}, {1, 0}});
  pr.p = {0.5, 0.5};
  pr.q = {0.5, 0.5};
  return pr;
}

TransportProblem<double> random_problem(std::size_t m, std::size_t n, std::uint64_t seed) {
  drot::CounterRng rng(seed);
  TransportProblem<double> pr;
  pr.cost = Matrix<double>(m, n);
  for (double& c : pr.cost.flat()) c = rng.next_unit();
  pr.p.assign(m, 1.0 / static_cast<double>(m));
  pr.q.assign(n, 1.0 / static_cast<double>(n));
  return pr;
}

}  // namespace

TEST_CASE("validate: accepts, rejects off-simplex, renormalizes on request") {
  CHECK_NOTHROW(drot::validate_problem(two_by_two()));
  auto bad = two_by_two();
  bad.p = {0.6, 0.6};
  try {
    drot::validate_problem(bad);
    FAIL("expected marginal_not_simplex");
  } catch (const drot::Error& e) {
    CHECK(e.code() == Errc::marginal_not_simplex);
    CHECK(std::string(e.what()).find("1.2") != std::string::npos);
  }
  drot::ValidateOptions opts;
  opts.renormalize = true;
  auto fixed = drot::validate_problem(bad, opts);
  CHECK(fixed.p[0] == 0.5);
  CHECK(fixed.p[1] == 0.5);
  auto neg = two_by_two();
  neg.cost(0, 1) = -1.0;
  CHECK_THROWS_WITH_AS(drot::validate_problem(neg), doctest::Contains("negative"), drot::Error);
  auto nan = two_by_two();
  nan.cost(1, 0) = std::numeric_limits<double>::quiet_NaN();
  try {
    drot::validate_problem(nan);
    FAIL("expected non_finite_entry");
  } catch (const drot::Error& e) {
    CHECK(e.code() == Errc::non_finite_entry);
  }
}

TEST_CASE("check_problem honours simplex_tol") {
  auto pr = two_by_two();
  pr.q = {0.5, 0.5005};
  CHECK_THROWS_AS(drot::check_problem(pr), drot::Error);
  CHECK_NOTHROW(drot::check_problem(pr, 1e-3));
  // fp32 uniform thirds: off the 1e-12 simplex in double, inside 1e-6
  TransportProblem<float> pf;
  pf.cost = Matrix<float>(3, 3, 0.5f);
  pf.p.assign(3, 1.0f / 3.0f);
  pf.q.assign(3, 1.0f / 3.0f);
  CHECK_THROWS_AS(drot::check_problem(pf), drot::Error);
  CHECK_NOTHROW(drot::check_problem(pf, 1e-6));
}

TEST_CASE("materialize_plan / materialize_y on a drot_step state") {
  const std::size_t m = 37, n = 29;
  auto pr = random_problem(m, n, 21);
  drot::DrotConfig cfg;
  cfg.order = drot::Order::reference;
  const double rho = cfg.resolved_rho(m, n);
  auto st = drot::init_state(pr, cfg);
  for (int k = 0; k < 5; ++k) drot::drot_step(st, pr, cfg);
  REQUIRE(st.xy.cost_folded);  // skip_cost: odd step count leaves X - rho C
  auto plan = drot::materialize_plan(st, pr.cost, rho);
  for (std::size_t k = 0; k < plan.x.size(); ++k) {
    const double v = st.xy.values.data()[k] + rho * pr.cost.data()[k];
    CHECK(plan.x.data()[k] == (v > 0 ? v : 0.0));
  }
  auto y = drot::materialize_y(st, pr.cost, rho);
  for (std::size_t j = 0; j < n; ++j)
    for (std::size_t i = 0; i < m; ++i)
      CHECK(y(i, j) == plan.x(i, j) + (st.row_shift[i] + st.col_shift[j]));
  drot::drot_step(st, pr, cfg);
  REQUIRE(!st.xy.cost_folded);
  auto plain = drot::materialize_plan(st, pr.cost, rho);
  for (std::size_t k = 0; k < plain.x.size(); ++k)
    CHECK(plain.x.data()[k] == st.xy.values.data()[k]);
  // the maintained identity step_impl asserts in debug builds
  // (solver.hpp:293-304): a = Y e - p
  auto ye = drot::row_sums(drot::materialize_y(st, pr.cost, rho));
  for (std::size_t i = 0; i < m; ++i) {
    const double rhs = ye[i] - pr.p[i];
    CHECK(std::abs(st.y_row_defect[i] - rhs) <= 1e-9 * (1.0 + std::abs(rhs)));
  }
}

TEST_CASE("ErgodicMean is the running mean") {
  drot::ErgodicMean em;
  CHECK(em.count() == 0);
  em.update(1.0);
  em.update(2.0);
  em.update(6.0);
  CHECK(em.count() == 3);
  CHECK(em.mean() == doctest::Approx(3.0).epsilon(1e-15));
}

TEST_CASE("engine accepts a shared pool and reports it") {
  auto pool = std::make_shared<drot::ThreadPool>(4);
  auto pr = random_problem(9, 7, 5);
  drot::FusedEngine<double> eng(drot::plan_tiles(9, 7, 2, 1, 4), pool);
  CHECK(&eng.pool() == pool.get());
  CHECK(eng.pool().workers() == 4);
  CHECK(eng.plan().tiles.size() == eng.plan().grid_rows * eng.plan().grid_cols);
  Matrix<double> xy(9, 7, 0.01);
  std::vector<double> phi(9, 0.001), varphi(7, -0.002);
  auto out = eng.fused_pass(xy, pr.cost, std::span<const double>(phi),
                            std::span<const double>(varphi), 0.01);
  CHECK(out.total_mass() == doctest::Approx(drot::vec_sum(std::span<const double>(out.col_sums))).epsilon(1e-12));
  drot::FusedEngine<double> own(drot::plan_tiles(9, 7, 64, 4, 0));
  CHECK(own.pool().workers() == 1);
}

TEST_CASE("gaussian instance: generator, fp32 cast, fast-order solve") {
  drot::GaussianSpec spec;
  spec.m = 120;
  spec.n = 96;
  auto pd = drot::gen_gaussian_problem(spec);
  auto pf = drot::gen_gaussian_problem_as<float>(spec);
  CHECK(pd.cost.rows() == 120);
  CHECK(pf.cost.cols() == 96);
  double cmax = 0;
  for (double c : pd.cost.flat()) cmax = std::max(cmax, c);
  CHECK(cmax == 1.0);
  for (std::size_t k = 0; k < pd.cost.size(); ++k)
    CHECK(pf.cost.data()[k] == static_cast<float>(pd.cost.data()[k]));
  drot::DrotConfig cfg;
  auto res = drot::solve(pd, cfg);
  CHECK(res.status == drot::SolveStatus::converged);
  auto rep = drot::residual_report(pd, res.plan, res.cert);
  CHECK(rep.r_primal <= 1e-4);
  CHECK(rep.objective == doctest::Approx(res.report.objective).epsilon(1e-9));
}
