// Reference-style client code compiled against the B200 drop-in header
// (include/drot_b200/drot.hpp) instead of the reference's drot/drot.hpp.
// The body is what a user of drot::solve<T> writes (cf. the SPEC example
// "C=[[0,1],[1,0]], p=(0.7,0.3), q=(0.4,0.6), tol=1e-7 -> objective 0.3",
// SPEC.md:209, and test_reference.cpp:14-20 cross_instance).
#include <cstdio>

#include "drot_b200/drot.hpp"

int main() {
  drot::TransportProblem<double> pr;
  pr.cost = drot::Matrix<double>::from_rows({{0.0, 1.0}, {1.0, 0.0}});
  pr.p = {0.7, 0.3};
  pr.q = {0.4, 0.6};
  drot::check_problem(pr);
  drot::DrotConfig cfg;
  cfg.tol_primal = cfg.tol_dual = cfg.tol_gap = 1e-7;
  cfg.order = drot::Order::reference;
  auto res = drot::solve(pr, cfg);
  std::printf("{\"status\": \"%s\", \"iterations\": %lld, \"objective\": %.17g, "
              "\"x00\": %.17g, \"x01\": %.17g, \"x10\": %.17g, \"x11\": %.17g, "
              "\"trace_rows\": %zu}\n",
              drot::to_string(res.status), static_cast<long long>(res.trace.iterations),
              res.report.objective, res.plan.x(0, 0), res.plan.x(0, 1), res.plan.x(1, 0),
              res.plan.x(1, 1), res.trace.rows.size());
  // residual_report of the returned pair, and the Sinkhorn baseline
  // (problem.hpp:174-225, reference.hpp:165-288) through the same header
  auto rep = drot::residual_report(pr, res.plan, res.cert);
  auto sk = drot::sinkhorn_solve(pr, 0.1, 1e-6, 20000);
  std::printf("{\"report_objective\": %.17g, \"sinkhorn_status\": \"%s\", "
              "\"sinkhorn_objective\": %.17g}\n",
              rep.objective, drot::to_string(sk.status), sk.report.objective);
  // errors surface as drot::Error with the reference's codes
  pr.p = {0.5, 0.6};
  try {
    drot::solve(pr, cfg);
    return 2;
  } catch (const drot::Error& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return e.code() == drot::Errc::marginal_not_simplex ? 0 : 3;
  }
}
