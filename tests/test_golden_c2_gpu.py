"""The headline fp32 fast path against the reference's own trajectory at C2
(m = n = 10 000 fp32, Gaussian seed 0, dyadic marginals, reference defaults,
tol 1e-4): tests/golden/c2_f32.json was produced on a B200 by
tests/golden/make_c2_golden.py in order=reference -- bitwise the reference's
solve<float> (solver.hpp:372-540), which the CPU would need ~2.5 h for.

Tolerances (SURVEY §8(c), fp32 fast order vs the reference): same status;
iterations within max(5, 0.5 %); objective relative 1e-4 (observed 2.3e-6);
support {x > 1e-6 max x} symmetric difference <= 1 % (observed 0.4 %); the
trace (objective, ergodic objective) within 1e-3 relative at every 10 000th
iteration."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLD, "c2_f32.json")) as f:
        g = json.load(f)
    g["support"] = np.load(os.path.join(GOLD, "c2_f32_support.npy")).astype(np.int64)
    return g


def test_c2_fast_order_matches_reference_trajectory(drot, gold):
    m = n = 10000
    prob = drot.gen_gaussian_problem_as(drot.GaussianSpec(m, n, 5.0, 0), np.float32)
    prob = drot.TransportProblem(prob.cost, drot.dyadic_marginal(m, np.float32),
                                 drot.dyadic_marginal(n, np.float32))
    res = drot.solve(prob, drot.DrotConfig(max_iters=gold["spec"]["cfg"]["max_iters"]))
    drot.release_device_cache()
    st, iters, rep, plan, rows = res.status, res.trace.iterations, res.report, res.plan.x, \
        res.trace.rows
    assert st.name == gold["status"] == "converged"
    it = gold["iterations"]
    assert abs(iters - it) <= max(5, it // 200), (iters, it)
    obj = gold["report_float"]["objective"]
    assert abs(rep.objective - obj) <= 1e-4 * abs(obj), (rep.objective, obj)
    for k in ("r_primal", "r_dual", "gap"):
        assert getattr(rep, k) <= 1e-4  # converged at the same tolerances
    x = plan.ravel(order="F")
    supp = np.flatnonzero(x > 1e-6 * float(x.max()))
    sym = np.setxor1d(supp, gold["support"], assume_unique=True).size
    assert sym <= 0.01 * gold["support"].size, (sym, gold["support"].size)
    by_iter = {r.iter: r for r in rows}
    for g in gold["trace_every_10000"][1:]:
        r = by_iter.get(int(g[0]))
        if r is None:
            continue
        assert abs(r.objective - g[4]) <= 1e-3 * abs(g[4]), (r.iter, r.objective, g[4])
        assert abs(r.ergodic_objective - g[5]) <= 1e-3 * abs(g[5]), (r.iter, r.ergodic_objective)
