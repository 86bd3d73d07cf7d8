"""The persistent solver kernel (fast order, one GPU; csrc/persistent.cu)
against the per-launch kernel path (K1 + merge + update + graph IF node,
selected with DROTB_PERSIST=0) and against itself:

* the first iteration sees identical inputs on both paths, so X after one
  iteration is bitwise equal (same elementwise arithmetic);
* splitting K iterations over several launches is bitwise equal to one
  launch (the schedule and every reduction order are static);
* solves to tolerance agree with the per-launch path and the reference to
  the fast-order tolerances (status, iterations within max(5, 0.5 %),
  objective rel 1e-5 fp64 / 1e-3 fp32).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _session(drot, m, n, dt, persist=True, **kw):
    old = os.environ.get("DROTB_PERSIST")
    os.environ["DROTB_PERSIST"] = "1" if persist else "0"
    try:
        s = drot.Session(m, n, dt, drot.DrotConfig(**kw))
    finally:
        if old is None:
            del os.environ["DROTB_PERSIST"]
        else:
            os.environ["DROTB_PERSIST"] = old
    assert (s.persistent_grid > 0) == persist
    return s


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("shape", [(1000, 700), (777, 333), (64, 3000), (5000, 40)])
def test_first_iteration_bitwise(drot, dt, shape):
    m, n = shape
    xs = []
    for persist in (True, False):
        s = _session(drot, m, n, dt, persist, tol_primal=-1.0, max_iters=10 ** 9)
        s.gen_gaussian(5.0, 1, "dyadic")
        s.init()
        s.enqueue(1)
        s.synchronize()
        st, it, _ = s.status()
        assert it == 1
        xs.append(s.plan()[0])
        s.close()
    np.testing.assert_array_equal(xs[0], xs[1])


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_split_launches_bitwise(drot, dt):
    m, n = 900, 800
    outs = []
    for chunks in ([10], [3, 3, 4], [1] * 10):
        s = _session(drot, m, n, dt, True, tol_primal=-1.0, max_iters=10 ** 9)
        s.gen_gaussian(5.0, 2, "dyadic")
        s.init()
        for c in chunks:
            s.enqueue(c)
        s.synchronize()
        st, it, rep = s.status()
        assert it == 10
        plan, mu, nu = s.plan()
        outs.append((plan, mu, nu, rep.objective))
        s.close()
    for o in outs[1:]:
        np.testing.assert_array_equal(o[0], outs[0][0])
        np.testing.assert_array_equal(o[1], outs[0][1])
        np.testing.assert_array_equal(o[2], outs[0][2])
        assert o[3] == outs[0][3]


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_solve_matches_per_launch_path(drot, dt):
    m, n = 600, 500
    res = []
    for persist in (True, False):
        s = _session(drot, m, n, dt, persist, max_iters=60000)
        s.gen_gaussian(5.0, 0, "dyadic")
        s.init()
        s.run()
        res.append(s.status())
        s.close()
    (st1, it1, r1), (st2, it2, r2) = res
    assert st1 == st2 == drot.SolveStatus.converged
    assert abs(it1 - it2) <= max(5, int(0.005 * it2))
    rel = 1e-5 if dt == np.float64 else 1e-3
    assert abs(r1.objective - r2.objective) <= rel * abs(r2.objective)
    for v in (r1.r_primal, r1.r_dual, r1.gap):
        assert v <= 1e-4


def test_trace_rows_match_per_launch_path(drot):
    m, n = 300, 200
    rows = []
    for persist in (True, False):
        old = os.environ.get("DROTB_PERSIST")
        os.environ["DROTB_PERSIST"] = "1" if persist else "0"
        try:
            C = np.asfortranarray(drot.random_matrix(m, n, 5))
            prob = drot.TransportProblem(C, np.full(m, 1.0 / m), np.full(n, 1.0 / n))
            r = drot.solve(prob, drot.DrotConfig(max_iters=500, tol_primal=-1.0))
        finally:
            if old is None:
                del os.environ["DROTB_PERSIST"]
            else:
                os.environ["DROTB_PERSIST"] = old
        rows.append(r.trace.rows)
    assert len(rows[0]) == len(rows[1]) == 500
    for a, b in zip(rows[0], rows[1]):
        assert a.iter == b.iter
        for k in ("r_primal", "r_dual", "gap", "objective", "ergodic_objective",
                  "fixed_point_residual"):
            x, y = getattr(a, k), getattr(b, k)
            tol = 1e-6 if k == "fixed_point_residual" else 1e-9
            assert x == y or (np.isnan(x) and np.isnan(y)) or \
                abs(x - y) <= tol * max(1e-12, abs(y)), (a.iter, k, x, y)
