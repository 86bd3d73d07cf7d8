"""The single-launch iteration (csrc/iter.cu, DROTB_TAIL=fused; opt-in) --
the sweep with the whole per-iteration tail folded into its prologue and
epilogue -- against the cooperative tail (csrc/tail.cu, the default):

* fp64 solves take the same iterations and reach the same objective, plan
  and duals (both reduce in fixed orders; only the association of a few
  O(m+n) sums differs);
* fixed-iteration runs, graphs vs eager launches: bitwise identical;
* the pending duals (phi = (a - 2r + coef)/n formed by the next launch) are
  materialized at the end of a run and by a mid-run plan() read;
* max_iters status and the final report.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class _env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _run(drot, m, n, dt, tail, iters=None, seed=4, **kw):
    with _env(DROTB_TAIL=tail, DROTB_PERSIST="0"):
        s = drot.Session(m, n, dt, drot.DrotConfig(**kw))
    s.gen_gaussian(5.0, seed, "dyadic")
    s.init()
    if iters is None:
        s.run()
    else:
        s.enqueue(iters)
        s.synchronize()
    st = s.status()
    plan, mu, nu = s.plan()
    s.close()
    return st, plan, mu, nu


@pytest.mark.parametrize("shape", [(500, 400), (37, 1000), (1100, 90)])
def test_fp64_solve_matches_coop_tail(drot, shape):
    m, n = shape
    (s1, i1, r1), p1, mu1, nu1 = _run(drot, m, n, np.float64, "fused", max_iters=100000)
    (s2, i2, r2), p2, mu2, nu2 = _run(drot, m, n, np.float64, "coop", max_iters=100000)
    assert s1 == s2 == drot.SolveStatus.converged
    assert abs(i1 - i2) <= 2
    assert abs(r1.objective - r2.objective) <= 1e-9 * abs(r2.objective)
    if i1 == i2:
        scale = float(np.abs(p2).max())
        assert float(np.abs(p1 - p2).max()) <= 1e-10 * scale
        assert float(np.abs(mu1 - mu2).max()) <= 1e-8 * float(np.abs(mu2).max())


def test_fp32_solve_close_to_coop_tail(drot):
    (s1, i1, r1), *_ = _run(drot, 500, 400, np.float32, "fused", max_iters=100000)
    (s2, i2, r2), *_ = _run(drot, 500, 400, np.float32, "coop", max_iters=100000)
    assert s1 == s2 == drot.SolveStatus.converged
    assert abs(i1 - i2) <= max(5, i2 // 100)
    assert abs(r1.objective - r2.objective) <= 1e-3 * abs(r2.objective)
    for v in (r1.r_primal, r1.r_dual, r1.gap):
        assert v <= 1e-4


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_graphs_equal_eager(drot, dt):
    a = _run(drot, 700, 500, dt, "fused", iters=40, tol_primal=-1.0, max_iters=10 ** 9)
    b = _run(drot, 700, 500, dt, "fused", iters=40, tol_primal=-1.0, max_iters=10 ** 9,
             use_graphs=False)
    assert a[0][1] == b[0][1] == 40
    for x, y in zip(a[1:], b[1:]):
        np.testing.assert_array_equal(x, y)


def test_fixed_iterations_close_to_coop(drot):
    a = _run(drot, 640, 480, np.float64, "fused", iters=60, tol_primal=-1.0, max_iters=10 ** 9)
    b = _run(drot, 640, 480, np.float64, "coop", iters=60, tol_primal=-1.0, max_iters=10 ** 9)
    for x, y in zip(a[1:], b[1:]):
        assert float(np.abs(x - y).max()) <= 1e-12 * max(1.0, float(np.abs(y).max()))


def test_mid_run_plan_then_continue(drot):
    """plan() between two batches materializes the pending duals; the run
    then continues from the same state as an uninterrupted one."""
    kw = dict(tol_primal=-1.0, max_iters=10 ** 9)
    with _env(DROTB_TAIL="fused", DROTB_PERSIST="0"):
        s = drot.Session(300, 200, np.float64, drot.DrotConfig(**kw))
    s.gen_gaussian(5.0, 9, "dyadic")
    s.init()
    s.enqueue(20)
    s.synchronize()
    s.plan()
    s.enqueue(20)
    s.synchronize()
    got = s.plan()
    s.close()
    want = _run(drot, 300, 200, np.float64, "fused", iters=40, seed=9, **kw)[1:]
    for x, y in zip(got, want):
        np.testing.assert_array_equal(x, y)


def test_max_iters_status(drot):
    (st, it, rep), *_ = _run(drot, 300, 300, np.float64, "fused", max_iters=777)
    (st2, it2, rep2), *_ = _run(drot, 300, 300, np.float64, "coop", max_iters=777)
    assert st == st2 == drot.SolveStatus.max_iters and it == it2 == 777
    assert abs(rep.objective - rep2.objective) <= 1e-9 * abs(rep2.objective)
