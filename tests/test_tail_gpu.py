"""The cooperative per-iteration tail (csrc/tail.cu, the default fast-order
path on one GPU) against the per-launch tail kernels (DROTB_TAIL=legacy) and
against itself:

* captured CUDA graphs and eager launches run the same kernels: bitwise
  identical iterates, duals and reports;
* solves to tolerance agree with the legacy tail and the reference to the
  fast-order tolerances; the confirm report inside the tail decides
  convergence exactly like the graph IF-node path (same status);
* a non-finite sweep stops the loop with numerical_failure.
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


def _run(drot, m, n, dt, iters=None, legacy=False, ctail="16", gen=4, **kw):
    with _env(DROTB_TAIL="legacy" if legacy else "coop", DROTB_CTAIL=ctail):
        s = drot.Session(m, n, dt, drot.DrotConfig(**kw))
    s.gen_gaussian(5.0, gen, "dyadic")
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


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_graphs_equal_eager(drot, dt):
    a = _run(drot, 700, 500, dt, iters=40, tol_primal=-1.0, max_iters=10 ** 9)
    b = _run(drot, 700, 500, dt, iters=40, tol_primal=-1.0, max_iters=10 ** 9, use_graphs=False)
    assert a[0][1] == b[0][1] == 40
    for x, y in zip(a[1:], b[1:]):
        np.testing.assert_array_equal(x, y)
    assert a[0][2].objective == b[0][2].objective


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_converges_like_legacy_tail(drot, dt):
    (s1, i1, r1), *_ = _run(drot, 500, 400, dt, max_iters=80000)
    (s2, i2, r2), *_ = _run(drot, 500, 400, dt, max_iters=80000, legacy=True)
    assert s1 == s2 == drot.SolveStatus.converged
    assert abs(i1 - i2) <= max(5, int(0.005 * i2))
    rel = 1e-5 if dt == np.float64 else 1e-3
    assert abs(r1.objective - r2.objective) <= rel * abs(r2.objective)
    for v in (r1.r_primal, r1.r_dual, r1.gap):
        assert v <= 1e-4


def test_max_iters_status_and_report(drot):
    (st, it, rep), *_ = _run(drot, 300, 300, np.float64, max_iters=777)
    assert st == drot.SolveStatus.max_iters and it == 777
    (st2, it2, rep2), *_ = _run(drot, 300, 300, np.float64, max_iters=777, legacy=True)
    assert it2 == 777
    assert abs(rep.objective - rep2.objective) <= 1e-9 * abs(rep2.objective)


def test_numerical_failure(drot):
    m, n = 64, 48
    C = np.full((m, n), 1e300)
    prob = drot.TransportProblem(np.asfortranarray(C), np.full(m, 1.0 / m), np.full(n, 1.0 / n))
    with _env(DROTB_TAIL="coop"):
        drot.release_device_cache()
        r = drot.solve(prob, drot.DrotConfig(rho_override=1e10))
        drot.release_device_cache()
    assert r.status == drot.SolveStatus.numerical_failure


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_fused_gate_matches_exact_gate(drot, dt):
    """The fused gate (closed-form dual value as the pre-filter, exact values
    patched into the trace one iteration later) against the two-barrier tail
    that gates on the summed dual value: same status, iterations within
    max(2, 0.1 %), trace rows equal to rounding."""
    m, n = 300, 260
    C = np.asfortranarray(drot.random_matrix(m, n, 9).astype(dt))
    p = drot.dyadic_marginal(m, dt)
    q = drot.dyadic_marginal(n, dt)
    res = []
    for gate in ("fused", "exact"):
        with _env(DROTB_TAIL="coop", DROTB_TAIL_GATE=gate):
            drot.release_device_cache()
            res.append(drot.solve(drot.TransportProblem(C, p, q), drot.DrotConfig(max_iters=60000)))
            drot.release_device_cache()
    a, b = res
    assert a.status == b.status == drot.SolveStatus.converged
    assert abs(a.trace.iterations - b.trace.iterations) <= max(2, b.trace.iterations // 1000)
    rel = 1e-9 if dt == np.float64 else 1e-4
    assert abs(a.report.objective - b.report.objective) <= rel * abs(b.report.objective)
    k = min(len(a.trace.rows), len(b.trace.rows))
    for ra, rb in zip(a.trace.rows[:k], b.trace.rows[:k]):
        assert ra.iter == rb.iter
        for f in ("gap", "fixed_point_residual", "objective", "r_primal"):
            x, y = getattr(ra, f), getattr(rb, f)
            assert x == y or (np.isnan(x) and np.isnan(y)) or abs(x - y) <= 1e-6 * max(abs(y), 1e-12), (ra.iter, f, x, y)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_l2_policies_do_not_change_results(drot, dt):
    """DROTB_L2HINT only changes L2 eviction priorities (sweep.cuh): the
    iterates must be bitwise identical with and without them."""
    runs = []
    for hint in ("0", "2"):
        with _env(DROTB_L2HINT=hint):
            runs.append(_run(drot, 700, 500, dt, iters=40, tol_primal=-1.0, max_iters=10 ** 9))
    a, b = runs
    assert a[0][1] == b[0][1] == 40
    for x, y in zip(a[1:], b[1:]):
        np.testing.assert_array_equal(x, y)



@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_max_iters_report_gap(drot, dt):
    """A max_iters run's final report (state_report, solver.hpp:527-538): gap =
    |objective - dual value| with the dual value of the returned duals -- the
    graph batch running on past the stop must not reset the last iteration's
    pending exact sums (r2 regression)."""
    m, n = 500, 400
    s = drot.Session(m, n, dt, drot.DrotConfig(max_iters=301))
    s.gen_gaussian(5.0, 3, "dyadic")
    s.init()
    s.run()
    st, it, rep = s.status()
    plan, mu, nu = s.plan()
    p = drot.dyadic_marginal(m, dt).astype(np.float64)
    q = drot.dyadic_marginal(n, dt).astype(np.float64)
    s.close()
    assert st.name == "max_iters" and it == 301
    dual = float(p @ mu.astype(np.float64) + q @ nu.astype(np.float64))
    assert abs(rep.gap - abs(rep.objective - dual)) <= 1e-9 * abs(rep.objective) + 1e-12, \
        (rep.gap, rep.objective, dual)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("shape", [(700, 500), (1500, 1380), (3000, 2000), (9000, 7000),
                                   (13440, 13440), (13441, 13440)])
def test_cluster_tail_equals_grid_tail(drot, dt, shape):
    """The cluster tail (KC, tail.cu: one 16- or 8-CTA cluster, DSMEM
    reductions) and the grid tail (148 CTAs, counter barriers) sum the same
    exact integers: bitwise identical iterates, duals and reports.  Up to
    15 * 192 = 2880 elements the cluster's CTAs have 256 threads (1500 + 1380
    is the last such size), then 512.  9000 +
    7000 elements exceed an 8-CTA cluster (7 updating CTAs: 12 544 slots,
    so the grid tail runs) but fit 16 (26 880: 13 440 + 13 440 uses every
    slot, one more row falls back to the grid tail)."""
    m, n = shape
    kw = dict(iters=30 if m < 10000 else 12, tol_primal=-1.0, max_iters=10 ** 9)
    grid = _run(drot, m, n, dt, ctail="0", **kw)
    for cap in ("16", "8"):
        clu = _run(drot, m, n, dt, ctail=cap, **kw)
        assert grid[0][1] == clu[0][1] == kw["iters"]
        for x, y in zip(grid[1:], clu[1:]):
            np.testing.assert_array_equal(x, y)
        assert grid[0][2].objective == clu[0][2].objective


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_cluster_tail_solve_equals_grid_tail(drot, dt):
    """To convergence (the fused gate fires, the confirm report runs inside
    the cluster): same status, iteration count and report, bitwise."""
    a = _run(drot, 500, 400, dt, ctail="0", max_iters=80000)
    b = _run(drot, 500, 400, dt, ctail="16", max_iters=80000)
    assert a[0][0] == b[0][0] == drot.SolveStatus.converged
    assert a[0][1] == b[0][1]
    for f in ("objective", "r_primal", "r_dual", "gap"):
        assert getattr(a[0][2], f) == getattr(b[0][2], f), f
    for x, y in zip(a[1:], b[1:]):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_cluster_tail_trace_equals_grid_tail(drot, dt):
    """The trace rows (written by the tail's deferred commit and patched with
    the exact dual value / fixed-point residual one iteration later, or by
    the finalize kernel) are identical for the cluster and the grid tail."""
    m, n = 260, 300
    C = np.asfortranarray(drot.random_matrix(m, n, 5).astype(dt))
    prob = drot.TransportProblem(C, drot.dyadic_marginal(m, dt), drot.dyadic_marginal(n, dt))
    res = []
    for ct in ("0", "16"):
        with _env(DROTB_TAIL="coop", DROTB_CTAIL=ct):
            drot.release_device_cache()
            res.append(drot.solve(prob, drot.DrotConfig(max_iters=60000, trace_every=7)))
            drot.release_device_cache()
    a, b = res
    assert a.status == b.status and a.trace.iterations == b.trace.iterations
    assert len(a.trace.rows) == len(b.trace.rows) > 10
    for ra, rb in zip(a.trace.rows, b.trace.rows):
        for f in ("iter", "r_primal", "r_dual", "gap", "objective", "ergodic_objective",
                  "fixed_point_residual"):
            x, y = getattr(ra, f), getattr(rb, f)
            assert x == y or (np.isnan(x) and np.isnan(y)), (ra.iter, f, x, y)
    np.testing.assert_array_equal(a.plan.x, b.plan.x)
