"""Config C4 at CPU-feasible size: sweep of rho0 and tolerance with the
convergence and sparsity-support check against the reference solve<double>
(SURVEY §8(c), §8(d) C4).  The full 30000^2 instance is covered by the
fixed-K trajectory tests; here each (rho0, tol) pair is solved to
termination by both solvers on a Gaussian 200 x 200 instance.

* fast order: same status, iteration count within max(5, 0.5 %), objective
  rel <= 1e-5, support symmetric difference <= 0.1 % of |supp| (+1 entry);
* the device-side support count (drotb_session_support) equals the count
  on the downloaded plan.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

M = N = 200
TAU = 1e-6  # supp = {x > TAU * max x}


@pytest.fixture(scope="module")
def inst(ref):
    C, _, _ = ref.gen_gaussian(M, N, 5.0, 0)
    return C, np.full(M, 1.0 / M), np.full(N, 1.0 / N)


def _supp(x):
    return x > TAU * x.max()


@pytest.mark.parametrize("rho0", [0.5, 2.0, 4.0])
@pytest.mark.parametrize("tol", [1e-3, 1e-4, 1e-5])
def test_rho_tol_sweep_support(drot, ref, inst, rho0, tol):
    from pyoracle import default_config
    C, p, q = inst
    kw = dict(rho0=rho0, tol_primal=tol, tol_dual=tol, tol_gap=tol, max_iters=300000,
              record_trace=0)
    want = ref.solve(C, p, q, M, N, default_config(**kw))
    cfg = drot.DrotConfig(order=drot.Order.fast, rho0=rho0, tol_primal=tol, tol_dual=tol,
                          tol_gap=tol, max_iters=300000, record_trace=False)
    got = drot.solve(drot.TransportProblem(C.reshape((M, N), order="F"), p, q), cfg)
    assert got.status.name == want.status
    assert abs(got.trace.iterations - want.iterations) <= max(5, int(0.005 * want.iterations))
    wo = want.report["objective"]
    assert abs(got.report.objective - wo) <= 1e-5 * abs(wo)
    sw = _supp(want.plan.reshape((M, N), order="F"))
    sg = _supp(got.plan.x)
    diff = int(np.logical_xor(sw, sg).sum())
    assert diff <= 0.001 * sw.sum() + 1, (diff, int(sw.sum()))


def test_device_support_count(drot, ref, inst):
    C, p, q = inst
    s = drot.Session(M, N, np.float64, drot.DrotConfig(max_iters=3001))  # ends on a fold pass
    s.set_problem(C.reshape((M, N), order="F"), p, q)
    s.init()
    s.run()
    plan, _, _ = s.plan()
    for rel, ab in ((TAU, 0.0), (0.0, 1e-8), (0.0, 0.0)):
        nnz, xmax = s.support(rel, ab)
        assert xmax == plan.max()
        assert nnz == int((plan > max(ab, rel * plan.max())).sum())
    s.close()
