"""residual_report / objective of an arbitrary (plan, cert) pair on the GPU
(problem.hpp:155-225) against the reference's own residual_report run live
(oracle/_ref): exact order bitwise, fast order to summation noise.  Mirrors
the reference's test_problem.cpp:109-160 (report vs a double loop,
repeatable) on random plans and certificates."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _inst(ref, m, n, seed, dt):
    C = ref.random_unit(seed, m * n).reshape((m, n), order="F")
    X = ref.random_unit(seed + 1, m * n, -0.1, 1.0).reshape((m, n), order="F") / (m * n)
    mu = ref.random_unit(seed + 2, m, -0.5, 0.5)
    nu = ref.random_unit(seed + 3, n, -0.5, 0.5)
    p = np.full(m, 1.0 / m)
    q = np.full(n, 1.0 / n)
    return [np.asarray(a, dt) for a in (C, p, q, X, mu, nu)]


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("shape", [(1, 1), (37, 53), (300, 200), (2049, 17), (5, 3000)])
def test_residual_report_matches_reference(drot, ref, dt, shape):
    m, n = shape
    C, p, q, X, mu, nu = _inst(ref, m, n, 11 + m, dt)
    want = ref.residual_report(C.ravel(order="F"), p, q, X.ravel(order="F"), mu, nu, m, n)
    prob = drot.TransportProblem(C, p, q)
    plan, cert = drot.TransportPlan(X), drot.DualCertificate(mu, nu)
    got = drot.residual_report(prob, plan, cert, exact=True)
    for k in ("r_primal", "r_dual", "gap", "objective"):
        assert getattr(got, k) == want[k], (k, getattr(got, k), want[k])
    fast = drot.residual_report(prob, plan, cert, exact=False)
    for k in ("r_primal", "r_dual", "gap", "objective"):
        assert abs(getattr(fast, k) - want[k]) <= 1e-11 * max(1.0, abs(want[k])), k
    assert drot.objective(prob, plan) == want["objective"]


def test_residual_report_shape_errors(drot, ref):
    C, p, q, X, mu, nu = _inst(ref, 20, 30, 5, np.float64)
    prob = drot.TransportProblem(C, p, q)
    with pytest.raises(drot.Error) as e:
        drot.residual_report(prob, drot.TransportPlan(X[:, :29]), drot.DualCertificate(mu, nu))
    assert e.value.code == drot.Errc.shape_mismatch
    with pytest.raises(drot.Error) as e:
        drot.residual_report(prob, drot.TransportPlan(X), drot.DualCertificate(mu[:19], nu))
    assert e.value.code == drot.Errc.shape_mismatch
