"""Sinkhorn baseline on the B200 (csrc/sinkhorn.cu) -- the paper's comparison
method -- against the reference's drot::sinkhorn_solve<T>
(reference.hpp:165-288) run live from oracle/_ref, plus ports of the
reference's own Sinkhorn tests (test_reference.cpp:194-260).

Parity is to tolerance: the GPU sums K v / K^T u in tile order and uses the
device expf/exp (<= 2 ulp from libm), so iterates agree to rounding and the
iteration count to one check interval."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _prob(drot, C, p, q, dt=np.float64):
    return drot.TransportProblem(np.asfortranarray(np.asarray(C, dt)), np.asarray(p, dt),
                                 np.asarray(q, dt))


def test_uniform_kernel_converges_immediately(drot):  # test_reference.cpp:194-203
    res = drot.sinkhorn_solve(_prob(drot, np.zeros((2, 2)), [0.5, 0.5], [0.5, 0.5]), 0.5, 1e-10,
                              100, check_every=1)
    assert res.status == drot.SolveStatus.converged
    assert res.trace.iterations <= 2
    np.testing.assert_allclose(res.plan.x, 0.25, rtol=1e-12)


def test_rejects_zero_marginals(drot):  # test_reference.cpp:205-211
    with pytest.raises(drot.Error) as e:
        drot.sinkhorn_solve(_prob(drot, np.zeros((2, 2)), [1.0, 0.0], [0.5, 0.5]), 0.1, 1e-6, 10)
    assert e.value.code == drot.Errc.zero_marginal
    with pytest.raises(drot.Error) as e:
        drot.sinkhorn_solve(_prob(drot, np.zeros((2, 2)), [0.5, 0.5], [0.5, 0.5]), 0.0, 1e-6, 10)
    assert e.value.code == drot.Errc.bad_config


def test_fp32_underflows_at_tiny_eta(drot, ref):  # test_reference.cpp:213-221
    C, p, q = ref.gen_gaussian(64, 64, 5.0, 31337)
    prob = _prob(drot, C.reshape((64, 64), order="F"), p, q, np.float32)
    res = drot.sinkhorn_solve(prob, 1e-4, 1e-4, 1000)
    assert res.status == drot.SolveStatus.numerical_failure
    want = ref.sinkhorn(C.astype(np.float32), p.astype(np.float32), q.astype(np.float32), 64, 64,
                        1e-4, 1e-4, 1000)
    assert want.status == "numerical_failure"
    assert res.trace.iterations == want.iterations


def test_accuracy_floor(drot, ref):  # test_reference.cpp:223-246
    C = np.array([[0.0, 1.0], [1.0, 0.0]])
    res = drot.sinkhorn_solve(_prob(drot, C, [0.7, 0.3], [0.4, 0.6]), 0.1, 1e-4, 20000)
    assert res.status == drot.SolveStatus.converged
    assert abs(res.report.objective - 0.3) < 0.07
    for seed in (21, 22, 23):
        Cg, p, q = ref.gen_gaussian(16, 16, 5.0, seed)
        res = drot.sinkhorn_solve(_prob(drot, Cg.reshape((16, 16), order="F"), p, q), 0.1, 1e-4,
                                  1000)
        assert res.status != drot.SolveStatus.numerical_failure
        opt = ref.lp_exact(Cg, p, q, 16, 16)[0]
        err = abs(res.report.objective - opt)
        assert err > 1e-4 * abs(opt)
        assert err < 0.1 * np.log(16.0) * 2


def test_plans_positive_and_entropy_biased(drot, ref):  # test_reference.cpp:248-260
    for trial in range(5):
        C = ref.random_unit(1234 + trial, 20)
        p = ref.random_unit(99 + trial, 4) + 0.05
        q = ref.random_unit(199 + trial, 5) + 0.05
        p, q = p / p.sum(), q / q.sum()
        res = drot.sinkhorn_solve(_prob(drot, C.reshape((4, 5), order="F"), p, q), 0.05, 1e-9,
                                  50000)
        assert res.status == drot.SolveStatus.converged
        assert (res.plan.x > 0).all()
        lp = ref.lp_exact(C, p, q, 4, 5)[0]
        assert res.report.objective >= lp - 1e-9
        assert res.report.r_primal <= 1e-8


@pytest.mark.parametrize("dt,shape,eta,tol", [(np.float64, (200, 150), 0.05, 1e-6),
                                              (np.float32, (300, 200), 0.1, 1e-4),
                                              (np.float64, (1000, 1000), 0.02, 1e-5)])
def test_matches_reference_sinkhorn(drot, ref, dt, shape, eta, tol):
    m, n = shape
    C, p, q = ref.gen_gaussian(m, n, 5.0, 3)
    C, p, q = C.astype(dt), p.astype(dt), q.astype(dt)
    want = ref.sinkhorn(C, p, q, m, n, eta, tol, 20000)
    got = drot.sinkhorn_solve(_prob(drot, C.reshape((m, n), order="F"), p, q, dt), eta, tol,
                              20000, exact_report=True)
    assert got.status.name == want.status
    assert abs(got.trace.iterations - want.iterations) <= 10  # one check interval
    # every row: r_dual = kResidualNotApplicable, the other fields left at the
    # TraceRow defaults (0) as the reference pushes them (reference.hpp:279-283)
    for a in got.trace.rows:
        assert a.r_dual == -1.0
        assert (a.gap, a.objective, a.ergodic_objective, a.fixed_point_residual) == (0, 0, 0, 0)
    rel = 1e-7 if dt == np.float64 else 1e-3
    assert abs(got.report.objective - want.report["objective"]) <= rel * abs(
        want.report["objective"])
    if got.trace.iterations == want.iterations:
        np.testing.assert_allclose(got.plan.x.ravel(order="F"), want.plan,
                                   rtol=1e-6 if dt == np.float64 else 1e-2, atol=1e-30)
        for a, b in zip(got.trace.rows, want.trace):
            assert a.iter == b["iter"]
            # fp32: the marginal error bottoms out at the rounding floor of
            # u * (K v) - p (~1e-9 here), so an absolute term is needed
            atol = 1e-14 if dt == np.float64 else 1e-8
            assert abs(a.r_primal - b["r_primal"]) <= (1e-6 if dt == np.float64 else 1e-2) * \
                b["r_primal"] + atol
