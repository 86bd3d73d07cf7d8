"""The Python mirror of the API around the solve path (problem.hpp:96-154,
solver.hpp:127-139, 204-230, tiles.cpp:20-47): validate_problem /
check_problem(simplex_tol), materialize_plan / materialize_y on the device,
ErgodicMean, TilePlan.tiles."""
import numpy as np
import pytest

import paper_2110_11738_b200 as drot

gpu = pytest.mark.gpu


def _two():
    return drot.TransportProblem(np.array([[0.0, 1.0], [1.0, 0.0]], order="F"),
                                 np.array([0.5, 0.5]), np.array([0.5, 0.5]))


def test_tile_list_is_tile_column_major():
    plan = drot.plan_tiles(130, 600, 64, 4)
    tiles = plan.tiles
    assert len(tiles) == plan.grid_rows * plan.grid_cols == 3 * 3
    seen = np.zeros((130, 600), np.int32)
    for k, t in enumerate(tiles):
        assert (t.grid_c, t.grid_r) == divmod(k, plan.grid_rows)
        seen[t.r0:t.r1, t.c0:t.c1] += 1
    assert (seen == 1).all()


def test_ergodic_mean():
    e = drot.ErgodicMean()
    for v in (1.0, 2.0, 6.0):
        e.update(v)
    assert e.count() == 3 and abs(e.mean() - 3.0) < 1e-15


@gpu
def test_validate_problem_paths():
    drot.validate_problem(_two())
    bad = _two()
    bad.p = np.array([0.6, 0.6])
    with pytest.raises(drot.Error) as ei:
        drot.validate_problem(bad)
    assert ei.value.code == drot.Errc.marginal_not_simplex and "1.2" in str(ei.value)
    fixed = drot.validate_problem(bad, drot.ValidateOptions(renormalize=True))
    assert fixed.p.tolist() == [0.5, 0.5]
    assert bad.p.tolist() == [0.6, 0.6]  # the input is not modified
    off = _two()
    off.q = np.array([0.5, 0.5005])
    with pytest.raises(drot.Error):
        drot.check_problem(off)
    drot.check_problem(off, 1e-3)
    # fp32 thirds: renormalize keeps them off the 1e-12 simplex (as the
    # reference does); a 1e-6 tolerance accepts them
    pf = drot.TransportProblem(np.full((3, 3), 0.5, np.float32, order="F"),
                               np.full(3, 1 / 3, np.float32), np.full(3, 1 / 3, np.float32))
    with pytest.raises(drot.Error):
        drot.validate_problem(pf, drot.ValidateOptions(renormalize=True))
    drot.validate_problem(pf, drot.ValidateOptions(renormalize=True, simplex_tol=1e-6))


@gpu
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_materialize_plan_and_y(dt):
    m, n = 45, 38
    C = drot.random_matrix(m, n, 7).astype(dt)
    pr = drot.TransportProblem(np.asfortranarray(C), drot.dyadic_marginal(m, dt),
                               drot.dyadic_marginal(n, dt))
    cfg = drot.DrotConfig(order=drot.Order.reference)
    rho = dt(cfg.resolved_rho(m, n))
    st = drot.init_state(pr, cfg)
    for _ in range(7):
        drot.drot_step(st, pr, cfg)
    assert st.xy.cost_folded
    plan = drot.materialize_plan(st, pr.cost, rho).x
    v = st.xy.values + rho * pr.cost
    want = np.where(v > 0, v, dt(0))
    assert plan.dtype == dt and np.array_equal(plan, want)
    y = drot.materialize_y(st, pr.cost, rho)
    assert np.array_equal(y, want + (st.row_shift[:, None] + st.col_shift[None, :]))
    drot.drot_step(st, pr, cfg)
    assert not st.xy.cost_folded
    assert np.array_equal(drot.materialize_plan(st, pr.cost, rho).x, st.xy.values)
