"""Row-sharded session (NCCL path) on the one GPU available:
world_size 1 runs the full sharded schedule -- local sweep, allreduce of
[v | scalars], replicated finish, update, allreduce of the row-side sums,
gate with collective pause/confirm -- and must reproduce the single-device
fast solve."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_sharded_world1_matches_single(drot, dt):
    m, n = 400, 300
    cfg = drot.DrotConfig(max_iters=200000)
    single = drot.Session(m, n, dt, cfg)
    single.gen_gaussian(5.0, 3, "dyadic")
    single.init()
    single.run()
    st1, it1, rep1 = single.status()
    plan1, mu1, nu1 = single.plan()
    single.close()

    r0, r1 = drot.shard_rows(m, 1, 0)
    assert (r0, r1) == (0, m)
    sh = drot.Session.sharded(m, n, dt, cfg, 0, 1, drot.nccl_unique_id(), r0, r1)
    sh.gen_gaussian(5.0, 3, "dyadic")
    sh.init()
    sh.run()
    st2, it2, rep2 = sh.status()
    plan2, mu2, nu2 = sh.plan()
    sh.close()
    assert st1 == st2 == drot.SolveStatus.converged
    assert abs(it1 - it2) <= max(5, int(0.005 * it1))
    rel = 1e-5 if dt == np.float64 else 1e-3
    assert abs(rep1.objective - rep2.objective) <= rel * abs(rep1.objective)
    for r in (rep2.r_primal, rep2.r_dual, rep2.gap):
        assert r <= 1e-4


def test_sharded_rejects_reference_order(drot):
    with pytest.raises(drot.Error) as e:
        drot.Session.sharded(100, 100, np.float64, drot.DrotConfig(order=drot.Order.reference),
                             0, 1, drot.nccl_unique_id(), 0, 100)
    assert e.value.code == drot.Errc.bad_config
