"""K7: on-device problem generation must equal the reference generators bit
for bit -- gen_gaussian_problem(_as<T>) (probgen.hpp:131-180) and the
random_matrix fixture (oracles.hpp:128-135) -- including a row shard, which
generates only its rows but normalizes by the global max."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _oracle():
    import os
    from pyoracle import LIB_PATHS, Oracle
    return Oracle("ref" if os.path.exists(LIB_PATHS["ref"]) else "orc")


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("shape,seed,sigma", [((300, 200), 0, 5.0), ((97, 1001), 7, 2.5),
                                              ((1000, 1000), 0, 5.0)])
def test_gaussian_cost_bitwise(drot, dt, shape, seed, sigma):
    m, n = shape
    C, p, q = _oracle().gen_gaussian(m, n, sigma, seed)
    want = C.reshape((m, n), order="F").astype(dt)
    s = drot.Session(m, n, dt, drot.DrotConfig())
    s.gen_gaussian(sigma, seed, "uniform" if dt == np.float64 else "dyadic")
    got = s.cost()
    s.close()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_uniform_cost_bitwise(drot, dt):
    m, n = 257, 190
    want = _oracle().random_unit(1, m * n).reshape((m, n), order="F").astype(dt)
    s = drot.Session(m, n, dt, drot.DrotConfig())
    s.gen_uniform(1, 0.0, 1.0, "random_simplex" if dt == np.float64 else "dyadic")
    got = s.cost()
    s.close()
    assert np.array_equal(got, want)


def test_uniform_cost_range_bitwise(drot):
    m, n = 128, 64
    want = _oracle().random_unit(42, m * n, -0.5, 1.0).reshape((m, n), order="F")
    s = drot.Session(m, n, np.float64, drot.DrotConfig())
    # lo < 0 makes C negative: generation succeeds, validation rejects it
    with pytest.raises(drot.Error) as ei:
        s.gen_uniform(42, -0.5, 1.0, "uniform")
    assert ei.value.code == drot.Errc.negative_cost
    assert np.array_equal(s.cost(), want)
    s.close()


def test_gaussian_shard_rows(drot):
    """A shard generates rows [r0, r1) of the global instance.  With a
    1-rank communicator the shard's p does not sum to one, so validation
    rejects the problem after generation; the rows must still match."""
    m, n = 640, 300
    C, _, _ = _oracle().gen_gaussian(m, n, 5.0, 3)
    full = C.reshape((m, n), order="F").astype(np.float32)
    r0, r1 = 128, 448
    sh = drot.Session.sharded(m, n, np.float32, drot.DrotConfig(), 0, 1,
                              drot.nccl_unique_id(), r0, r1)
    with pytest.raises(drot.Error) as ei:
        sh.gen_gaussian(5.0, 3, "dyadic")
    assert ei.value.code == drot.Errc.marginal_not_simplex
    assert np.array_equal(sh.cost(), full[r0:r1])
    sh.close()


def test_random_simplex_marginals_accepted(drot):
    """C3-style instance: random cost, random_simplex marginals (fp64 passes
    the 1e-12 simplex check)."""
    m, n = 400, 50
    s = drot.Session(m, n, np.float64, drot.DrotConfig(max_iters=50))
    s.gen_uniform(3, 0.0, 1.0, "random_simplex")
    s.init()
    s.run()
    st, it, _ = s.status()
    s.close()
    assert it == 50
