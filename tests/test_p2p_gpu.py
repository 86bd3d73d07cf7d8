"""Row shards with the per-iteration exchange fused into the cooperative tail
over peer memory (tail.cu shard_tail_kernel; no NCCL).

* world = 1: the full protocol runs against the rank's own buffer and must
  reproduce the single-GPU fast-order solve to the fast-order tolerances;
* world = 2 in ONE process on ONE GPU: two shard sessions on two streams,
  driven from two host threads, exchange through each other's buffers
  (plain device pointers instead of IPC handles) -- the exchange, the flag
  protocol, the parity buffers, the setup collectives and the paused
  collective confirm all run for real.  Both ranks must agree bit for bit
  on every replicated quantity (status, iterations, report, nu), and the
  joined solution must match the one-rank solve.
Two tails must be co-resident for the in-process world = 2 run: the tail
grid is reduced to one CTA per SM and launched as an ordinary grid there
(DROTB_TAIL_CTAS, DROTB_TAIL_NONCOOP -- the driver does not overlap two
cooperative grids on one device; one process per GPU never needs this).
"""
import os
import threading

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


def _single(drot, m, n, dt, cfg, seed):
    with _env(DROTB_TAIL="coop", DROTB_PERSIST="0"):
        s = drot.Session(m, n, dt, cfg)
    s.gen_gaussian(5.0, seed, "dyadic")
    s.init()
    s.run()
    st = s.status()
    plan, mu, nu = s.plan()
    s.close()
    return st, plan, mu, nu


def _parallel(fns):
    errs = []

    def wrap(f):
        try:
            f()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "exchange deadlock"
    if errs:
        raise errs[0]


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_world1_matches_single_gpu(drot, dt):
    m, n = 500, 400
    cfg = drot.DrotConfig(max_iters=100000)
    (st1, it1, r1), plan1, mu1, nu1 = _single(drot, m, n, dt, cfg, 3)
    with _env(DROTB_TAIL_CTAS="2"):
        s = drot.Session.sharded_p2p(m, n, dt, cfg, 0, 1, 0, m)
    s.attach_peers(pointers=[s.exchange_pointer()])
    s.gen_gaussian(5.0, 3, "dyadic")
    s.init()
    s.run()
    st2, it2, r2 = s.status()
    plan2, mu2, nu2 = s.plan()
    s.close()
    assert st1 == st2 == drot.SolveStatus.converged
    assert abs(it1 - it2) <= max(5, it1 // 200)
    rel = 1e-5 if dt == np.float64 else 1e-3
    assert abs(r1.objective - r2.objective) <= rel * abs(r1.objective)
    for v in (r2.r_primal, r2.r_dual, r2.gap):
        assert v <= 1e-4


@pytest.fixture()
def noncoop_tail():
    with _env(DROTB_TAIL_NONCOOP="1"):
        yield


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_world2_in_process(drot, dt, noncoop_tail):
    m, n = 700, 500
    # eager launches: graph instantiation must not wait on the peer session's
    # spinning exchange kernel on the same device (in-process test only)
    cfg = drot.DrotConfig(max_iters=100000, use_graphs=False)
    (st1, it1, r1), plan1, mu1, nu1 = _single(drot, m, n, dt, cfg, 5)
    import torch
    ranges = [drot.shard_rows(m, 2, r) for r in range(2)]
    with _env(DROTB_TAIL_CTAS="1"):
        ss = [drot.Session.sharded_p2p(m, n, dt, cfg, r, 2, *ranges[r]) for r in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    for s, stm in zip(ss, streams):
        s.set_stream(stm.cuda_stream)
    ptrs = [s.exchange_pointer() for s in ss]
    for s in ss:
        s.attach_peers(pointers=ptrs)
    _parallel([lambda s=s: s.gen_gaussian(5.0, 5, "dyadic") for s in ss])
    _parallel([s.init for s in ss])
    _parallel([s.run for s in ss])
    out = [None, None]

    def fin(r):
        out[r] = (ss[r].status(), ss[r].plan())

    _parallel([lambda r=r: fin(r) for r in range(2)])
    for s in ss:
        s.close()
    (sa, ia, ra), (pa, mua, nua) = out[0]
    (sb, ib, rb), (pb, mub, nub) = out[1]
    # replicated state: bit-identical on both ranks
    assert sa == sb and ia == ib
    assert (ra.objective, ra.r_primal, ra.r_dual, ra.gap) == (rb.objective, rb.r_primal,
                                                              rb.r_dual, rb.gap)
    np.testing.assert_array_equal(nua, nub)
    # the joined solution against the one-GPU solve
    assert sa == st1 == drot.SolveStatus.converged
    assert abs(ia - it1) <= max(5, it1 // 200)
    rel = 1e-5 if dt == np.float64 else 1e-3
    assert abs(ra.objective - r1.objective) <= rel * abs(r1.objective)
    plan = np.concatenate([pa, pb], axis=0)
    scale = float(np.abs(plan1).max())
    tol = (1e-6 if dt == np.float64 else 1e-3) if ia == it1 else 2e-2
    assert float(np.abs(plan - plan1).max()) <= tol * scale
