"""World-size-2 CPU tests (gloo) of the row-sharded multi-GPU path.

* the product's row partition (drotb_shard_rows) covers every row once, in
  64-row-aligned contiguous blocks, for 1/2/4/8 ranks;
* the sharded exchange schedule the CUDA path implements:
  per iteration an allreduce of [v partial | sum r, |r|^2, pass scalars],
  replicated finish (s = v - q, beta, coef), local phi / replicated varphi
  update, and an allreduce of the row-side dual-value / trace sums -- run
  here by 2 gloo ranks on CPU with a numpy model of the per-shard work --
  reproduces the single-process reference iteration (C oracle) to rounding,
  including the gate decision sequence.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_rows_partition():
    import paper_2110_11738_b200 as drot
    for m in (1, 63, 64, 65, 1000, 10000, 100000, 100001):
        for world in (1, 2, 4, 8):
            ranges = [drot.shard_rows(m, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == m
            for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
                assert a1 == b0
            # 512-row sweep blocks (bit-identical to one GPU) when every rank
            # can own one, else 64-row blocks
            unit = 512 if m >= 512 * world else 64
            for r0, r1 in ranges:
                assert r0 % unit == 0 and r0 <= r1
            sizes = [r1 - r0 for r0, r1 in ranges]
            assert max(sizes) - min(sizes) <= unit


def _model_iterations(rank, world, port, m, n, iters, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2110_11738_b200 as drot
    rng = np.random.default_rng(7)
    C = rng.random((m, n))
    p = np.full(m, 1.0 / m)
    q = np.full(n, 1.0 / n)
    rho = 2.0 / (m + n)
    r0, r1 = drot.shard_rows(m, world, rank)
    Cl, pl = C[r0:r1], p[r0:r1]

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    # init_state (solver.hpp:143-186), sharded: column sums are collective
    X = np.outer(pl, q)
    a = X.sum(axis=1) - pl
    b = allreduce(X.sum(axis=0)) - q
    alpha = allreduce(np.array([a.sum()]))[0] / (m + n)
    phi, varphi = np.zeros(r1 - r0), np.zeros(n)
    fold = False
    gates = []
    for k in range(iters):
        # local sweep on the shard (skip-C alternation, fused.hpp:140-155)
        if not fold:
            t = ((X + phi[:, None]) + varphi[None, :]) - rho * Cl
        else:
            t = (X + phi[:, None]) + varphi[None, :]
        xp = np.maximum(t, 0)
        cost = (Cl * xp).sum() if not fold else 0.0
        X = xp - rho * Cl if not fold else xp
        u = xp.sum(axis=1)
        r = u - pl
        # exchange 1: [v partial | sum r, |r|^2, cost]
        pack = allreduce(np.concatenate([xp.sum(axis=0), [r.sum(), (r * r).sum(), cost]]))
        v, sum_r, nr2, cost_g = pack[:n], pack[n], pack[n + 1], pack[n + 2]
        s = v - q
        beta = sum_r / (m + n)
        coef = 2 * beta - alpha
        phi = (a - 2 * r + coef) / n
        varphi = (b - 2 * s + coef) / m
        a, b, alpha = a - r, b - s, alpha - beta
        # exchange 2: row-side dual value; column side is replicated
        dual_i = allreduce(np.array([(pl * phi).sum() / rho]))[0]
        dual = dual_i + (q * varphi).sum() / rho
        r_primal = np.sqrt(nr2 + (s * s).sum())
        gates.append((r_primal, dual, cost_g))
        fold = not fold
    out[rank] = (gates, allreduce(np.array([(X if fold else X).sum()]))[0])
    dist.destroy_process_group()


def _worker(rank, world, port, m, n, iters, q):
    out = {}
    _model_iterations(rank, world, port, m, n, iters, out)
    q.put((rank, out[rank]))


def _run(world, m, n, iters):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, iters, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    return res


def test_sharded_schedule_world2_matches_single_process():
    m, n, iters = 150, 90, 60
    two = _run(2, m, n, iters)
    one = _run(1, m, n, iters)
    g2, g1 = two[0][0], one[0][0]
    assert two[0][0] == two[1][0]  # replicated scalars agree on every rank
    for (rp2, d2, c2), (rp1, d1, c1) in zip(g2, g1):
        assert rp2 == pytest.approx(rp1, rel=1e-9, abs=1e-15)
        assert d2 == pytest.approx(d1, rel=1e-9, abs=1e-15)
        assert c2 == pytest.approx(c1, rel=1e-9, abs=1e-15)


def test_world1_model_matches_oracle_iterates():
    """The numpy model at world 1 is the reference iteration: its gate
    quantities track the C oracle's trace (rounding-level agreement)."""
    import sys
    from pyoracle import Oracle, default_config
    m, n, iters = 150, 90, 60
    one = _run(1, m, n, iters)[0][0]
    rng = np.random.default_rng(7)
    C = rng.random((m, n))
    orc = Oracle("orc")
    out = orc.solve(C.ravel(order="F"), np.full(m, 1.0 / m), np.full(n, 1.0 / n), m, n,
                    default_config(max_iters=iters, tol_primal=-1.0))
    for row, (rp, dual, cost) in zip(out.trace, one):
        assert row["r_primal"] == pytest.approx(rp, rel=1e-8, abs=1e-14)
