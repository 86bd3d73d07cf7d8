"""Row shards with the per-iteration exchange fused into the tail over peer
memory (tail.cu tail_kernel with world > 1; no NCCL).  Every sum that crosses
rows or ranks is exact (64-bit fixed-point column sums, hi / lo integer
accumulators for the scalars, added into every rank's buffers with integer
atomics), the shards are aligned to the sweep's 512-row CTA blocks and the
sweep tiles come from the global shape -- so a sharded solve is BIT-IDENTICAL
to the one-GPU solve, for any rank count:

* world = 1: the rank's own buffer; bitwise the one-GPU session;
* world = 2, 3 in ONE process on ONE GPU: shard sessions on separate streams,
  driven from host threads, exchange through each other's buffers (plain
  device pointers instead of IPC handles) -- forwarding, cross-rank counters,
  parity buffers, setup collectives and the in-tail confirm run for real.
  Iterations, status, report and the joined plan equal the one-GPU solve's
  bit for bit.
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
    with _env(DROTB_TAIL="coop"):
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
    assert it1 == it2
    assert (r1.objective, r1.r_primal, r1.r_dual, r1.gap) == \
        (r2.objective, r2.r_primal, r2.r_dual, r2.gap)
    assert np.array_equal(plan1, plan2) and np.array_equal(nu1, nu2) and np.array_equal(mu1, mu2)


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("world", [2, 3])
def test_world_n_in_process(drot, dt, world):
    """world shards of one process on one GPU (tests/p2p_world2.py)."""
    import json
    import subprocess
    import sys
    m, n = 1600, 500  # >= 512 rows per rank: shards on the sweep's CTA blocks
    npdt = np.float64 if dt == "f64" else np.float32
    cfg = drot.DrotConfig(max_iters=100000)
    (st1, it1, r1), plan1, mu1, nu1 = _single(drot, m, n, npdt, cfg, 5)
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER")
    proc = subprocess.run([sys.executable, os.path.join(here, "p2p_world2.py"), dt, str(m),
                           str(n), str(world)], capture_output=True, text=True, timeout=600,
                          env=env)
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-2000:]
    out = json.loads(proc.stdout.strip().splitlines()[-1])
    # replicated state: bit-identical on every rank
    for o in out[1:]:
        assert o["status"] == out[0]["status"] and o["iterations"] == out[0]["iterations"]
        assert o["report"] == out[0]["report"]
        assert o["nu"] == out[0]["nu"]
    ia, ra = out[0]["iterations"], out[0]["report"]
    assert out[0]["status"] == st1.name == "converged"
    # bit-identical to the one-GPU solve
    assert ia == it1
    assert ra == [r1.objective, r1.r_primal, r1.r_dual, r1.gap]
    plan = np.concatenate([np.array(o["plan"]) for o in out], axis=0)
    assert np.array_equal(plan, plan1.astype(np.float64))
    assert np.array_equal(np.array(out[0]["nu"]), nu1.astype(np.float64))


def test_ipc_two_processes(drot, tmp_path):
    """Two processes, one shard each, peers attached through CUDA IPC handles
    (tests/p2p_ipc_worker.py) -- against the one-GPU solve of the same 40
    iterations."""
    import json
    import socket
    import subprocess
    import sys
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER", MASTER_ADDR="127.0.0.1",
               MASTER_PORT=str(port))
    outs = [str(tmp_path / f"r{r}.json") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(here, "p2p_ipc_worker.py"), str(r),
                               "2", outs[r]], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    logs = []
    for pr in procs:
        try:
            logs.append(pr.communicate(timeout=400)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise AssertionError("IPC exchange did not finish")
    assert all(pr.returncode == 0 for pr in procs), "\n".join(l[-1500:] for l in logs)
    res = [json.load(open(o)) for o in outs]
    assert res[0]["iterations"] == res[1]["iterations"] == 40
    assert res[0]["report"] == res[1]["report"] and res[0]["nu"] == res[1]["nu"]
    cfg = drot.DrotConfig(tol_primal=-1.0, max_iters=40)
    (st1, it1, r1), plan1, mu1, nu1 = _single(drot, 640, 480, np.float64, cfg, 7)
    assert it1 == 40
    assert abs(res[0]["report"][0] - r1.objective) <= 1e-9 * abs(r1.objective)
    plan = np.concatenate([np.array(r["plan"]) for r in res], axis=0)
    assert float(np.abs(plan - plan1).max()) <= 1e-9 * float(np.abs(plan1).max())
