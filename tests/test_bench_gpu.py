"""bench.py end to end on the GPU: the N = 1 line, and the N = 2 torchrun path
(DROTB_BENCH_SHARE_GPU=1: both ranks on cuda:0, a gloo process group, the
peer-memory exchange between two processes through CUDA IPC -- time-sliced,
so its numbers mean nothing, but every leg of the multi-GPU line runs: the
weak-scaling headline, the same-instance C2 time-to-tol (bit-identical to
N = 1: same iteration count) and the C5 strong-scaling leg)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAST = ["--steps", "10", "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--no-sinkhorn",
        "--no-f64", "--ttt-max-iters", "300"]


def _line(out):
    lines = [ln for ln in out.strip().splitlines() if ln.startswith("{")]
    assert lines, out[-3000:]
    return json.loads(lines[-1])


def test_bench_n1_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *FAST, "--no-c5"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 1 and d["steps"] == 10 and d["value"] > 0
    assert d["graph_captures_in_timed_region"] == 0 and d["gpu_launches"] > 0
    assert 0.5 < d["roofline"]["frac"] <= 1.05
    ttt = d["time_to_tol_c2"]
    assert ttt["iterations"] == 300 and ttt["status"] == "max_iters"


def test_bench_n2_torchrun_shared_gpu():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, DROTB_BENCH_SHARE_GPU="1", CUDA_MODULE_LOADING="EAGER")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", *FAST],
                       capture_output=True, text=True, timeout=1500, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["exchange"] == "p2p"
    ttt = d["time_to_tol_c2"]
    assert "same instance" in ttt["config"]
    assert ttt["iterations"] == 300 and ttt["status"] == "max_iters"
    c5 = d["c5_strong"]
    assert c5.get("ms_per_iteration", 0) > 0 or "skipped" in c5, c5
