"""Dev aid: where does the per-iteration time go beyond the fused sweep?

Times K iterations at 10k x 10k fp32 three ways on one stream with CUDA
events (torch): untimed batch graphs (what run() uses), the timed graph of
run_timed (event nodes around every sweep), and eager launches; and with
record_trace on/off.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_11738_b200 as drot  # noqa: E402


def timed_enqueue(s, stream, k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    s.enqueue(k)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / k


def run(m, n, dt, label, K=200, **kw):
    cfg = drot.DrotConfig(tol_primal=-1.0, max_iters=10 ** 12, **kw)
    s = drot.Session(m, n, dt, cfg)
    stream = torch.cuda.Stream()
    s.set_stream(stream.cuda_stream)
    s.gen_gaussian(5.0, 0, "dyadic")
    s.init()
    timed_enqueue(s, stream, 64)
    us = timed_enqueue(s, stream, K)
    r = s.run_timed(K)
    print(f"{label:40s} {m}x{n} {np.dtype(dt).name}: enqueue {us:7.1f} us/iter | run_timed "
          f"{r['total_ms'] * 1e3 / K:7.1f} us/iter, sweep {r['pass_ms'] * 1e3 / K:6.1f} us",
          flush=True)
    s.close()


if __name__ == "__main__":
    for dt in (np.float32,):
        run(10000, 10000, dt, "graphs, trace")
        run(10000, 10000, dt, "graphs, no trace", record_trace=False)
        run(10000, 10000, dt, "eager, trace", use_graphs=False)
        run(10000, 10000, dt, "graphs, no skip_cost", skip_cost=False)
    run(1000, 1000, np.float64, "graphs, trace", K=2000)
    run(1000, 1000, np.float64, "eager, trace", K=2000, use_graphs=False)
