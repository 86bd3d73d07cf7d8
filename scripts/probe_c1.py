"""Dev aid: C1 drot.solve() wall time (first and repeated calls) and the
fixed per-call overhead (max_iters 1 / 1000 calls of the same shape)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_11738_b200 as drot  # noqa: E402

m = n = 1000
C = drot.counter_uniform(1, m * n)
prob = drot.TransportProblem(C.reshape((m, n), order="F"), np.full(m, 1.0 / m), np.full(n, 1.0 / n))
for k in range(3):
    t0 = time.perf_counter()
    res = drot.solve(prob, drot.DrotConfig())
    print(f"call {k}: {time.perf_counter() - t0:.3f} s, {res.trace.iterations} iterations", flush=True)
for it in (1, 1000, 10000):
    ts = []
    for k in range(3):
        t0 = time.perf_counter()
        res = drot.solve(prob, drot.DrotConfig(max_iters=it))
        ts.append(time.perf_counter() - t0)
    print(f"max_iters {it}: {min(ts) * 1e3:.2f} ms ({res.trace.iterations} iterations)", flush=True)
# the same iteration count without the gate (tol -1): the gate / confirm cost
for label, kw in (("gated", {}), ("no gate", {"tol_primal": -1.0})):
    ts = []
    for k in range(2):
        t0 = time.perf_counter()
        res = drot.solve(prob, drot.DrotConfig(max_iters=36041, **kw))
        ts.append(time.perf_counter() - t0)
    print(f"{label}: {min(ts):.3f} s ({res.trace.iterations} iterations)", flush=True)
