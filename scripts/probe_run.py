"""Dev aid: where the solve loop's time goes at 1000^2 fp64 (uniform cost,
reference defaults): drot.solve() vs Session.run() vs Session.enqueue() over
the same 10 000 iterations, wall clock."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_11738_b200 as drot  # noqa: E402

m = n = 1000
N = 10000
C = drot.counter_uniform(1, m * n)
prob = drot.TransportProblem(C.reshape((m, n), order="F"), np.full(m, 1.0 / m), np.full(n, 1.0 / n))
cfg = drot.DrotConfig(max_iters=N)
drot.solve(prob, cfg)
t0 = time.perf_counter()
drot.solve(prob, cfg)
print(f"solve():   {(time.perf_counter() - t0) * 1e6 / N:.2f} us/iter (incl. setup)", flush=True)
for mode in ("run", "enqueue"):
    s = drot.Session(m, n, np.float64, drot.DrotConfig(max_iters=N if mode == "run" else 10 ** 9))
    s.gen_uniform(1, 0.0, 1.0, "uniform")
    s.init()
    s.prepare(N)
    s.synchronize()
    t0 = time.perf_counter()
    if mode == "run":
        s.run()
    else:
        s.enqueue(N)
        s.synchronize()
    print(f"{mode}: {(time.perf_counter() - t0) * 1e6 / N:.2f} us/iter", s.status()[1], flush=True)
    s.close()
