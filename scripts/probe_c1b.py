import os, sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2110_11738_b200 as drot
m = n = 1000
C = drot.counter_uniform(1, m * n)
prob = drot.TransportProblem(C.reshape((m, n), order="F"), np.full(m, 1.0 / m), np.full(n, 1.0 / n))
for rep in range(3):
    t0 = time.perf_counter()
    drot.solve(prob, drot.DrotConfig(max_iters=200))
    t1 = time.perf_counter()
    res = drot.solve(prob, drot.DrotConfig())
    t2 = time.perf_counter()
    print(f"rep {rep}: warm(200) {t1 - t0:.3f} s, full {t2 - t1:.3f} s, {res.trace.iterations} it", flush=True)
