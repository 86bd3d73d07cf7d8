import os, sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import torch
import paper_2110_11738_b200 as drot
m = n = 1000
for label, kw in [("default tol", {}), ("tol -1", {"tol_primal": -1.0}), ("no trace", {"record_trace": False}),
                  ("maxit 1e12", {"max_iters": 10 ** 12, "tol_primal": -1.0})]:
    kw2 = dict(kw)
    kw2.setdefault("max_iters", 10000)
    s = drot.Session(m, n, np.float64, drot.DrotConfig(**kw2))
    s.gen_uniform(1, 0.0, 1.0, "uniform")
    s.init()
    s.enqueue(16); s.synchronize()
    t0 = time.perf_counter()
    if kw2["max_iters"] == 10000:
        s.run()
    else:
        s.enqueue(9984); s.synchronize()
    t = time.perf_counter() - t0
    print(f"{label}: {t * 1e6 / 9984:.2f} us/iter (run)" , s.status()[1], flush=True)
    s.close()
