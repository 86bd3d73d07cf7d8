"""Short fixed workload for ncu captures (m = n = SIZE Gaussian, fast order,
eager launches: ncu profiles kernels one by one, so no graphs).

  python scripts/ncu_probe.py SIZE DTYPE ITERS
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2110_11738_b200 as drot

m = n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
dt = np.float32 if (len(sys.argv) < 3 or sys.argv[2] == "f32") else np.float64
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 8
cfg = drot.DrotConfig(tol_primal=-1.0, max_iters=10**9, use_graphs=False)
s = drot.Session(m, n, dt, cfg)
s.gen_gaussian(5.0, 0, "dyadic")
s.init()
s.enqueue(iters)
s.synchronize()
print("done", s.status()[1])
