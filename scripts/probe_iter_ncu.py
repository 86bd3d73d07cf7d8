"""Dev aid: a few iterations of the single-launch iteration for ncu."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_11738_b200 as drot  # noqa: E402

m = n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
s = drot.Session(m, n, np.float32, drot.DrotConfig(tol_primal=-1.0, max_iters=10 ** 9))
s.gen_gaussian(5.0, 0, "dyadic")
s.init()
s.enqueue(8)
s.status()
s.close()
