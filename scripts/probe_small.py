"""Dev aid: per-iteration time at small sizes (tail-bound) per L2 policy."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_11738_b200 as drot  # noqa: E402

for hint in ("2", "0", "2", "0"):
    os.environ["DROTB_L2HINT"] = hint
    for (m, dt) in ((1000, np.float64), (2000, np.float32)):
        s = drot.Session(m, m, dt, drot.DrotConfig(tol_primal=-1.0, max_iters=10 ** 9))
        s.gen_gaussian(5.0, 0, "dyadic")
        s.init()
        s.enqueue(100)
        best = None
        for _ in range(3):
            r = s.run_timed(400)
            if best is None or r["total_ms"] < best["total_ms"]:
                best = r
        s.close()
        print(f"{m}^2 {np.dtype(dt).name} l2hint {hint}: {best['total_ms'] / 400 * 1e3:.2f} us/iter, "
              f"sweep {best['pass_ms'] / 400 * 1e3:.2f} us", flush=True)
