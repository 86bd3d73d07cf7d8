"""Dev aid: L2 policy variants (DROTB_L2HINT bits) on the default path."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_11738_b200 as drot  # noqa: E402

for dt in (np.float32, np.float64):
    for hint in ("2",):
        os.environ["DROTB_L2HINT"] = hint
        m = n = 10000
        s = drot.Session(m, n, dt, drot.DrotConfig(tol_primal=-1.0, max_iters=10 ** 9))
        s.gen_gaussian(5.0, 0, "dyadic")
        s.init()
        s.enqueue(20)
        best = None
        for _ in range(3):
            r = s.run_timed(200)
            if best is None or r["total_ms"] < best["total_ms"]:
                best = r
        print(f"{np.dtype(dt).name} l2hint {hint}: {best['total_ms'] / 200 * 1e3:.1f} us/iter, sweep "
              f"{best['pass_ms'] / 200 * 1e3:.1f} us, {200 / best['total_ms'] * 1e3:.0f} it/s",
              flush=True)
        s.close()
