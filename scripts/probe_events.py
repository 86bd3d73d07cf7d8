"""Dev aid: cost of the per-sweep timing events inside the timed graphs."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2110_11738_b200 as drot  # noqa: E402

m = n = 10000
s = drot.Session(m, n, np.float32, drot.DrotConfig(tol_primal=-1.0, max_iters=10 ** 9))
st = torch.cuda.Stream()
s.set_stream(st.cuda_stream)
s.gen_gaussian(5.0, 0, "dyadic")
s.init()
s.enqueue(20)
s.synchronize()
for rep in range(3):
    r = s.run_timed(200)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.enqueue(200)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"timed graph (per-sweep events): {r['total_ms'] / 200 * 1e3:.1f} us/iter; "
          f"batch graphs, bracketing events only: {e0.elapsed_time(e1) / 200 * 1e3:.1f} us/iter",
          flush=True)
s.close()
