"""Dev aid: graph-timed microseconds per solve-loop iteration (no stamps),
fast order, m = n = SIZE Gaussian, averaged over K iterations after warm-up.
usage: python scripts/probe_iter.py SIZE f32|f64 [K]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_11738_b200 as drot  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
dt = {"f32": np.float32, "f64": np.float64}[sys.argv[2] if len(sys.argv) > 2 else "f64"]
K = int(sys.argv[3]) if len(sys.argv) > 3 else 400
s = drot.Session(m, m, dt, drot.DrotConfig(tol_primal=-1.0, max_iters=10 ** 12))
st = torch.cuda.Stream()
s.set_stream(st.cuda_stream)
if os.environ.get("PROBE_UNIFORM"):
    s.gen_uniform(1, 0.0, 1.0, "uniform")
else:
    s.gen_gaussian(5.0, 0, "dyadic")
s.init()
s.enqueue(16)
s.prepare(K)
s.synchronize()
best = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.enqueue(K)
    e1.record(st)
    torch.cuda.synchronize()
    best.append(e0.elapsed_time(e1) * 1e3 / K)
print(f"{m}x{m} {np.dtype(dt).name} ctail={os.environ.get('DROTB_CTAIL', 'default')}: "
      f"{min(best):.2f} us/iter (reps {', '.join(f'{b:.2f}' for b in best)})")
s.close()
