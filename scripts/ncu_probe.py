"""Short fixed workload for ncu captures (10k x 10k fp32 Gaussian, fast order).

  python scripts/ncu_probe.py SIZE DTYPE ITERS [CHUNK]

Default (persistent solver kernel): ITERS iterations in launches of CHUNK
iterations (CHUNK=2: one fold + one skip sweep per launch).  With
DROTB_PERSIST=0 the per-launch kernels run eagerly (no graphs: ncu cannot
profile kernels inside graphs with conditional nodes).
"""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2110_11738_b200 as drot
m = n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
dt = np.float32 if (len(sys.argv) < 3 or sys.argv[2] == "f32") else np.float64
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 8
chunk = int(sys.argv[4]) if len(sys.argv) > 4 else 2
cfg = drot.DrotConfig(tol_primal=-1.0, max_iters=10**9, use_graphs=False)
s = drot.Session(m, n, dt, cfg)
s.gen_gaussian(5.0, 0, "dyadic")
s.init()
done = 0
while done < iters:
    s.enqueue(min(chunk, iters - done))
    done += chunk
s.synchronize()
print("done", s.status()[1], "persistent grid", s.persistent_grid)
