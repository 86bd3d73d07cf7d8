import os, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2110_11738_b200 as drot
m = int(sys.argv[1]); dt = np.float64 if sys.argv[2] == "f64" else np.float32
os.environ["DROTB_SMALL_MB"] = sys.argv[3]
C = drot.counter_uniform(1, m * m).astype(dt)
prob = drot.TransportProblem(C.reshape((m, m), order="F"), drot.dyadic_marginal(m, dt), drot.dyadic_marginal(m, dt))
r = drot.solve(prob, drot.DrotConfig(max_iters=10))
print("ok", r.trace.iterations, r.status)
