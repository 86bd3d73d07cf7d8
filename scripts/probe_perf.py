"""Quick per-iteration timing probe (development aid; bench.py is the contract)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2110_11738_b200 as drot

def probe(m, n, dt, order="fast", skip=True, K=200, W=10, trace=True):
    cfg = drot.DrotConfig(order=drot.Order[order], tol_primal=-1.0, max_iters=10**9,
                          skip_cost=skip, record_trace=trace)
    s = drot.Session(m, n, dt, cfg)
    t0 = time.time()
    s.gen_gaussian(5.0, 0, "dyadic")
    t1 = time.time()
    s.init()
    s.enqueue(W)
    s.synchronize()
    t2 = time.perf_counter()
    s.enqueue(K)
    s.synchronize()
    t3 = time.perf_counter()
    dt_it = (t3 - t2) / K
    bf, bs_ = s.pass_bytes()
    avg_bytes = (bf + bs_) / 2 if skip else bf
    print(f"{m}x{n} {np.dtype(dt).name} order={order} skip={skip} trace={trace}: "
          f"{dt_it*1e6:.1f} us/iter, {1/dt_it:.0f} it/s, {avg_bytes/dt_it/1e9:.0f} GB/s "
          f"(gen {t1-t0:.1f}s)", flush=True)
    st = s.status()
    s.close()

if __name__ == "__main__":
    probe(10000, 10000, np.float32)
    probe(10000, 10000, np.float32, skip=False)
    probe(10000, 10000, np.float32, trace=False)
    probe(10000, 10000, np.float64, K=100)
    probe(1000, 1000, np.float64, K=2000)
    probe(1000, 1000, np.float64, order="reference", K=200)
    probe(40000, 5000, np.float32)
