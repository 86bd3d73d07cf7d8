"""Dev aid: world-1 p2p shard vs the single-GPU session (iterations, book)."""
import os, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2110_11738_b200 as drot
from paper_2110_11738_b200 import _lib
m, n = 500, 400
for dt in (np.float64, np.float32):
    cfg = drot.DrotConfig(max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 100000)
    s1 = drot.Session(m, n, dt, cfg); s1.gen_gaussian(5.0, 3, "dyadic"); s1.init(); s1.run()
    print("single", dt.__name__, s1.status()); s1.close()
    os.environ["DROTB_TAIL_CTAS"] = "2"
    s = drot.Session.sharded_p2p(m, n, dt, cfg, 0, 1, 0, m)
    del os.environ["DROTB_TAIL_CTAS"]
    s.attach_peers(pointers=[s.exchange_pointer()])
    s.gen_gaussian(5.0, 3, "dyadic"); s.init(); s.run()
    print("shard ", dt.__name__, s.status()); s.close()
