import os, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2110_11738_b200 as drot
m, n = 500, 400
dt = np.float32
cfg = drot.DrotConfig(max_iters=100000)
def shard(tag):
    os.environ["DROTB_TAIL_CTAS"] = "2"
    s = drot.Session.sharded_p2p(m, n, dt, cfg, 0, 1, 0, m)
    del os.environ["DROTB_TAIL_CTAS"]
    s.attach_peers(pointers=[s.exchange_pointer()])
    s.gen_gaussian(5.0, 3, "dyadic"); s.init(); s.run()
    print(tag, s.status()[:2]); s.close()
def single(tag):
    s1 = drot.Session(m, n, dt, cfg); s1.gen_gaussian(5.0, 3, "dyadic"); s1.init(); s1.run()
    print(tag, s1.status()[:2]); s1.close()
mode = sys.argv[1]
if mode == "a":
    shard("shard alone"); shard("shard again")
else:
    single("single"); shard("shard after single"); shard("shard again")
