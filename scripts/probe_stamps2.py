"""Dev aid: phase timeline of the cooperative tail (DROTB_TAIL_STAMPS=1)."""
import ctypes as C, os, sys
import numpy as np
os.environ["DROTB_TAIL_STAMPS"] = "1"
sys.path.insert(0, ".")
import torch
import paper_2110_11738_b200 as drot
from paper_2110_11738_b200 import _lib
for (m, n, dt) in [(10000, 10000, np.float32), (1000, 1000, np.float64)]:
    s = drot.Session(m, n, dt, drot.DrotConfig(tol_primal=-1.0, max_iters=10**12, use_graphs=False))
    st = torch.cuda.Stream(); s.set_stream(st.cuda_stream)
    s.gen_gaussian(5.0, 0, "dyadic"); s.init(); s.enqueue(10); s.synchronize()
    buf = (C.c_uint64 * 8)()
    _lib.load().drotb_session_tail_stamps(s.handle, buf)
    acc = np.zeros(7)
    K = 40
    for _ in range(K):
        s.enqueue(1); s.synchronize()
        _lib.load().drotb_session_tail_stamps(s.handle, buf)
        v = np.array(list(buf), dtype=np.float64)
        acc += (v[1:8] - v[0]) / 1e3
    acc /= K
    names = ["A done", "RB1 done", "all past RB1", "B done", "loads issued", "warp sums done", "thread0 sums done"]
    print(f"{m}x{n} {np.dtype(dt).name}: " + ", ".join(f"{nm} {x:.1f}" for nm, x in zip(names, acc)) + " us after first CTA entry")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); s.enqueue(50); e1.record(st); torch.cuda.synchronize()
    r = s.run_timed(50)
    print(f"   eager {e0.elapsed_time(e1)*1e3/50:.1f} us/iter, sweep {r['pass_ms']*1e3/50:.1f} us")
    s.close()
