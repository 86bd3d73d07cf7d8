"""Dev aid: device timeline of the solve loop (DROTB_TAIL_STAMPS=1), CUDA
graphs as in the bench.  The stamps are global atomics: they slow the tail
by several us -- read the phases' order and relative length here, and time
iterations with scripts/probe_iter.py.  Per iteration (averaged over 60): K1 entry / exit,
tail entry, merge done, scalar section done, update done, tail exit, all
relative to the first K1 CTA entry of that iteration.
usage: python scripts/probe_timeline.py [m] [dtype] [iters]"""
import ctypes as C
import os
import sys

import numpy as np

os.environ["DROTB_TAIL_STAMPS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_11738_b200 as drot  # noqa: E402
from paper_2110_11738_b200 import _lib  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
dt = {"f32": np.float32, "f64": np.float64}[sys.argv[2] if len(sys.argv) > 2 else "f32"]
K = int(sys.argv[3]) if len(sys.argv) > 3 else 64
s = drot.Session(m, m, dt, drot.DrotConfig(tol_primal=-1.0, max_iters=10 ** 12))
st = torch.cuda.Stream()
s.set_stream(st.cuda_stream)
s.gen_gaussian(5.0, 0, "dyadic")
s.init()
s.enqueue(8)
s.prepare(K)
s.synchronize()
buf = (C.c_uint64 * 3072)()
_lib.load().drotb_session_tail_stamps(s.handle, buf)  # reset
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
s.enqueue(K)
e1.record(st)
torch.cuda.synchronize()
_lib.load().drotb_session_tail_stamps(s.handle, buf)
a = np.array(list(buf), dtype=np.float64).reshape(64, 24, 2)
it0 = 8
names = ["K1 entry", "K1 exit", "tail entry", "merge done", "book stored", "update done", "tail exit",
         "K1 swept/strips", "r/s stored", "K1 released", "barrier passed", "totals loaded",
         "join (all roles)", "update done(w2)", "upd sums red(w2)", "decide done(w0)",
         "pt16", "pt17", "pt18", "pt19", "pt20", "pt21", "pt22", "pt23"]
NP = len(names)
rows = []
for k in range(it0 + 2, it0 + K - 1):
    sl = a[k & 63]
    base = sl[0, 0]
    nxt = a[(k + 1) & 63][0, 0]
    if base == 2 ** 64 - 1 or nxt == 2 ** 64 - 1:
        continue
    rows.append([(sl[p, 0] - base) / 1e3 for p in range(NP)] +
                [(sl[p, 1] - base) / 1e3 for p in range(NP)] + [(nxt - base) / 1e3])
r = np.array(rows)
mean = r.mean(axis=0)
print(f"{m}x{m} {np.dtype(dt).name}: {len(r)} iterations, graph-timed "
      f"{e0.elapsed_time(e1) * 1e3 / K:.1f} us/iter; mean us after the first K1 CTA entry:")
order = [0, 9, 7, 1, 2, 8, 3, 10, 11, 15, 13, 14, 12, 4, 5, 6]
for p in order:
    if mean[p] > 1e9:  # point not recorded
        continue
    print(f"  {names[p]:14s} min {mean[p]:8.1f}  max {mean[NP + p]:8.1f}")
nx = mean[2 * NP]
print(f"  next K1 entry      {nx:8.1f}")
print(f"  gaps: K1 last exit -> tail first entry {mean[2] - mean[NP + 1]:.1f} us; "
      f"tail last exit -> next K1 entry {nx - mean[NP + 6]:.1f} us; "
      f"tail span {mean[NP + 6] - mean[2]:.1f} us; K1 span {mean[NP + 1] - mean[0]:.1f} us")
for k in (0, 1):  # the two iteration parities (fold / skip-cost sweeps) separately
    sub = r[k::2]
    mk = sub.mean(axis=0)
    print(f"  parity {k}: K1 span {np.mean(sub[:, NP + 1] - sub[:, 0]):.1f} us, "
          f"iteration {np.mean(sub[:, 2 * NP]):.1f} us; " +
          ", ".join(f"{names[p]} {mk[p]:.1f}/{mk[NP + p]:.1f}" for p in order if mk[p] < 1e9))
s.close()
