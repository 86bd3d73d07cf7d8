"""Dev aid: kernel start / end times of the solve loop from CUPTI (torch
profiler), no device-side instrumentation: per-iteration K1 and tail
durations and the gaps between them, for m = n = SIZE.
usage: python scripts/probe_cupti.py SIZE f32|f64 [K]"""
import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2110_11738_b200 as drot  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
dt = {"f32": np.float32, "f64": np.float64}[sys.argv[2] if len(sys.argv) > 2 else "f64"]
K = int(sys.argv[3]) if len(sys.argv) > 3 else 64
s = drot.Session(m, m, dt, drot.DrotConfig(tol_primal=-1.0, max_iters=10 ** 12))
st = torch.cuda.Stream()
s.set_stream(st.cuda_stream)
s.gen_gaussian(5.0, 0, "dyadic")
s.init()
s.enqueue(16)
s.prepare(K)
s.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.enqueue(K)
    s.synchronize()
path = os.path.join(tempfile.gettempdir(), "cupti_trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
ks = sorted((e["ts"], e["ts"] + e["dur"], e["name"]) for e in ev
            if e.get("cat") == "kernel")
k1 = [(a, b) for a, b, n in ks if "pass_kernel" in n]
tl = [(a, b) for a, b, n in ks if "tail" in n and "finalize" not in n]
print(f"{m}x{m} {np.dtype(dt).name}: {len(k1)} sweeps, {len(tl)} tails")
if k1 and tl:
    k1d = np.array([b - a for a, b in k1])
    tld = np.array([b - a for a, b in tl])
    n_ = min(len(k1), len(tl)) - 1
    g1 = np.array([tl[i][0] - k1[i][1] for i in range(n_)])       # sweep end -> tail start
    g2 = np.array([k1[i + 1][1] - tl[i][1] for i in range(n_)])   # tail end -> next sweep end
    it = np.array([k1[i + 1][1] - k1[i][1] for i in range(n_)])
    print(f"  sweep (K1) duration  mean {k1d.mean():.2f} us (min {k1d.min():.2f})")
    print(f"  tail duration        mean {tld.mean():.2f} us (min {tld.min():.2f})")
    print(f"  sweep end -> tail start  mean {g1.mean():.2f} us")
    print(f"  tail end -> next sweep end  mean {g2.mean():.2f} us")
    print(f"  iteration (sweep end to sweep end)  mean {it.mean():.2f} us")
    print("  first kernels:", [(n.split('<')[0][-24:], round(b - a, 2)) for a, b, n in ks[:6]])
s.close()
