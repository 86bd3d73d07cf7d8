"""Dev aid: the bench's plain timed region on torch's current stream."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2110_11738_b200 as drot  # noqa: E402

m = n = 10000
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
s = drot.Session(m, n, np.float32, drot.DrotConfig())
stream = torch.cuda.current_stream(dev)
print("stream handle", stream.cuda_stream)
s.set_stream(stream.cuda_stream)
s.gen_gaussian(5.0, 0, "dyadic")
s.init()
s.run_timed(10)
torch.cuda.synchronize()
for rep in range(2):
    l0 = drot.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s.enqueue(200)
    e1.record(stream)
    torch.cuda.synchronize()
    print("plain", e0.elapsed_time(e1), "ms, launches", drot.kernel_launches() - l0, "status", s.status()[:2])
    r = s.run_timed(200)
    print("timed", r["total_ms"], "ms, sweep", r["pass_ms"] / 200)
s.close()
