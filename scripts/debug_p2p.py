"""Dev aid: world = 2 shards in one process, one iteration at a time, with a
watchdog that dumps both exchange buffers' flags through a side stream."""
import ctypes as C
import os
import sys
import threading
import time

import numpy as np

os.environ["CUDA_MODULE_LOADING"] = "EAGER"  # see tests/test_p2p_gpu.py
os.environ["DROTB_TAIL_CTAS"] = "1"
os.environ["DROTB_TAIL_NONCOOP"] = "1"
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2110_11738_b200 as drot  # noqa: E402

cudart = C.CDLL("libcudart.so.12")
m, n = 700, 500
cfg = drot.DrotConfig(max_iters=100000, use_graphs=False)
ranges = [drot.shard_rows(m, 2, r) for r in range(2)]
ss = [drot.Session.sharded_p2p(m, n, np.float64, cfg, r, 2, *ranges[r]) for r in range(2)]
streams = [torch.cuda.Stream() for _ in range(2)]
for s, stm in zip(ss, streams):
    s.set_stream(stm.cuda_stream)
ptrs = [s.exchange_pointer() for s in ss]
for s in ss:
    s.attach_peers(pointers=ptrs)
from paper_2110_11738_b200 import _lib  # noqa: E402
dbg = []
for s in ss:
    a = (C.c_uint64 * 4)()
    _lib.load().drotb_session_debug_ptrs(s.handle, a)
    dbg.append(list(a))
print("debug ptrs", dbg, flush=True)
progress = [0, 0]
stage = ["", ""]


def par(fs):
    th = [threading.Thread(target=f) for f in fs]
    [t.start() for t in th]
    return th


def work(r, nit):
    s = ss[r]
    stage[r] = "gen"
    s.gen_gaussian(5.0, 5, "dyadic")
    stage[r] = "init"
    s.init()
    print(f"rank {r} init done", flush=True)
    for k in range(nit):
        stage[r] = f"enqueue {k}"
        s.enqueue(1)
        stage[r] = f"sync {k}"
        s.synchronize()
        progress[r] = k + 1
        print(f"rank {r} iteration {k + 1}", flush=True)
    stage[r] = "done"


print("start", flush=True)
th = par([lambda r=r: work(r, 12) for r in range(2)])
side = C.c_void_p()
cudart.cudaStreamCreateWithFlags(C.byref(side), 1)
pin = C.c_void_p()
cudart.cudaMallocHost(C.byref(pin), 1024)
t0 = time.time()
while any(t.is_alive() for t in th) and time.time() - t0 < 40:
    time.sleep(5)
    flags = []
    for p in ptrs:
        cudart.cudaMemcpyAsync(pin, C.c_void_p(p), 16, 2, side)
        cudart.cudaMemcpyAsync(C.c_void_p(pin.value + 16), C.c_void_p(p + 256), 16, 2, side)
        cudart.cudaStreamSynchronize(side)
        buf = (C.c_uint64 * 4).from_address(pin.value)
        flags.append((list(buf)[:2], list(buf)[2:4]))
    bars = []
    for d in dbg:
        cudart.cudaMemcpyAsync(pin, C.c_void_p(d[1]), 8, 2, side)
        for g in range(16):
            cudart.cudaMemcpyAsync(C.c_void_p(pin.value + 8 + 4 * g), C.c_void_p(d[1] + 4 * 32 * (1 + g)), 4, 2, side)
        cudart.cudaMemcpyAsync(C.c_void_p(pin.value + 128), C.c_void_p(d[0] + 40), 8, 2, side)
        cudart.cudaStreamSynchronize(side)
        w = (C.c_uint32 * 18).from_address(pin.value)
        it = C.c_int64.from_address(pin.value + 128).value
        bars.append((list(w)[:2], list(w)[2:18], it))
    print("   bars (top count, gen | group counts | book.iter?)", bars, flush=True)
    print(f"t={time.time()-t0:.0f}s progress={progress} stage={stage} iter/setup flags={flags}",
          flush=True)
print("alive:", [t.is_alive() for t in th], flush=True)
os._exit(0)
