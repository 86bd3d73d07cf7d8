"""Worker of tests/test_p2p_gpu.py::test_world2_in_process (run in a fresh
process: CUDA_MODULE_LOADING=EAGER must be set before CUDA initializes --
with lazy loading, the first launch of a kernel may wait for the device to
drain, which a peer session's spinning exchange on the same device never
does).  Prints one JSON object."""
import json
import os
import sys
import threading

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ["DROTB_TAIL_CTAS"] = "1"
# several spinning tails + the next K1 must fit on one device at once
os.environ["DROTB_TAIL_GRID"] = str(148 // max(1, int(sys.argv[4]) - 1) // 2 * 2)
os.environ["DROTB_TAIL_NONCOOP"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2110_11738_b200 as drot  # noqa: E402


def par(fns):
    errs = []

    def wrap(f):
        try:
            f()
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    if any(t.is_alive() for t in th):
        print(json.dumps({"error": "exchange deadlock"}), flush=True)
        os._exit(3)
    if errs:
        raise RuntimeError(errs[0])


def main():
    dt = np.float64 if sys.argv[1] == "f64" else np.float32
    m, n, world = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    cfg = drot.DrotConfig(max_iters=100000, use_graphs=False)
    ranges = [drot.shard_rows(m, world, r) for r in range(world)]
    ss = [drot.Session.sharded_p2p(m, n, dt, cfg, r, world, *ranges[r]) for r in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    for s, stm in zip(ss, streams):
        s.set_stream(stm.cuda_stream)
    ptrs = [s.exchange_pointer() for s in ss]
    for s in ss:
        s.attach_peers(pointers=ptrs)
    par([lambda s=s: s.gen_gaussian(5.0, 5, "dyadic") for s in ss])
    par([s.init for s in ss])
    par([s.run for s in ss])
    out = [None] * world

    def fin(r):
        st, it, rep = ss[r].status()
        plan, mu, nu = ss[r].plan()
        out[r] = {"status": st.name, "iterations": it,
                  "report": [rep.objective, rep.r_primal, rep.r_dual, rep.gap],
                  "nu": nu.astype(np.float64).tolist(), "plan": plan.astype(np.float64).tolist()}

    par([lambda r=r: fin(r) for r in range(world)])
    for s in ss:
        s.close()
    print(json.dumps(out), flush=True)


main()
os._exit(0)
