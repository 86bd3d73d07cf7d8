"""Worker of tests/test_p2p_gpu.py::test_ipc_two_processes: one shard per
process on the SAME GPU, peers attached through CUDA IPC handles exchanged
over torch.distributed (gloo) -- the one-process-per-GPU production path.
The two contexts time-slice the device, so each exchange costs up to a time
slice; the run is short.  Writes a JSON result to argv[3]."""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402
import paper_2110_11738_b200 as drot  # noqa: E402


def main():
    rank, world, out_path = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, n, iters = 640, 480, 40
    cfg = drot.DrotConfig(tol_primal=-1.0, max_iters=iters, use_graphs=False)
    r0, r1 = drot.shard_rows(m, world, rank)
    s = drot.Session.sharded_p2p(m, n, np.float64, cfg, rank, world, r0, r1)
    handles = [None] * world
    dist.all_gather_object(handles, s.exchange_handle())
    s.attach_peers(handles=handles)
    s.gen_gaussian(5.0, 7, "dyadic")
    s.init()
    s.run()
    st, it, rep = s.status()
    plan, mu, nu = s.plan()
    s.close()
    with open(out_path, "w") as f:
        json.dump({"status": st.name, "iterations": it,
                   "report": [rep.objective, rep.r_primal, rep.r_dual, rep.gap],
                   "nu": nu.tolist(), "plan": plan.tolist()}, f)
    dist.barrier()
    dist.destroy_process_group()


main()
