"""Time-to-1e-4 on the north_star scaling instance (BASELINE configs[4]):
m = n = 10^5 fp32 Gaussian (seed 0), dyadic-uniform marginals, reference
defaults (rho0 = 2, tol 1e-4 x 3), rows sharded over the GPUs of one node,
generated on each rank's device.  Not part of bench.py's default run: the
solve needs ~1e5+ iterations (minutes even on 8 GPUs).  The sharded solve is
bit-identical to the one-GPU solve, so every GPU count reports the same
iteration count.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
      scripts/c5_time_to_tol.py [--size 100000] [--max-iters 2000000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=100000)
    ap.add_argument("--max-iters", type=int, default=2000000)
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"])
    args = ap.parse_args()
    import torch
    import paper_2110_11738_b200 as drot
    from bench import make_shard
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = drot.DrotConfig(max_iters=args.max_iters, record_trace=False, device=local)
    size = args.size
    if world > 1:
        sess = make_shard(drot, dist, args, size, size, np.float32, cfg, rank, world)
    else:
        sess = drot.Session(size, size, np.float32, cfg)
    stream = torch.cuda.Stream()
    sess.set_stream(stream.cuda_stream)
    sess.gen_gaussian(5.0, 0, "dyadic")
    sess.init()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    e0.record(stream)
    sess.run()
    e1.record(stream)
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    if dist is not None:
        t = torch.tensor([sec], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    st, iters, rep = sess.status()
    sess.close()
    if rank == 0:
        print(json.dumps({"config": f"C5 {size}x{size} fp32, {world} GPU(s)", "seconds": sec,
                          "wall_seconds_rank0": time.perf_counter() - t0, "iterations": iters,
                          "status": st.name, "ms_per_iteration": 1e3 * sec / max(iters, 1),
                          "objective": rep.objective, "r_primal": rep.r_primal,
                          "r_dual": rep.r_dual, "gap": rep.gap}), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
