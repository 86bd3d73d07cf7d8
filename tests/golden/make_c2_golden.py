"""Generates the C2 golden (tests/golden/c2_f32.json + c2_f32_support.npy):
the reference's solve<float> (solver.hpp:372-540) on the headline instance,
run to tol 1e-4 ON THE B200 in order=reference.

Why not the CPU reference itself: at m = n = 10 000 fp32 it needs ~55 ms per
iteration on 16 host threads and ~1.5e5 iterations (~2.5 h); order=reference
is the repo's bitwise restatement of that exact trajectory (iterates, duals,
gate decisions and iteration counts identical to the unmodified reference,
asserted against oracle/_ref on 13 configurations, 30 committed golden
digests and fixed-K runs at this very size in tests/test_fullsize_gpu.py).

Instance: gen_gaussian_problem_as<float>(m=n=10 000, sigma_t=5, seed 0)
(probgen.hpp:131-180), dyadic-uniform fp32 marginals, the
reference defaults (rho0 = 2, tol 1e-4 x 3, skip_cost, trace on) except
max_iters = 400 000 (the default 1e5 stops short of the tolerance).

Run on a GPU box:  python tests/golden/make_c2_golden.py [out_dir]
It also solves the same instance in the default fast order and prints the
comparison the GPU test asserts (tests/test_golden_c2_gpu.py).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

M = N = 10000
MAX_ITERS = 400000


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def problem():
    from pyoracle import Oracle, dyadic_marginal
    C, _, _ = Oracle("orc").gen_gaussian(M, N, 5.0, 0)
    C = C.astype(np.float32).reshape((M, N), order="F")
    return C, dyadic_marginal(M, np.float32), dyadic_marginal(N, np.float32)


def support(plan):
    x = plan.ravel(order="F")
    return np.flatnonzero(x > 1e-6 * float(x.max())).astype(np.int64)


def solve(drot, C, p, q, order):
    cfg = drot.DrotConfig(order=drot.Order[order], max_iters=MAX_ITERS)
    t0 = time.time()
    res = drot.solve(drot.TransportProblem(C, p, q), cfg)
    return res, time.time() - t0


def main(out_dir):
    import paper_2110_11738_b200 as drot
    C, p, q = problem()
    res, wall = solve(drot, C, p, q, "reference")
    plan = res.plan.x
    tr = np.array([[r.iter, r.r_primal, r.r_dual, r.gap, r.objective, r.ergodic_objective,
                    r.fixed_point_residual] for r in res.trace.rows], dtype=np.float64)
    supp = support(plan)
    gold = {
        "spec": {"m": M, "n": N, "dtype": "float32", "cost": "gaussian", "seed": 0,
                 "sigma_t": 5.0, "marginals": "dyadic", "cfg": {"max_iters": MAX_ITERS}},
        "generator": "tests/golden/make_c2_golden.py on a B200, order=reference (bitwise "
                     "reference solve<float>)",
        "iterations": res.trace.iterations,
        "status": res.status.name,
        "report": {k: float(getattr(res.report, k)).hex()
                   for k in ("r_primal", "r_dual", "gap", "objective")},
        "report_float": {k: float(getattr(res.report, k))
                         for k in ("r_primal", "r_dual", "gap", "objective")},
        "plan_sha256": sha(plan.ravel(order="F")),
        "mu_sha256": sha(res.cert.mu),
        "nu_sha256": sha(res.cert.nu),
        "trace_rows": len(res.trace.rows),
        "trace_sha256": sha(tr),
        "trace_every_10000": tr[::10000].tolist(),
        "nnz_1e-8": int((plan > 1e-8).sum()),
        "support_1e-6_rel": int(supp.size),
        "plan_sum": float(plan.astype(np.float64).sum()),
        "wall_s_b200_reference_order": wall,
    }
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "c2_f32.json"), "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    np.save(os.path.join(out_dir, "c2_f32_support.npy"), supp.astype(np.int32))
    print(json.dumps({k: v for k, v in gold.items() if k != "trace_every_10000"}), flush=True)
    drot.release_device_cache()
    fast, fwall = solve(drot, C, p, q, "fast")
    fs = support(fast.plan.x)
    sym = np.setxor1d(fs, supp, assume_unique=True).size
    print(json.dumps({"fast_iterations": fast.trace.iterations, "fast_status": fast.status.name,
                      "fast_objective": fast.report.objective,
                      "objective_rel": abs(fast.report.objective - gold["report_float"]["objective"])
                      / abs(gold["report_float"]["objective"]),
                      "support_fast": int(fs.size), "support_symdiff": int(sym),
                      "fast_wall_s": fwall}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "golden"))
