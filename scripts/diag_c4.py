"""Dev aid: trace rows of reference vs fast order around the end of one
golden case (default c4grid_f32_rho2_tol1e-3)."""
import json, os, sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
import paper_2110_11738_b200 as drot
from pyoracle import Oracle
from test_solve_gpu import golden_problem, dcfg
name = sys.argv[1] if len(sys.argv) > 1 else "c4grid_f32_rho2_tol1e-3"
gold = json.load(open("tests/golden/golden.json"))[name]
ref = Oracle("ref")
prob, x0, kw = golden_problem(drot, ref, gold)
out = {}
for order in ("reference", "fast"):
    r = drot.solve(prob, dcfg(drot, order, **kw), x0)
    out[order] = r
    print(order, os.environ.get("DROTB_FX", ""), os.environ.get("DROTB_TAIL_GATE", ""), r.status.name, r.trace.iterations, r.report)
R, F = out["reference"].trace.rows, out["fast"].trace.rows
it = gold["iterations"]
for k in list(range(it - 4, it + 2)):
    if k - 1 < len(R) and k - 1 < len(F):
        a, b = R[k - 1], F[k - 1]
        print(k, f"ref rp {a.r_primal:.6e} rd {a.r_dual:.6e} gap {a.gap:.6e} | fast rp {b.r_primal:.6e} rd {b.r_dual:.6e} gap {b.gap:.6e}")
