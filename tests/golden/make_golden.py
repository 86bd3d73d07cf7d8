"""Generates tests/golden/golden.json from the UNMODIFIED reference
(oracle/_ref/libdrotref.so, built by `make -C oracle` from /root/reference).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py [case ...]

Each case records the reference's solve outputs bit-exactly: iteration
count, status, the ResidualReport doubles (hex), SHA-256 of the plan / mu /
nu bytes (column-major, the reference's storage order) and of the trace rows,
plus support sizes.  The inputs are regenerated identically by the reference's
own generators (CounterRng, gen_gaussian_problem) on the GPU box, so only
these small digests are committed.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import Oracle, default_config, dyadic_marginal  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hexf(x: float) -> str:
    return float(x).hex()


def problem(R: Oracle, spec: dict):
    m, n, dt = spec["m"], spec["n"], np.dtype(spec["dtype"])
    kind = spec["cost"]
    if kind == "uniform_random":
        C = R.random_unit(spec["seed"], m * n)
    elif kind == "gaussian":
        C, pd, qd = R.gen_gaussian(m, n, seed=spec["seed"],
                                   dirichlet=spec["marginals"] == "dirichlet")
    else:
        raise ValueError(kind)
    marg = spec["marginals"]
    if marg == "uniform":
        p = np.full(m, 1.0 / m)
        q = np.full(n, 1.0 / n)
    elif marg == "dyadic":
        p = dyadic_marginal(m, dt).astype(np.float64)
        q = dyadic_marginal(n, dt).astype(np.float64)
    elif marg == "dirichlet":  # probgen.hpp:115-127 (Dirichlet(1..1), substreams 4/5)
        p, q = pd, qd
    elif marg == "random_simplex":  # test_reference.cpp:22-29 pattern
        from pyoracle import Oracle as _O  # noqa
        orc = Oracle("orc")
        import ctypes as Cc
        f = orc.lib.orc_random_simplex
        f.argtypes = [Cc.c_int64, Cc.c_uint64, Cc.c_void_p]
        f.restype = None
        p = np.empty(m)
        q = np.empty(n)
        f(m, spec["seed"] ^ 0x1111, p.ctypes.data)
        f(n, spec["seed"] ^ 0x2222, q.ctypes.data)
    else:
        raise ValueError(marg)
    return C.astype(dt), p.astype(dt), q.astype(dt)


def warm_start(R: Oracle, spec: dict):
    """Optional x0 (solver.hpp:143-159): a nonnegative m x n matrix in
    column-major order, CounterRng(seed) uniforms scaled by 1/(m*n)."""
    x0 = spec.get("x0")
    if x0 is None:
        return None
    m, n = spec["m"], spec["n"]
    return (R.random_unit(x0["seed"], m * n) * (x0["scale"] / (m * n))).astype(spec["dtype"])


CASES = {
    # SURVEY §8(c) golden runs (reference solve<double>, defaults)
    "c1_f64": dict(m=1000, n=1000, dtype="float64", cost="uniform_random", seed=1,
                   marginals="uniform", cfg={}),
    "gauss1000_f64": dict(m=1000, n=1000, dtype="float64", cost="gaussian", seed=0,
                          marginals="uniform", cfg={}),
    "gauss1000_f32": dict(m=1000, n=1000, dtype="float32", cost="gaussian", seed=0,
                          marginals="dyadic", cfg={}),
    "rect_f64": dict(m=600, n=300, dtype="float64", cost="uniform_random", seed=7,
                     marginals="random_simplex", cfg={}),
    # fixed-K trajectories (tolerances unreachable)
    "gauss2000_f64_k300": dict(m=2000, n=2000, dtype="float64", cost="gaussian", seed=0,
                               marginals="uniform",
                               cfg=dict(max_iters=300, tol_primal=-1.0)),
    "gauss2000_f32_k300": dict(m=2000, n=2000, dtype="float32", cost="gaussian", seed=0,
                               marginals="dyadic",
                               cfg=dict(max_iters=300, tol_primal=-1.0)),
    "rect4000x500_f32_k200": dict(m=4000, n=500, dtype="float32", cost="uniform_random",
                                  seed=5, marginals="dyadic",
                                  cfg=dict(max_iters=200, tol_primal=-1.0)),
    # round 2: converged runs SURVEY §6 measured but round 1 never pinned
    "dirichlet1000_f64": dict(m=1000, n=1000, dtype="float64", cost="gaussian", seed=0,
                              marginals="dirichlet", cfg={}),
    "gauss2000_f64": dict(m=2000, n=2000, dtype="float64", cost="gaussian", seed=0,
                          marginals="uniform", cfg={}),
    # valid warm start x0 (solver.hpp:143-159)
    "warm_x0_f64": dict(m=300, n=300, dtype="float64", cost="uniform_random", seed=3,
                        marginals="uniform", x0=dict(seed=11, scale=2.0), cfg={}),
    "warm_x0_f32": dict(m=256, n=200, dtype="float32", cost="gaussian", seed=2,
                        marginals="dyadic", x0=dict(seed=12, scale=1.0), cfg={}),
}

# C4 grid (BASELINE configs[3]) at 256^2 fp32: rho0 x tol, including the
# warm-up preset 1/ln m (solver.hpp:47-49) and tol 1e-6, where the reference
# stalls until max_iters; max_iters = the reference default 1e5.
C4_RHO = {"0.5": 0.5, "1": 1.0, "2": 2.0, "4": 4.0, "invlnm": None}
C4_TOL = ["1e-3", "1e-4", "1e-5", "1e-6"]
for _rk, _rv in C4_RHO.items():
    for _tk in C4_TOL:
        _t = float(_tk)
        _rho = _rv if _rv is not None else 1.0 / __import__("math").log(256)
        CASES[f"c4grid_f32_rho{_rk}_tol{_tk}"] = dict(
            m=256, n=256, dtype="float32", cost="gaussian", seed=0, marginals="dyadic",
            cfg=dict(rho0=_rho, tol_primal=_t, tol_dual=_t, tol_gap=_t))


def run_case(R: Oracle, name: str, spec: dict) -> dict:
    C, p, q = problem(R, spec)
    m, n = spec["m"], spec["n"]
    cfg = default_config(**spec["cfg"])
    t0 = time.time()
    out = R.solve(C, p, q, m, n, cfg, x0=warm_start(R, spec))
    wall = time.time() - t0
    tr = np.array([[r[k] for k in ("iter", "r_primal", "r_dual", "gap", "objective",
                                   "ergodic_objective", "fixed_point_residual")]
                   for r in out.trace], dtype=np.float64)
    plan = out.plan.astype(np.float64)
    mx = float(plan.max()) if plan.size else 0.0
    return {
        "spec": spec,
        "iterations": out.iterations,
        "status": out.status,
        "report": {k: hexf(v) for k, v in out.report.items()},
        "report_float": out.report,
        "plan_sha256": sha(out.plan),
        "mu_sha256": sha(out.mu),
        "nu_sha256": sha(out.nu),
        "trace_rows": len(out.trace),
        "trace_sha256": sha(tr),
        "trace_last": out.trace[-1] if out.trace else None,
        "nnz_1e-8": int((plan > 1e-8).sum()),
        "support_1e-6_rel": int((plan > 1e-6 * mx).sum()),
        "plan_sum": float(plan.sum()),
        "wall_s_ref_8threads": wall,
    }


def main(names):
    R = Oracle("ref")
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    data["_meta"] = {
        "generator": "tests/golden/make_golden.py",
        "reference": "oracle/_ref/libdrotref.so (unmodified /root/reference/proj/core, "
                     "-O3 -DNDEBUG -std=gnu++20)",
        "host_workers": R.hardware_workers(),
    }
    for name in names or CASES:
        print("case", name, flush=True)
        data[name] = run_case(R, name, CASES[name])
        print(" ", data[name]["iterations"], data[name]["status"],
              data[name]["report_float"], f"{data[name]['wall_s_ref_8threads']:.1f}s", flush=True)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
