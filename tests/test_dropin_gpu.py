"""C++ clients of the drop-in headers on the B200 (built by tests/cpp/Makefile):
the reference-style dropin_solve (SPEC example, bitwise vs the reference
solve), dropin_api (validation, materialize_plan/_y, ErgodicMean, the pool
constructor, the Gaussian generator), and the reference's OWN
proj/tests/test_fused.cpp compiled unchanged against include/drot_b200."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
BIN = os.path.join(CPP, "_bin")


def _exe(name):
    # rebuild what can be rebuilt here (own clients always; the reference's
    # tests only where /root/reference exists -- else the binaries built in
    # the CPU container travel with the snapshot)
    subprocess.run(["make", "-s", "-C", CPP], capture_output=True, text=True)
    path = os.path.join(BIN, name)
    if not os.access(path, os.X_OK):
        pytest.skip(f"{name} not built (needs the reference tree at build time)")
    return path


def _summary(r):
    assert r.returncode == 0, r.stdout + r.stderr
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_cpp_dropin_runs(ref):
    import numpy as np
    from pyoracle import default_config
    r = subprocess.run([_exe("dropin_solve")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [json.loads(x) for x in r.stdout.strip().splitlines()]
    out = lines[0]
    assert out["status"] == "converged"
    assert abs(out["objective"] - 0.3) <= 1e-6
    # identical to the reference solve on the same instance (bitwise order)
    C = np.array([0.0, 1.0, 1.0, 0.0])  # column-major [[0,1],[1,0]]
    want = ref.solve(C, np.array([0.7, 0.3]), np.array([0.4, 0.6]), 2, 2,
                     default_config(tol_primal=1e-7, tol_dual=1e-7, tol_gap=1e-7))
    assert out["iterations"] == want.iterations
    assert out["objective"] == want.report["objective"]
    assert out["x00"] == want.plan[0] and out["x11"] == want.plan[3]
    # residual_report of (plan, cert) through the header: exact order = the report
    assert lines[1]["report_objective"] == out["objective"]
    assert lines[1]["sinkhorn_status"] == "converged"
    assert abs(lines[1]["sinkhorn_objective"] - 0.3) < 0.07  # test_reference.cpp:231-232
    assert lines[2]["error"].startswith("marginal_not_simplex: ")


def test_cpp_dropin_api():
    s = _summary(subprocess.run([_exe("dropin_api")], capture_output=True, text=True,
                                timeout=300))
    assert s["test_cases"] == 6 and s["failed_cases"] == 0, s


def test_reference_test_fused_unchanged():
    """proj/tests/test_fused.cpp (all 12 cases) against the drop-in."""
    s = _summary(subprocess.run([_exe("ref_test_fused")], capture_output=True, text=True,
                                timeout=300))
    assert s["test_cases"] == 12 and s["failed_cases"] == 0, s
