"""The reference-style C++ client (tests/cpp/dropin_solve.cpp) built against
the drop-in header runs on the GPU and reproduces the SPEC example."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_runs(tmp_path, ref):
    import numpy as np
    from pyoracle import default_config
    exe = tmp_path / "dropin"
    lib_dir = os.path.join(ROOT, "paper_2110_11738_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_solve.cpp"), "-o", str(exe),
                    "-L", lib_dir, "-ldrotb200", f"-Wl,-rpath,{lib_dir}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
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
