"""The drop-in headers as a SOURCE-compatible replacement of the reference's
(no GPU needed): the reference's own tests/test_fused.cpp and
test_matrix_rng.cpp compile unchanged against include/drot_b200 (plus the
doctest shim tests/cpp/doctest.h), and test_matrix_rng -- Matrix, CounterRng,
plan_tiles/TileRange, ThreadPool, all host-side -- passes here.  The GPU half
(test_fused, dropin_api) runs in tests/test_dropin_gpu.py."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
BIN = os.path.join(CPP, "_bin")
REF_TESTS = "/root/reference/proj/tests"


def _make():
    if not os.path.exists(os.path.join(ROOT, "paper_2110_11738_b200", "libdrotb200.so")):
        pytest.skip("libdrotb200.so not built")
    r = subprocess.run(["make", "-s", "-C", CPP], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_own_clients_compile():
    _make()
    for exe in ("dropin_solve", "dropin_api"):
        assert os.access(os.path.join(BIN, exe), os.X_OK), exe


@pytest.mark.skipif(not os.path.exists(REF_TESTS), reason="reference tree absent")
def test_reference_tests_compile_unchanged():
    _make()
    for exe in ("ref_test_fused", "ref_test_matrix_rng"):
        assert os.access(os.path.join(BIN, exe), os.X_OK), exe


@pytest.mark.skipif(not os.path.exists(REF_TESTS), reason="reference tree absent")
def test_reference_matrix_rng_tests_pass():
    _make()
    r = subprocess.run([os.path.join(BIN, "ref_test_matrix_rng")], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    summary = json.loads(r.stdout.strip().splitlines()[-1])
    assert summary["test_cases"] == 9 and summary["failed_cases"] == 0, summary
