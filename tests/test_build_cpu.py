"""Build-level guards (no GPU): the sm_100a cubin of the hot kernels keeps the
resource budget its occupancy design assumes.

K1 (pass_kernel_async) is designed for 3 resident 128-thread CTAs per SM
(64 KB of cp.async ring + staging each): that needs <= 170 registers per
thread (65536 / 384).  A build at 199-210 registers (2 CTAs per SM) measured
373.8 vs 324.1 us per fp64 sweep at 10k^2 (r1 tuning) -- this test catches
that regression without a GPU.  No hot kernel may spill to local memory.
"""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2110_11738_b200", "libdrotb200.so")


def _res_usage():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB) or not os.path.exists(exe):
        pytest.skip("library or cuobjdump missing")
    out = subprocess.run([exe, "-res-usage", LIB], capture_output=True, text=True).stdout
    res = {}
    fn = None
    for line in out.splitlines():
        m = re.search(r"Function ([^ :]+)", line)
        if m:
            fn = m.group(1)
            continue
        if fn and "REG:" in line:
            reg = int(re.search(r"REG:(\d+)", line).group(1))
            local = int(re.search(r"LOCAL:(\d+)", line).group(1))
            res[fn] = (reg, local)
            fn = None
    return res


def test_k1_register_budget():
    res = _res_usage()
    k1 = {f: v for f, v in res.items() if "pass_kernel_async" in f}
    assert k1, "pass_kernel_async not found in the cubin"
    for f, (reg, local) in k1.items():
        assert reg <= 170, (f, reg)
        assert local == 0, (f, local)


def test_hot_kernels_do_not_spill():
    res = _res_usage()
    for key in ("tail_kernel", "sk_sweep", "gaussian_cost_kernel"):
        ks = {f: v for f, v in res.items() if key in f}
        assert ks, key
        for f, (reg, local) in ks.items():
            assert local == 0, (f, local)
