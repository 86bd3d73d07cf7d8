"""bench.py's reference arm (CPU, no GPU needed): one JSON line with the
contract's keys and a positive rate, on a reduced size."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    ref = os.path.join(ROOT, "oracle", "_ref", "libdrotref.so")
    orc = os.path.join(ROOT, "oracle", "_ref", "liborc.so")
    if not (os.path.exists(ref) or os.path.exists(orc)):
        pytest.skip("oracle not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "20", "--warmup", "3", "--size", "1500"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert k in line, k
    assert line["value"] > 0 and line["steps"] == 20 and line["warmup"] == 3
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0
