import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running parity run")
    # The CPU oracles are test infrastructure: build the plain-C restatement
    # (and, where /root/reference exists, the reference shim) if missing.
    if not os.path.exists(os.path.join(ROOT, "oracle", "build", "liborc.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=False)


@pytest.fixture(scope="session")
def ref():
    from pyoracle import Oracle
    return Oracle("ref")


@pytest.fixture(scope="session")
def orc():
    from pyoracle import Oracle
    return Oracle("orc")


@pytest.fixture(scope="session")
def drot():
    import paper_2110_11738_b200 as d
    return d
