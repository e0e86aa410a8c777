import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity campaign")


def _ensure_oracle():
    lib = os.path.join(ROOT, "oracle", "_build", "libfmp_oracle.so")
    src = os.path.join(ROOT, "oracle", "fmp_oracle.c")
    if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)


@pytest.fixture(scope="session")
def oracle():
    """The C restatement (always buildable here and on the GPU box)."""
    _ensure_oracle()
    from oracle import Oracle
    return Oracle("restatement")


@pytest.fixture(scope="session")
def reference():
    """The reference library compiled from /root/reference (oracle/_ref)."""
    from oracle import PATHS, Oracle
    if not os.path.exists(PATHS["reference"]):
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return Oracle("reference")


@pytest.fixture(scope="session")
def fmp():
    import paper_1205_4139_b200 as fmp
    return fmp
