import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden(name):
    return os.path.join(ROOT, "tests", "golden", name)


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


def pytest_sessionfinish(session, exitstatus):
    """Under the device-check build (PGA_LIB=.../libpga_check.so, see
    tests/test_gpu_checks.py) the whole GPU suite must leave the device
    invariant counters at zero."""
    lib = os.environ.get("PGA_LIB", "")
    if not lib.endswith("libpga_check.so") or exitstatus != 0:
        return
    import paper_1403_4099_b200 as pga
    v = pga.pga_debug_violations()
    print("\ndevice invariant violations over the session: %d" % v)
    if v:
        session.exitstatus = 1
