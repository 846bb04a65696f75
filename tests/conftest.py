import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running exhaustive check")


def _ensure_oracle():
    port = os.path.join(ROOT, "oracle", "libcqoracle.so")
    ref = os.path.join(ROOT, "oracle", "_ref", "libcqref.so")
    if not os.path.exists(port):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "port"], check=True,
                       capture_output=True)
    if not os.path.exists(ref) and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref", "-j8"], check=True,
                       capture_output=True)


_ensure_oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libcqref.so not built (needs /root/reference)")
    return Ref()

