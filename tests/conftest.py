import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built_host_libs():
    """Build the host-side libraries (datagen, oracle) once if missing."""
    need = [os.path.join(ROOT, "datagen", "libsivfgen.so"), os.path.join(ROOT, "oracle", "libsivf_oracle.so")]
    if not all(os.path.exists(p) for p in need):
        import subprocess

        subprocess.check_call(["make", "-C", ROOT, "datagen", "oracle"])
    yield
