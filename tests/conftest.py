import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session", autouse=True)
def _built_libraries():
    """Build the checker (oracle) and, where nvcc exists, libhcg.so in-tree.

    On the GPU box the .so files arrive prebuilt with the snapshot; rebuilding
    is a no-op there unless sources changed."""
    oracle_dir = os.path.join(ROOT, "oracle")
    if not os.path.exists(os.path.join(oracle_dir, "liboracle.so")):
        subprocess.run(["make", "-s", "-C", oracle_dir], check=True)
    from paper_1209_0410_b200 import _build
    if os.path.exists("/usr/local/cuda/bin/nvcc"):
        _build.build()
    yield
