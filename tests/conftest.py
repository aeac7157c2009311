import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the native artefacts once (make is incremental)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", ROOT, "gen/libgwtfgen.so", "oracle/liboracle.so"], check=True)
    yield
