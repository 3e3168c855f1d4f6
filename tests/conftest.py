import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) device; parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle (and, where the sources exist, the reference) once."""
    import oracle
    oracle.build(quiet=True)
    yield


@pytest.fixture(scope="session")
def gpu_available():
    from paper_2110_13368_b200 import device_count
    return device_count() > 0
