import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libgconn.so)")
    config.addinivalue_line("markers", "slow: large inputs")


@pytest.fixture(scope="session")
def golden():
    from golden_data import Golden
    return Golden()
