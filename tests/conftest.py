import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu on the GPU box")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference scheduler (oracle/_ref).  Skips when it was not built."""
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref/libmsref.so not built (needs /root/reference at build time)")
    return R


@pytest.fixture(scope="session")
def ms():
    from paper_2601_04071_b200 import microslice as M
    return M
