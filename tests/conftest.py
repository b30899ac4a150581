import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running (large n)")


@pytest.fixture(scope="session")
def ctx():
    """A device context; GPU tests fail loudly (no fallback) if it cannot be made."""
    from paper_1706_00773_b200 import capi

    return capi.default_context(0)


@pytest.fixture(scope="session")
def port():
    import oracle.port as p

    p.lib()
    return p
