import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running (full-size shapes)")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle

    return oracle.lib()


@pytest.fixture(scope="session")
def cascade():
    """The product library; on a GPU box it must load (no fallback)."""
    import paper_2506_20675_b200 as pkg

    pkg.lib()
    return pkg
