import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running full-size case")


@pytest.fixture(scope="session")
def oracle_libs():
    """(reference, restatement) — building them here if needed (gcc only)."""
    import oracle

    if not os.path.exists(oracle.ORC_SO) or (
            not os.path.exists(oracle.REF_SO) and os.path.isdir("/root/reference/proj/src")):
        oracle.build()
    ref = oracle.ref() if os.path.exists(oracle.REF_SO) else None
    return ref, oracle.orc()


@pytest.fixture(scope="session")
def built_lib():
    from paper_2604_16883_b200 import build

    return build.build_library()
