"""Shared fixtures. `-m gpu` tests need a B200 and call the CUDA path through the
C ABI; everything else runs on CPU (oracle vs reference, host logic, ABI exports)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: large-scene parity (seconds of CPU reference time)")


@pytest.fixture(scope="session")
def reference():
    from oracle import oracle
    if not oracle.reference_available():
        oracle.build()
    return oracle.Reference()


@pytest.fixture(scope="session")
def restatement():
    from oracle import oracle
    if not os.path.exists(oracle.RESTATEMENT_SO):
        oracle.build()
    return oracle.Restatement()


@pytest.fixture(scope="session")
def gpu():
    from paper_2603_18707_b200 import api
    r = api.Rasterizer(0)  # raises if no B200: GPU tests must not pass on a fallback
    yield r
    r.close()
