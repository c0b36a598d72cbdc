import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def refbridge():
    from oracle import refbridge as rb
    if not rb.available():
        pytest.skip("oracle/_ref not built (no /root/reference here and no prebuilt copy)")
    return rb


@pytest.fixture(scope="session")
def rt():
    from paper_2601_09258_b200 import runtime
    return runtime


@pytest.fixture(scope="session")
def analyzer(rt):
    an = rt.Analyzer()
    yield an
    an.close()
