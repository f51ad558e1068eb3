import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")


def have_ref():
    from oracle.refcore import REF_SO
    return os.path.exists(REF_SO)


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import port
    return port.lib()


@pytest.fixture(scope="session")
def ctx():
    from paper_2412_10084_b200 import api
    c = api.Context(0)
    yield c
    c.close()


def pytest_collection_modifyitems(config, items):
    # GPU tests need the built product library; fail loudly (no fallback) if
    # it is missing rather than skipping silently.
    pass
