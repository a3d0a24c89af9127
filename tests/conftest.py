"""Shared fixtures.  `gpu` tests need a B200 (run with -m gpu on the GPU box);
everything else runs on the CPU here."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libcpdb.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def port():
    from oracle.pyoracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def ctx():
    import paper_2503_18759_b200 as cpd
    return cpd.default_context()
