"""Shared fixtures.  `-m gpu` tests need a B200 and the in-tree libsgwg.so;
`-m "not gpu"` tests run on CPU (oracle pins, ABI surface, host logic, gloo)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and libsgwg.so")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ctx():
    from paper_2007_10196_b200 import sgwg
    c = sgwg.Context(0, arith="exact")
    yield c


@pytest.fixture(scope="session")
def ctx_fast():
    from paper_2007_10196_b200 import sgwg
    c = sgwg.Context(0, arith="fast")
    yield c
