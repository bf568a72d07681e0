import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

TEAPOT = os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def teapot_path():
    return TEAPOT


@pytest.fixture(scope="session")
def oracle_teapot():
    from oracle import oracle
    return oracle.OracleModel.load(TEAPOT)
