import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long CPU oracle runs")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as O
    if not O.available("orc"):
        O.build()
    return O.Oracle("orc")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O
    if not O.available("ref"):
        pytest.skip("reference oracle (oracle/_ref) not built here")
    return O.Oracle("ref")


def spec_text(name):
    return open(os.path.join(ROOT, "configs", name + ".json")).read()
