import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long CPU test")


@pytest.fixture(scope="session")
def root():
    return ROOT


@pytest.fixture(scope="session")
def code_c1():
    from synth.codes import make_met_code
    return make_met_code("r0.1", 2048)


@pytest.fixture(scope="session")
def code_c2():
    from synth.codes import make_met_code
    return make_met_code("r0.1", 65536)
