import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libvqcs_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def dev():
    import paper_2406_19212_b200 as vqb
    return vqb.device()


@pytest.fixture(scope="session")
def ref():
    """The strongest CPU checker: the reference library compiled from
    /root/reference (oracle/_ref), else the restatement."""
    import oracle
    return oracle.checker()


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.restatement()
