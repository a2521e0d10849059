import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / the driver's GPU tier)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import LIBS, REF_SRC, Oracle, build_oracles
    if not os.path.exists(LIBS["ref"]):
        if not os.path.isdir(REF_SRC):
            pytest.skip("reference build (oracle/_ref) not available on this machine")
        build_oracles(("ref",))
    return Oracle("ref")
