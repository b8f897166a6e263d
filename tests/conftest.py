import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def oracle_port():
    from oracle import oracle as O
    if not os.path.exists(O.PORT_LIB):
        O.build()
    return O.Oracle("port")


@pytest.fixture(scope="session")
def oracle_ref():
    from oracle import oracle as O
    if not os.path.exists(O.REF_LIB):
        pytest.skip("oracle/_ref (reference headers built against the Eigen shim) not built")
    return O.Oracle("reference")
