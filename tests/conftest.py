import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def oracle_lib():
    import helpers as H
    if not os.path.exists(H.ORACLE_SO):
        if os.path.isdir("/root/reference/proj"):
            H.build_oracle()
        else:
            pytest.skip("oracle/_ref/liboracle.so not built and /root/reference absent")
    return H.oracle()


@pytest.fixture(scope="session")
def harness_lib():
    import helpers as H
    return H.harness()
