import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "ref: needs oracle/_ref (reference compiled in place)")


@pytest.fixture(scope="session")
def oracle():
    from oracle_bind import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_bind import Ref

    if not Ref.available():
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    return Ref()


@pytest.fixture(scope="session")
def L():
    from paper_2603_23891_b200 import lodgs

    return lodgs


@pytest.fixture(scope="session")
def gpu(L):
    n = L.device_count()
    if n < 1:
        pytest.fail("no CUDA device visible: the -m gpu tests must run on the B200 box")
    return 0
