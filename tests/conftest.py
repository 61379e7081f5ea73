import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "ref: needs the compiled reference (oracle/_ref)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle, build_oracle

    build_oracle(with_ref=False)
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.pyoracle import REF_SO, Reference

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (reference sources absent on this host)")
    return Reference()
