import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as o
    if not os.path.exists(o.PORT_SO):
        o.build(reference=False)
    return o.port()


@pytest.fixture(scope="session")
def reference():
    from oracle import oracle as o
    if not os.path.exists(o.REF_SO):
        if os.path.isdir(o.REFERENCE_SRC):
            o.build(reference=True)
        else:
            pytest.skip("oracle/_ref/libtsgm_ref.so not built and reference sources absent")
    return o.reference()
