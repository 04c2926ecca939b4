import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: full-size parity (seconds to minutes)")


@pytest.fixture(scope="session")
def port():
    import oracle
    if not os.path.exists(oracle.PORT_SO):
        oracle.build()
    return oracle.Port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.ref_available():
        try:
            oracle.build()
        except Exception:
            pass
    if not oracle.ref_available():
        pytest.skip("reference shim (oracle/_ref/libsfref.so) not built here")
    return oracle.Ref()


@pytest.fixture(scope="session")
def ctx():
    import paper_2403_05802_b200 as sfg
    return sfg.Context(0)
