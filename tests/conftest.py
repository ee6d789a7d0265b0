import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs only under gpurun / round-end GPU tier)")
    config.addinivalue_line("markers", "slow: longer CPU cases")


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ko():
    from oracle.oracle import Oracle, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "libkeep_oracle.so")):
        build()
    return Oracle("ko")


@pytest.fixture(scope="session")
def kr():
    from oracle.oracle import Oracle, available
    if not available("kr"):
        pytest.skip("reference shim oracle/_ref not built (no /root/reference here)")
    return Oracle("kr")
