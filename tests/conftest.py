import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref():
    """The reference compiled from /root/reference (oracle/_ref); skip if it was not built."""
    import oracle

    if not os.path.exists(oracle.REF_SO):
        if os.path.isdir(oracle.REFERENCE_ROOT):
            oracle.build(ref=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return oracle.ref()


@pytest.fixture(scope="session")
def port():
    import oracle

    if not os.path.exists(oracle.PORT_SO):
        oracle.build(ref=False)
    return oracle.port()


@pytest.fixture(scope="session")
def golden():
    import json

    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)
