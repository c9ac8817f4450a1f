import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE config sizes)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.pyoracle import Reference

    try:
        return Reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built (reference tree absent)")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def dev():
    """The product's ctypes view; fails loudly (no CPU fallback) when no GPU is usable."""
    import paper_2308_02856_b200 as P

    assert P.device_count() > 0, "no sm_100 device visible to libssbh_cuda.so"
    return P


def words(hexlist):
    return np.array([int(h, 16) for h in hexlist], dtype=np.uint64)
