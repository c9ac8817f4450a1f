import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_addoption(parser):
    parser.addoption(
        "--ssbh-override", action="append", default=[], metavar="KEY=VALUE",
        help="plan-construction override for the whole run (ssbh_set_plan_overrides), e.g. "
             "engine=1 (LOP3 engine), shared_tiled=1, split_levels=0; repeatable")


def _session_overrides(config):
    out = {}
    for kv in config.getoption("--ssbh-override"):
        key, val = kv.split("=", 1)
        out[key] = int(val)
    return out


@pytest.fixture(autouse=True)
def _plan_overrides(request):
    """Every test starts from the session's plan overrides (defaults unless --ssbh-override)
    and any override a test sets is undone afterwards."""
    base = _session_overrides(request.config)
    try:
        import paper_2308_02856_b200 as P
    except ImportError:
        yield
        return
    P.set_overrides(**base)
    yield
    P.set_overrides(**base)


@pytest.fixture
def ovr(request):
    """ovr(split_levels=3, ...): plan overrides for the rest of this test, merged over the
    session's; reset by _plan_overrides afterwards."""
    import paper_2308_02856_b200 as P

    base = _session_overrides(request.config)

    def apply(**kw):
        vals = dict(base)
        vals.update(kw)
        P.set_overrides(**vals)
        return P.get_overrides()

    return apply


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
