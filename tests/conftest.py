import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size configuration (seconds to minutes)")


@pytest.fixture(scope="session", autouse=True)
def _build_oracle():
    import oracle
    oracle.build()


@pytest.fixture(scope="session", autouse=True)
def _build_library():
    from paper_2009_10247_b200 import build
    build.build()


@pytest.fixture(params=["compact", "batched"])
def stable_kernel(request, monkeypatch):
    """lp_stable_models on both device paths: the compact kernel (live sub-program in shared
    memory, the default when it fits) and the batched persistent kernel
    (LP_NO_COMPACT_STABLE, read by lp_load)."""
    if request.param == "batched":
        monkeypatch.setenv("LP_NO_COMPACT_STABLE", "1")
    return request.param
