import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    return O


@pytest.fixture(scope="session")
def restatement(oracle):
    return oracle.restatement()


@pytest.fixture(scope="session")
def reference(oracle):
    ref = oracle.reference()
    if ref is None:
        pytest.skip("oracle/_ref/libamqft_ref.so not built (reference sources absent)")
    return ref


@pytest.fixture
def no_tile(monkeypatch):
    """Plans created under this fixture skip the in-shared-memory four-step
    (path 6, tile_kernel.cuh) so the tests of the kernels it displaced as the
    default for fp32 CDFT N = 256-4096 (fused, cooperative, four-step) keep
    exercising them: the library reads AMQFT_AB_TILE at plan creation."""
    monkeypatch.setenv("AMQFT_AB_TILE", "none")
