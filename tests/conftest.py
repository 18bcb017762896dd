import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu on the GPU box")
    config.addinivalue_line("markers", "slow: long-running (large R-MAT sizes)")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


@pytest.fixture(scope="session")
def ctx():
    from paper_2504_06408_b200 import default_context
    return default_context(0)


@pytest.fixture
def bins_ctx(ctx):
    """The context with the per-bin accumulators forced (no bitmap-rank path):
    tests that target a specific bin (hash, dense panels, bit-rank) use it."""
    ctx.set_pipeline(ctx.PIPE_BINS)
    try:
        yield ctx
    finally:
        ctx.set_pipeline(ctx.PIPE_AUTO)
