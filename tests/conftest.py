import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: full-size configuration (minutes)")


@pytest.fixture(scope="session")
def O():
    import oracle

    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def sph():
    import paper_2408_04440_b200 as m

    return m


@pytest.fixture(scope="session")
def G():
    """Golden vectors generated from the reference's own sources (tools/make_golden.py)."""
    import numpy as np

    return dict(np.load(os.path.join(ROOT, "tests", "golden", "ref_vectors.npz")))
