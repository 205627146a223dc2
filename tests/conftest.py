import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libihom_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def orc():
    import oracle
    if not os.path.exists(oracle.LIB_PATH):
        oracle.build()
    return oracle


@pytest.fixture(scope="session")
def ih():
    import paper_2301_08911_b200 as ih
    if not os.path.exists(ih.LIB_PATH):
        ih.build()
    return ih


def mt_uniform(n, seed, lo, hi):
    """Seeded uniform field (tests/oracles.cpp:208-222 uses mt19937_64; numpy's PCG64 stands in)."""
    return np.random.default_rng(seed).uniform(lo, hi, n)
