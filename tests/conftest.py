"""Shared test configuration.

Markers: `gpu` tests need a B200 (run on the GPU box with `pytest -m gpu`); everything
else runs on CPU. The CUDA library and the Python module are built in-tree by
`__graft_entry__.build()`; tests never rebuild the product.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    import oracle_lib

    oracle_lib.lib()
    return oracle_lib


@pytest.fixture(scope="session")
def plg():
    import paper_2403_03772_b200 as m

    return m


@pytest.fixture(scope="session")
def engine(plg):
    return plg.Engine(0)


def random_matrix(rng: np.random.Generator, d: int, m: int) -> np.ndarray:
    """test_ordering.cpp:19-25: uniform(-1, 1) entries, column-major."""
    return np.asfortranarray(rng.uniform(-1.0, 1.0, size=(m, d)))


def two_level_data(plg, seed: int, d: int, m: int) -> np.ndarray:
    """test_ordering.cpp:48-54 / acceptance.cpp:39-50: gen_two_level_dag + sample_lingam."""
    dag = plg.gen_two_level_dag(d, seed=seed)
    return plg.sample_lingam(dag, m, seed=seed)
