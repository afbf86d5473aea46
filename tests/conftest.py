import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and liblabelprop_cuda.so")


def partition_matches(assignment, cliques: int, size: int) -> bool:
    """Exactly one community per clique (same predicate as the reference's
    tests/conftest.py:18-22)."""
    want = np.repeat(np.arange(cliques), size)
    pairs = set(zip(np.asarray(assignment).tolist(), want.tolist()))
    return len(pairs) == cliques and len(set(np.asarray(assignment).tolist())) == cliques


def load_graph(z, name):
    from paper_2301_09125_b200.graph import Graph

    off = np.asarray(z[f"{name}/offsets"], dtype=np.int64)
    nbr = np.asarray(z[f"{name}/neighbors"], dtype=np.int64)
    w = np.asarray(z[f"{name}/weights"], dtype=np.float64)
    for a in (off, nbr, w):
        a.setflags(write=False)
    return Graph(off.size - 1, nbr.size, off, nbr, w, float(z[f"{name}/total_weight"]))


@pytest.fixture(scope="session")
def golden_rak():
    return np.load(os.path.join(GOLDEN, "rak.npz"))


@pytest.fixture(scope="session")
def golden_copra():
    return np.load(os.path.join(GOLDEN, "copra.npz"))


@pytest.fixture(scope="session")
def golden_slpa():
    return np.load(os.path.join(GOLDEN, "slpa.npz"))


@pytest.fixture(scope="session")
def golden_prng():
    return np.load(os.path.join(GOLDEN, "prng.npz"))


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.lib()
    return O


@pytest.fixture(scope="session")
def gpu():
    """Skip unless a GPU and the CUDA library are present (gpu-marked tests
    only; the product path itself never falls back)."""
    from paper_2301_09125_b200 import _lib

    _lib.lib()
    if _lib.device_count() < 1:
        pytest.skip("no CUDA device")
    return _lib
