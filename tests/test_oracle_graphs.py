"""The oracle's independent benchmark-graph builders (oracle/graphs.py, used
by bench.py's reference arm so that it never loads the product library)
produce exactly the product's graphs (paper_2301_09125_b200.synth: native
host builders here, GPU builders on a device box)."""

import numpy as np
import pytest

from oracle import graphs as OG
from paper_2301_09125_b200 import synth


def _same(a, b):
    return (a.vertex_count == b.vertex_count and a.edge_count == b.edge_count
            and np.array_equal(a.offsets, b.offsets) and np.array_equal(a.neighbors, b.neighbors)
            and np.array_equal(a.weights, b.weights) and a.total_weight == b.total_weight)


@pytest.mark.parametrize("scale,seed", [(10, 1), (13, 4)])
def test_rmat(scale, seed):
    assert _same(OG.rmat(scale, seed=seed), synth.rmat(scale, seed=seed))


def test_rmat_weighted():
    assert _same(OG.rmat(12, seed=2, weighted=True), synth.rmat(12, seed=2, weighted=True))


def test_planted():
    assert _same(OG.planted_partition(6000, 60, seed=3), synth.planted_partition(6000, 60, seed=3))


def test_grid():
    assert _same(OG.road_grid(96, seed=2), synth.road_grid(96, seed=2))


def test_csr_canonical_form():
    """Duplicates merged (either direction), generated self-loops dropped,
    one self-loop per vertex, rows ascending."""
    g = OG.csr_undirected(4, [0, 1, 2, 2, 3], [1, 0, 2, 3, 2])
    assert g.offsets.tolist() == [0, 2, 4, 6, 8]
    assert g.neighbors.tolist() == [0, 1, 0, 1, 2, 3, 2, 3]
