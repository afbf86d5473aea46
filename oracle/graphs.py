"""BASELINE.json benchmark graphs built without the product library.

TEST INFRASTRUCTURE ONLY (like the rest of ``oracle/``): bench.py's
reference arm builds its graph here so that the timed CPU path never maps
``liblabelprop_cuda.so``, and tests/test_oracle_graphs.py checks the
product's generators (``paper_2301_09125_b200.synth``, native and GPU
builders) against these arc for arc.

The recipes are the seeded stand-ins of DESIGN.md §5 for the paper's
SuiteSparse corpus (the reference ships no R-MAT / planted / grid
generator).  R-MAT pairs and the canonical CSR build
(the form of the reference's ``preprocess(from_arcs(...))``,
graph.py:58-84,254-306) are C (``or_gen_rmat_pairs``, ``or_csr_undirected``
in lp_oracle.c); planted and grid pairs are numpy ``default_rng`` draws.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import oracle as O


@dataclass(frozen=True)
class OGraph:
    """The CSR fields the oracle functions read (same names as the
    reference's ``Graph``, graph.py:44-50)."""

    vertex_count: int
    edge_count: int
    offsets: np.ndarray
    neighbors: np.ndarray
    weights: np.ndarray
    total_weight: float


def _lib():
    L = O.lib()
    if not getattr(L, "_graphs_bound", False):
        p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        L.or_gen_rmat_pairs.argtypes = [C.c_int32, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_uint64, p, p]
        L.or_gen_rmat_pairs.restype = C.c_int
        L.or_csr_undirected.argtypes = [C.c_int64, C.c_int64, p, p, p, p]
        L.or_csr_undirected.restype = C.c_int64
        L._graphs_bound = True
    return L


def csr_undirected(n: int, u, v) -> OGraph:
    u = np.ascontiguousarray(u, dtype=np.int64).ravel()
    v = np.ascontiguousarray(v, dtype=np.int64).ravel()
    off = np.empty(n + 1, dtype=np.int64)
    nbr = np.empty(2 * u.size + n, dtype=np.int64)
    m = _lib().or_csr_undirected(n, u.size, u, v, off, nbr)
    if m < 0:
        raise ValueError("bad pair list")
    nbr = nbr[:m].copy()
    return OGraph(n, int(m), off, nbr, np.ones(m, dtype=np.float64), float(m + n))


def rmat(scale: int = 22, edge_factor: int = 16, seed: int = 1, weighted: bool = False) -> OGraph:
    m = edge_factor << scale
    src = np.empty(m, dtype=np.int64)
    dst = np.empty(m, dtype=np.int64)
    if _lib().or_gen_rmat_pairs(scale, m, 0.57, 0.19, 0.19, seed, src, dst):
        raise ValueError("bad R-MAT arguments")
    g = csr_undirected(1 << scale, src, dst)
    del src, dst
    return with_edge_weights(g, seed=seed + 1000) if weighted else g


def planted_partition(n: int = 100_000, communities: int = 1_000, intra: int = 16, inter: int = 4,
                      seed: int = 1) -> OGraph:
    """Vertex v in community v // (n / communities); ``intra`` partners
    uniform in its community (not itself), ``inter`` uniform over all."""
    size = n // communities
    rng = np.random.default_rng(seed)
    v = np.arange(n, dtype=np.int64)
    local = v % size
    r = rng.integers(0, size - 1, size=(n, intra), dtype=np.int64)
    r = r + (r >= local[:, None])  # skip the vertex itself
    same = (v - local)[:, None] + r
    other = rng.integers(0, n, size=(n, inter), dtype=np.int64)
    src = np.repeat(v, intra + inter)
    dst = np.hstack([same, other]).reshape(-1)
    return csr_undirected(n, src, dst)


def road_grid(side: int = 4096, drop: float = 0.10, shortcuts: float = 0.02, seed: int = 1) -> OGraph:
    """side x side 4-neighbour grid, ``drop`` of the grid edges removed, and
    ``shortcuts`` x (grid edges) diagonal shortcuts between random cells."""
    rng = np.random.default_rng(seed)
    cell = np.arange(side * side, dtype=np.int64).reshape(side, side)
    u = np.concatenate([cell[:, :-1].reshape(-1), cell[:-1, :].reshape(-1)])
    v = np.concatenate([cell[:, 1:].reshape(-1), cell[1:, :].reshape(-1)])
    total = u.size
    kept = rng.random(total) >= drop
    u, v = u[kept], v[kept]
    k = int(round(shortcuts * total))
    r = rng.integers(0, side - 1, size=k)
    c = rng.integers(0, side - 1, size=k)
    anti = rng.random(k) < 0.5
    a = np.where(anti, cell[r, c + 1], cell[r, c])
    b = np.where(anti, cell[r + 1, c], cell[r + 1, c + 1])
    return csr_undirected(side * side, np.concatenate([u, a]), np.concatenate([v, b]))


def _mix64(x):
    x = x ^ (x >> np.uint64(30))
    x = x * np.uint64(0xBF58476D1CE4E5B9)
    x = x ^ (x >> np.uint64(27))
    x = x * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def with_edge_weights(g: OGraph, seed: int = 1, low: float = 1.0, high: float = 2.0) -> OGraph:
    """One float32 U[low, high) per unordered pair (splitmix of the pair and
    the seed, 24 mantissa bits), both arc directions equal; self-loops 1."""
    n = g.vertex_count
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(g.offsets))
    cols = g.neighbors
    lo = np.minimum(rows, cols).astype(np.uint64)
    hi = np.maximum(rows, cols).astype(np.uint64)
    with np.errstate(over="ignore"):
        x = _mix64(lo * np.uint64(0x9E3779B97F4A7C15) ^ (hi + np.uint64(seed) * np.uint64(0xBF58476D1CE4E5B9)))
    u24 = (x >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / (1 << 24))
    w = (np.float32(low) + np.float32(high - low) * u24).astype(np.float64)
    loops = rows == cols
    w[loops] = 1.0
    return OGraph(n, g.edge_count, g.offsets, g.neighbors, w, float(w.sum() + w[loops].sum()))


BENCH_GRAPHS = {
    "rmat22": lambda: rmat(22, seed=1),
    "rmat22w": lambda: rmat(22, seed=1, weighted=True),
    "planted": lambda: planted_partition(100_000, 1_000, seed=1),
    "grid": lambda: road_grid(4096, seed=1),
}
