"""CSR graph substrate (host side).

Mirrors the reference's ``labelprop.graph`` contract
(`pkg/src/labelprop/graph.py:34-50` for the ``Graph`` record, `:58-84`
``from_arcs``, `:254-306` ``preprocess``, `:320-344` ``degree_weights`` /
``check_symmetric``) so that a ``Graph`` built here is arc-for-arc equal to
the one the reference builds from the same arcs:

* rows sorted by neighbour id (the strict scan order, `graph.py:39-41`);
* duplicate arcs merged by weight sum (`graph.py:65-72`);
* ``preprocess``: symmetrised by max weight, optional unit weights, exactly
  one weight-1 self-loop per vertex (`graph.py:278-305`);
* ``total_weight`` counts self-loops twice (`graph.py:76`).

The text loaders of the reference (MatrixMarket / edge list) are outside
the hot-path scope and are not rebuilt.

``undirected_csr`` is the fast path the benchmark generators use: it
produces the same canonical graph as ``preprocess(from_arcs(...))`` for a
unit-weight undirected edge list, without the general lexsort.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Graph:
    """Immutable CSR graph (same fields as reference `graph.py:44-50`)."""

    vertex_count: int
    edge_count: int
    offsets: np.ndarray
    neighbors: np.ndarray
    weights: np.ndarray
    total_weight: float

    # The device copy (uploaded once, reused across runs) is cached by the
    # CUDA layer outside the object (_lib.device_graph), so a Graph stays
    # picklable and holds no GPU state.


def _ro(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


def from_arcs(vertex_count: int, u, v, w) -> Graph:
    """CSR from arc arrays; duplicate arcs merge by weight sum (ref `graph.py:58-84`)."""
    u = np.asarray(u, dtype=np.int64).ravel()
    v = np.asarray(v, dtype=np.int64).ravel()
    w = np.asarray(w, dtype=np.float64).ravel()
    n = int(vertex_count)
    if u.size:
        # sort arcs by (row, col); merge equal (row, col) runs
        order = np.lexsort((v, u))
        u, v, w = u[order], v[order], w[order]
        head = np.ones(u.size, dtype=bool)
        head[1:] = (u[1:] != u[:-1]) | (v[1:] != v[:-1])
        first = np.flatnonzero(head)
        w = np.add.reduceat(w, first)
        u = u[first]
        v = v[first]
    offsets = np.zeros(n + 1, dtype=np.int64)
    if u.size:
        offsets[1:] = np.cumsum(np.bincount(u, minlength=n))
    total = float(w.sum() + w[u == v].sum())
    return Graph(n, int(u.size), _ro(offsets), _ro(v.copy()), _ro(w.copy()), total)


def arc_rows(graph: Graph) -> np.ndarray:
    """Row (source vertex) of every stored arc."""
    return np.repeat(np.arange(graph.vertex_count, dtype=np.int64), np.diff(graph.offsets))


def preprocess(graph: Graph, unit_weights: bool = True, self_loops: bool = True) -> Graph:
    """Canonicalise for detection (ref `graph.py:254-306`).

    Off-diagonal arcs are symmetrised keeping the larger weight of the two
    directions; ``unit_weights`` forces every weight to 1; ``self_loops``
    replaces any existing loops with exactly one weight-1 loop per vertex.
    """
    n = graph.vertex_count
    if n == 0:
        return from_arcs(0, [], [], [])
    rows = arc_rows(graph)
    cols = np.asarray(graph.neighbors, dtype=np.int64)
    w = np.asarray(graph.weights, dtype=np.float64)
    loop = rows == cols
    a, b, ww = rows[~loop], cols[~loop], w[~loop]
    lo = np.minimum(a, b)
    hi = np.maximum(a, b)
    key = lo * n + hi
    srt = np.argsort(key, kind="stable")
    key, lo, hi, ww = key[srt], lo[srt], hi[srt], ww[srt]
    if key.size:
        head = np.ones(key.size, dtype=bool)
        head[1:] = key[1:] != key[:-1]
        first = np.flatnonzero(head)
        ww = np.maximum.reduceat(ww, first)
        lo, hi = lo[first], hi[first]
    if unit_weights:
        ww = np.ones_like(ww)
    if self_loops:
        lu = np.arange(n, dtype=np.int64)
        lw = np.ones(n, dtype=np.float64)
    else:
        lu = rows[loop]
        lw = np.ones(lu.size, dtype=np.float64) if unit_weights else w[loop]
    uu = np.concatenate([lo, hi, lu])
    vv = np.concatenate([hi, lo, lu])
    return from_arcs(n, uu, vv, np.concatenate([ww, ww, lw]))


def undirected_csr(n: int, u, v, weights=None) -> Graph:
    """Canonical preprocessed graph from an undirected edge list.

    Equivalent to ``preprocess(from_arcs(n, u, v, 1), unit_weights=True)``
    (with ``weights``: the same graph carrying per-edge weights, max over
    duplicate pairs).  Unit-weight lists go through the native builder
    (``lp_csr_build_undirected``, OpenMP); weighted ones through numpy.
    """
    if weights is None:
        from . import _lib

        u = np.ascontiguousarray(u, dtype=np.int64).ravel()
        v = np.ascontiguousarray(v, dtype=np.int64).ravel()
        if u.shape != v.shape:
            raise ValueError("u and v must have equal length")
        offsets = np.empty(n + 1, dtype=np.int64)
        nbr = np.empty(2 * u.size + n, dtype=np.int64)
        m = C.c_int64(0)
        _lib.check(_lib.lib().lp_csr_build_undirected(n, u.size, u, v, offsets, nbr, C.byref(m)))
        nbr = nbr[: m.value].copy()
        wts = np.ones(m.value, dtype=np.float64)
        total = float(m.value + n)
        return Graph(n, int(m.value), _ro(offsets), _ro(nbr), _ro(wts), total)
    return undirected_csr_numpy(n, u, v, weights)


def undirected_csr_numpy(n: int, u, v, weights=None) -> Graph:
    """Canonical preprocessed graph from an undirected edge list, fast.

    Equivalent to ``preprocess(from_arcs(n, u, v, 1), unit_weights=True)``
    (and, when ``weights`` is given per input edge, to the same graph with
    those weights applied symmetrically, max over duplicates): generated
    self-loops are dropped, duplicate pairs collapse, both directions are
    emitted, and every vertex gets one weight-1 self-loop.  Row ``r`` is
    laid out as ``[reverse arcs (col < r) sorted] + [r] + [forward arcs
    (col > r) sorted]`` which is exactly ascending neighbour order, so only
    two sorts of |E| keys are needed.
    """
    u = np.asarray(u, dtype=np.int64).ravel()
    v = np.asarray(v, dtype=np.int64).ravel()
    keep = u != v
    lo = np.minimum(u[keep], v[keep])
    hi = np.maximum(u[keep], v[keep])
    key = lo * n + hi
    if weights is None:
        key = np.unique(key)
        fw = None
    else:
        w = np.asarray(weights, dtype=np.float64).ravel()[keep]
        srt = np.argsort(key, kind="stable")
        key, w = key[srt], w[srt]
        head = np.ones(key.size, dtype=bool)
        head[1:] = key[1:] != key[:-1]
        first = np.flatnonzero(head)
        fw = np.maximum.reduceat(w, first) if key.size else w
        key = key[first]
    lo = key // n
    hi = key - lo * n
    # reverse arcs hi -> lo, sorted by (hi, lo)
    rkey = hi * n + lo
    rsrt = np.argsort(rkey, kind="stable")
    r_row = hi[rsrt]
    r_col = lo[rsrt]
    fcnt = np.bincount(lo, minlength=n)
    rcnt = np.bincount(hi, minlength=n)
    deg = fcnt + rcnt + 1
    offsets = np.zeros(n + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(deg)
    m = int(offsets[-1])
    nbr = np.empty(m, dtype=np.int64)
    wts = np.ones(m, dtype=np.float64)
    # reverse block of row r starts at offsets[r]
    rstart = np.zeros(n + 1, dtype=np.int64)
    rstart[1:] = np.cumsum(rcnt)
    r_pos = offsets[r_row] + (np.arange(r_row.size, dtype=np.int64) - rstart[r_row])
    nbr[r_pos] = r_col
    # self loop
    loop_pos = offsets[:-1] + rcnt
    nbr[loop_pos] = np.arange(n, dtype=np.int64)
    # forward block (already sorted by (lo, hi))
    fstart = np.zeros(n + 1, dtype=np.int64)
    fstart[1:] = np.cumsum(fcnt)
    f_pos = loop_pos[lo] + 1 + (np.arange(lo.size, dtype=np.int64) - fstart[lo])
    nbr[f_pos] = hi
    if fw is not None:
        wts[f_pos] = fw
        wts[r_pos] = fw[rsrt]
    total = float(wts.sum() + n)  # self loops (weight 1) count twice
    return Graph(n, m, _ro(offsets), _ro(nbr), _ro(wts), total)


def degree_weight(graph: Graph, vertex: int) -> float:
    """Weighted degree of one vertex, self-loop twice (ref `graph.py:309-317`)."""
    n = graph.vertex_count
    if not 0 <= vertex < n:
        raise ValueError(f"vertex {vertex} out of range [0, {n})")
    lo, hi = int(graph.offsets[vertex]), int(graph.offsets[vertex + 1])
    row = graph.neighbors[lo:hi]
    wts = graph.weights[lo:hi]
    return float(wts.sum() + wts[row == vertex].sum())


def degree_weights(graph: Graph) -> np.ndarray:
    """Weighted degree of every vertex, self-loops twice (ref `graph.py:320-327`)."""
    rows = arc_rows(graph)
    w = np.asarray(graph.weights, dtype=np.float64)
    deg = np.bincount(rows, weights=w, minlength=graph.vertex_count)
    loop = rows == graph.neighbors
    deg += np.bincount(rows[loop], weights=w[loop], minlength=graph.vertex_count)
    return deg


def check_symmetric(graph: Graph) -> None:
    """Raise ``ValueError`` unless every arc has its equal-weight reverse.

    Same contract and message as ref `graph.py:330-344`.
    """
    n = graph.vertex_count
    if n == 0:
        return
    rows = arc_rows(graph)
    cols = np.asarray(graph.neighbors, dtype=np.int64)
    fwd = rows * n + cols
    rev = cols * n + rows
    o1 = np.argsort(fwd, kind="stable")
    o2 = np.argsort(rev, kind="stable")
    if not np.array_equal(fwd[o1], rev[o2]) or not np.allclose(
        graph.weights[o1], graph.weights[o2]
    ):
        raise ValueError("graph is not symmetric; run preprocess() before detecting")


def graphs_equal(a: Graph, b: Graph) -> bool:
    """Arc-for-arc equality."""
    return (
        a.vertex_count == b.vertex_count
        and a.edge_count == b.edge_count
        and np.array_equal(a.offsets, b.offsets)
        and np.array_equal(a.neighbors, b.neighbors)
        and np.array_equal(a.weights, b.weights)
    )
