"""Seeded graph generators and the brute-force modularity check.

Two groups:

* the reference's test fixtures (`pkg/src/labelprop/synth.py:40-165`):
  ``disjoint_cliques``, ``ring_of_cliques``, ``gnp``, ``star``, ``path``,
  ``gen_graph`` and ``brute_modularity``.  ``gnp`` consumes numpy's
  ``default_rng(seed)`` exactly as the reference's geometric gap-skipping
  sampler does (`synth.py:68-92`), so the same seed yields the same graph on
  both sides and parity tests compare like with like;
* the BASELINE.json benchmark graphs, which the reference does not ship
  (SURVEY.md §0 item 7): ``planted_partition`` (config 0 / SLPA config 4),
  ``rmat`` (configs 1 and 3) and ``road_grid`` (config 2).  All are seeded
  with ``numpy.random.default_rng(seed)`` and built through
  ``undirected_csr`` into the canonical preprocessed form (unit weights, one
  self-loop per vertex).  These stand in for the paper's SuiteSparse corpus
  (`PAPER.md:43-79`), which is not available.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes as C

import numpy as np

from .graph import Graph, from_arcs, preprocess, undirected_csr


@dataclass(frozen=True)
class SyntheticGraphSpec:
    """Recipe for a generated test graph (ref `synth.py:17-31`)."""

    kind: str
    n: int = 0
    p: float = 0.0
    cliques: int = 0
    clique_size: int = 0
    seed: int = 1


def _undirected(n, us, vs, unit_weights=True, self_loops=True) -> Graph:
    u = np.concatenate([np.asarray(a, dtype=np.int64) for a in us]) if us else np.zeros(0, np.int64)
    v = np.concatenate([np.asarray(a, dtype=np.int64) for a in vs]) if vs else np.zeros(0, np.int64)
    return preprocess(from_arcs(n, u, v, np.ones(u.size)), unit_weights=unit_weights,
                      self_loops=self_loops)


def _clique_pairs(first: int, size: int):
    a, b = np.triu_indices(size, k=1)
    return a.astype(np.int64) + first, b.astype(np.int64) + first


def disjoint_cliques(cliques: int, clique_size: int, **pre) -> Graph:
    """``cliques`` disconnected cliques of ``clique_size`` vertices."""
    pairs = [_clique_pairs(c * clique_size, clique_size) for c in range(cliques)]
    return _undirected(cliques * clique_size, [p[0] for p in pairs], [p[1] for p in pairs], **pre)


def ring_of_cliques(cliques: int, clique_size: int, **pre) -> Graph:
    """Cliques in a ring, clique c's last vertex bridged to clique c+1's first."""
    n = cliques * clique_size
    us, vs = [], []
    for c in range(cliques):
        a, b = _clique_pairs(c * clique_size, clique_size)
        us += [a, np.array([(c + 1) * clique_size - 1])]
        vs += [b, np.array([((c + 1) * clique_size) % n])]
    return _undirected(n, us, vs, **pre)


def gnp(n: int, p: float, seed: int = 1, **pre) -> Graph:
    """Erdos-Renyi G(n, p) by geometric gap skipping over the upper triangle.

    Draw-for-draw the sampler of ref `synth.py:68-92` (same batch size and
    ``default_rng`` calls), so equal seeds give equal graphs.
    """
    if not 0.0 <= p <= 1.0:
        raise ValueError("p must be in [0, 1]")
    if n < 2 or p == 0.0:
        return _undirected(max(n, 0), [], [])
    pairs = n * (n - 1) // 2
    rng = np.random.default_rng(seed)
    batch = max(int(pairs * p * 1.1) + 16, 1024)
    chunks = []
    last = -1
    while last < pairs - 1:
        idx = last + np.cumsum(rng.geometric(p, size=batch))
        chunks.append(idx[idx < pairs])
        if idx[-1] >= pairs:
            break
        last = int(idx[-1])
    lin = np.concatenate(chunks) if chunks else np.zeros(0, np.int64)
    starts = np.zeros(n, dtype=np.int64)
    np.cumsum(np.arange(n - 1, 0, -1), out=starts[1:])
    i = np.searchsorted(starts, lin, side="right") - 1
    j = lin - starts[i] + i + 1
    return _undirected(n, [i], [j], **pre)


def star(n: int, **pre) -> Graph:
    """Hub 0 joined to n-1 leaves."""
    if n < 2:
        return _undirected(max(n, 0), [], [])
    return _undirected(n, [np.zeros(n - 1, np.int64)], [np.arange(1, n, dtype=np.int64)], **pre)


def path(n: int, **pre) -> Graph:
    """Path 0 - 1 - ... - n-1."""
    if n < 2:
        return _undirected(max(n, 0), [], [])
    a = np.arange(n - 1, dtype=np.int64)
    return _undirected(n, [a], [a + 1], **pre)


def gen_graph(spec: SyntheticGraphSpec) -> Graph:
    """Build the graph a ``SyntheticGraphSpec`` describes (ref `synth.py:118-130`)."""
    kinds = {
        "disjoint-cliques": lambda s: disjoint_cliques(s.cliques, s.clique_size),
        "ring-of-cliques": lambda s: ring_of_cliques(s.cliques, s.clique_size),
        "random-gnp": lambda s: gnp(s.n, s.p, s.seed),
        "star": lambda s: star(s.n),
        "path": lambda s: path(s.n),
    }
    if spec.kind not in kinds:
        raise ValueError(f"unknown synthetic graph kind {spec.kind!r}")
    return kinds[spec.kind](spec)


def brute_modularity(graph: Graph, assignment) -> float:
    """O(V^2) modularity from the dense adjacency matrix (ref `synth.py:133-165`).

    Independent of the CSR scorer on purpose; limited to 256 vertices.
    """
    n = graph.vertex_count
    if n > 256:
        raise ValueError("brute_modularity is limited to 256 vertices")
    lab = np.asarray(assignment, dtype=np.int64)
    if lab.shape != (n,):
        raise ValueError("assignment length must equal vertex_count")
    if n == 0:
        return 0.0
    adj = np.zeros((n, n))
    for r in range(n):
        for e in range(int(graph.offsets[r]), int(graph.offsets[r + 1])):
            c = int(graph.neighbors[e])
            adj[r, c] += graph.weights[e] * (2.0 if c == r else 1.0)
    deg = adj.sum(axis=1)
    total = adj.sum()
    if total <= 0:
        return 0.0
    same = lab[:, None] == lab[None, :]
    return float(((adj - np.outer(deg, deg) / total) * same).sum() / total)


# --------------------------------------------------------------------------
# Benchmark generators (BASELINE.json configs; not part of the reference)
# --------------------------------------------------------------------------

def planted_partition(n: int = 100_000, communities: int = 1_000, intra: int = 16,
                      inter: int = 4, seed: int = 1) -> Graph:
    """Config 0 (and SLPA config 4 at n=1M): planted communities.

    Vertex ``v`` belongs to community ``v // (n / communities)``.  Each
    vertex draws ``intra`` partners uniformly from its own community (never
    itself) and ``inter`` partners uniformly from the whole graph.  The
    pairs are symmetrised, deduplicated and generated self-loops dropped;
    preprocessing then adds one unit self-loop per vertex.
    """
    if n % communities:
        raise ValueError("n must be a multiple of communities")
    size = n // communities
    rng = np.random.default_rng(seed)
    v = np.arange(n, dtype=np.int64)
    local = v % size
    r = rng.integers(0, size - 1, size=(n, intra), dtype=np.int64)
    r += r >= local[:, None]
    intra_dst = (v - local)[:, None] + r
    inter_dst = rng.integers(0, n, size=(n, inter), dtype=np.int64)
    src = np.repeat(v, intra + inter)
    dst = np.concatenate([intra_dst, inter_dst], axis=1).ravel()
    return undirected_csr(n, src, dst)


def rmat_edges(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
               c: float = 0.19, seed: int = 1):
    """Raw R-MAT edge list (native, ``lp_gen_rmat``): one quadrant draw per
    bit level from a counter RNG keyed by (seed, edge, level); no noise, no
    vertex-id scrambling (vertex 0 is the largest hub)."""
    from . import _lib

    m = edge_factor << scale
    src = np.empty(m, dtype=np.int64)
    dst = np.empty(m, dtype=np.int64)
    _lib.check(_lib.lib().lp_gen_rmat(scale, m, a, b, c, seed, src, dst))
    return src, dst


def _rmat_gpu(scale: int, edge_factor: int, seed: int):
    """The same graph built on the GPU (``lp_gen_rmat_csr``) when a device is
    present (LP_BUILD_GPU=0 forces the host builder); None otherwise."""
    import os

    from . import _lib
    from .graph import _ro

    if os.environ.get("LP_BUILD_GPU", "1") == "0" or scale < 12:
        return None
    try:
        if _lib.device_count() < 1:
            return None
    except Exception:
        return None
    n = 1 << scale
    m_pairs = edge_factor << scale
    offsets = np.empty(n + 1, dtype=np.int64)
    nbr = np.empty(2 * m_pairs + n, dtype=np.int64)
    m = C.c_int64(0)
    _lib.check(_lib.lib().lp_gen_rmat_csr(scale, m_pairs, 0.57, 0.19, 0.19, seed, -1, offsets, nbr, nbr.size,
                                          C.byref(m)))
    nbr = nbr[: m.value].copy()
    return Graph(n, int(m.value), _ro(offsets), _ro(nbr), _ro(np.ones(m.value, dtype=np.float64)), float(m.value + n))


def rmat(scale: int = 22, edge_factor: int = 16, seed: int = 1, weighted: bool = False) -> Graph:
    """Configs 1 / 3: symmetrised R-MAT, duplicates and self-loops dropped.

    ``weighted`` gives every undirected edge one float32 weight drawn
    uniformly from [1, 2) (both arc directions equal, so the graph stays
    symmetric); self-loops keep weight 1.
    """
    g = _rmat_gpu(scale, edge_factor, seed)
    if g is None:
        src, dst = rmat_edges(scale, edge_factor, seed=seed)
        g = undirected_csr(1 << scale, src, dst)
    if weighted:
        g = with_edge_weights(g, seed=seed + 1000)
    return g


def with_edge_weights(g: Graph, seed: int = 1, low: float = 1.0, high: float = 2.0) -> Graph:
    """Same graph, each undirected edge re-weighted by one float32 U[low, high).

    The weight is a function of the unordered pair so both arc directions
    agree; self-loops stay at 1.0.  Values are float32-representable so the
    float32 device copy and the float64 host copy hold the same numbers.
    """
    rows = np.repeat(np.arange(g.vertex_count, dtype=np.int64), np.diff(g.offsets))
    cols = np.asarray(g.neighbors, dtype=np.int64)
    lo = np.minimum(rows, cols).astype(np.uint64)
    hi = np.maximum(rows, cols).astype(np.uint64)
    # splitmix64 of the pair and the seed -> 24 random mantissa bits
    with np.errstate(over="ignore"):
        x = _splitmix(lo, hi, seed)
    frac = (x >> np.uint64(40)).astype(np.float64) / float(1 << 24)
    w = (np.float32(low) + np.float32(high - low) * frac.astype(np.float32)).astype(np.float32)
    w = w.astype(np.float64)
    w[rows == cols] = 1.0
    total = float(w.sum() + w[rows == cols].sum())
    w.setflags(write=False)
    return Graph(g.vertex_count, g.edge_count, g.offsets, g.neighbors, w, total)


def _splitmix(lo, hi, seed):
    x = lo * np.uint64(0x9E3779B97F4A7C15) ^ (hi + np.uint64(seed) * np.uint64(0xBF58476D1CE4E5B9))
    x ^= x >> np.uint64(30)
    x *= np.uint64(0xBF58476D1CE4E5B9)
    x ^= x >> np.uint64(27)
    x *= np.uint64(0x94D049BB133111EB)
    x ^= x >> np.uint64(31)
    return x


def road_grid(side: int = 4096, drop: float = 0.10, shortcuts: float = 0.02, seed: int = 1) -> Graph:
    """Config 2: ``side`` x ``side`` 4-neighbour grid, road-network-like.

    ``drop`` of the grid edges are deleted at random and diagonal shortcuts
    numbering ``shortcuts`` x (grid edge count) are added between random
    cells and one of their diagonal neighbours.
    """
    rng = np.random.default_rng(seed)
    ids = np.arange(side * side, dtype=np.int64).reshape(side, side)
    hu, hv = ids[:, :-1].ravel(), ids[:, 1:].ravel()
    vu, vv = ids[:-1, :].ravel(), ids[1:, :].ravel()
    u = np.concatenate([hu, vu])
    v = np.concatenate([hv, vv])
    keep = rng.random(u.size) >= drop
    grid_edges = u.size
    u, v = u[keep], v[keep]
    k = int(round(shortcuts * grid_edges))
    r = rng.integers(0, side - 1, size=k)
    c = rng.integers(0, side - 1, size=k)
    anti = rng.random(k) < 0.5
    su = np.where(anti, ids[r, c + 1], ids[r, c])
    sv = np.where(anti, ids[r + 1, c], ids[r + 1, c + 1])
    return undirected_csr(side * side, np.concatenate([u, su]), np.concatenate([v, sv]))
