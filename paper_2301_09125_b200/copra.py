"""COPRA (multi-label propagation with belonging coefficients) on the B200.

Drop-in for the reference's ``labelprop.copra`` (`pkg/src/labelprop/
copra.py`): ``CopraParams`` keeps the reference's fields, defaults and
validation (`copra.py:34-50`) plus defaulted ``batches`` / ``backend``;
``copra_detect`` keeps the signature and result contract
(`copra.py:292-297`); ``collect_and_threshold`` and ``best_label`` keep the
helper semantics (`copra.py:300-338`).

The sweeps (`copra.py:124-238`) run in one call into
``liblabelprop_cuda.so`` (``lp_copra_run``, kernels in
``csrc/lp_copra_kernels.cuh``).  Belongings are float64 and every
arithmetic step follows the reference's order, so label sets match the CPU
restatement bit for bit; ``batches=0`` is the reference's in-place
index-order sweep, ``1`` synchronous.  The only randomness -- the fallback
draw among tied maxima when no label reaches 1/k (`copra.py:72-93`) -- uses
the counter hash instead of the sequential xorshift stream.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import Graph, check_symmetric
from .prng import XorShift32, draw_bounded
from .quality import score
from .result import DetectionResult

CHUNK = 1024  # the reference's parallel work unit (copra.py:31); no CUDA counterpart


@dataclass(frozen=True)
class CopraParams:
    tolerance: float = 0.01
    max_labels: int = 8
    max_iterations: int = 100
    workers: int = 1
    seed: int = 1
    # --- additions (defaults keep the reference signature valid) ---
    batches: int = 0       # 0 = reference visit (in place, index order); 1 = synchronous
    backend: str = "cuda"

    def __post_init__(self):
        if not 0.0 < self.tolerance <= 1.0:
            raise ValueError("tolerance must be in (0, 1]")
        if self.max_labels < 1:
            raise ValueError("max_labels must be >= 1")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.batches < 0:
            raise ValueError("batches must be >= 0")
        if self.backend != "cuda":
            raise ValueError("only the 'cuda' backend exists (no CPU fallback)")


def _opts(params: CopraParams) -> _lib.CopraOpts:
    o = _lib.CopraOpts()
    o.tolerance = float(params.tolerance)
    o.max_labels = int(params.max_labels)
    o.max_iterations = int(params.max_iterations)
    o.batches = int(params.batches)
    o.seed = int(params.seed) & 0xFFFFFFFF
    return o


def copra_run(graph: Graph, params: CopraParams | None = None, *, want_sets: bool = True, profile: bool = False,
              device_graph: "_lib.DeviceGraph | None" = None):
    """One COPRA run on the GPU.

    Returns ``(best, iterations, labs, bels, sizes, stats, changed_per_sweep)``;
    ``labs``/``bels`` are ``(n, max_labels)`` rows sorted by label with
    entries past ``sizes[v]`` zero (None without ``want_sets``).
    """
    if params is None:
        params = CopraParams()
    n = graph.vertex_count
    L = params.max_labels
    if n == 0:
        z = np.zeros((0, L))
        return (np.zeros(0, dtype=np.int64), 0, z.astype(np.int64), z, np.zeros(0, dtype=np.int64), {},
                np.zeros(0, dtype=np.int64))
    dg = device_graph if device_graph is not None else _lib.device_graph(graph)
    opts = _opts(params)
    if profile:
        opts.flags |= _lib.RAK_PROFILE
    best = np.empty(n, dtype=np.int64)
    labs = np.empty((n, L), dtype=np.int64) if want_sets else None
    bels = np.empty((n, L), dtype=np.float64) if want_sets else None
    sizes = np.empty(n, dtype=np.int64) if want_sets else None
    changed = np.zeros(params.max_iterations, dtype=np.int64)
    stats = _lib.RunStats()
    _lib.check(_lib.lib().lp_copra_run(dg.handle, C.byref(opts), _lib.ptr(labs), _lib.ptr(bels), _lib.ptr(sizes),
                                       _lib.ptr(best), _lib.ptr(changed), C.byref(stats)))
    it = int(stats.iterations)
    return best, it, labs, bels, sizes, stats.as_dict(), changed[:it].copy()


def _detect_full(graph: Graph, params: CopraParams, check_invariants: bool = False):
    """Run COPRA and return the full final state (ref `copra.py:241-289`):
    ``(best, iterations, elapsed, stats, labs, bels, sizes)``; ``stats`` =
    [max |sum(bels) - 1|, min size, max size] (computed on the host here)."""
    if __debug__:
        check_symmetric(graph)
    n = graph.vertex_count
    stats = np.array([0.0, np.inf, -np.inf])
    start = time.perf_counter()
    best, it, labs, bels, sizes, _, _ = copra_run(graph, params)
    elapsed = time.perf_counter() - start
    if check_invariants and n:
        stats[0] = float(np.max(np.abs(bels.sum(axis=1) - 1.0)))
        stats[1] = float(sizes.min())
        stats[2] = float(sizes.max())
    return best, it, elapsed, stats, labs, bels, sizes


def copra_detect(graph: Graph, params: CopraParams | None = None) -> DetectionResult:
    """Run COPRA on a preprocessed graph; the assignment is each best label (ref `copra.py:292-297`)."""
    if params is None:
        params = CopraParams()
    if __debug__:
        check_symmetric(graph)
    if graph.vertex_count == 0:
        return DetectionResult(np.zeros(0, dtype=np.int64), 0, 0.0, 0.0)
    start = time.perf_counter()
    best, it, _, _, _, st, changed = copra_run(graph, params, want_sets=False)
    elapsed = time.perf_counter() - start
    st["changed"] = changed
    return DetectionResult(best, it, elapsed, score(graph, best), st)


def _select_labels(touched, tally, max_labels, rng):
    """Host restatement of `copra.py:53-108` (reference xorshift fallback draw)."""
    total = 0.0
    for lab in touched:
        total += tally[lab]
    out = []
    kept = 0.0
    for lab in touched:
        w = tally[lab]
        if w * max_labels >= total and len(out) < max_labels:
            out.append([lab, w])
            kept += w
    if not out:
        best_w = max(tally[lab] for lab in touched)
        ties = [lab for lab in touched if tally[lab] == best_w]
        j = draw_bounded(rng._state, 0, len(ties)) if len(ties) > 1 else 0
        return [ties[j]], [1.0]
    inv = 1.0 / kept
    for e in out:
        e[1] *= inv
    out.sort(key=lambda e: e[0])
    return [e[0] for e in out], [e[1] for e in out]


def collect_and_threshold(labels, weights, max_labels: int, rng: XorShift32):
    """Apply the normalize/threshold/fallback/renormalize step to one tally
    (ref `copra.py:300-324`).  Returns (labels, belongings) sorted by label id."""
    labs = np.asarray(labels, dtype=np.int64)
    wts = np.asarray(weights, dtype=np.float64)
    if labs.size == 0:
        raise ValueError("empty tally: callers handle neighborless vertices")
    if max_labels < 1:
        raise ValueError("max_labels must be >= 1")
    touched, tally = [], {}
    for lab, w in zip(labs.tolist(), wts.tolist()):
        if tally.get(lab, 0.0) == 0.0:  # first touch as the reference tests it (copra.py:316-319)
            touched.append(lab)
        tally[lab] = tally.get(lab, 0.0) + w
    out_l, out_b = _select_labels(touched, tally, max_labels, rng)
    return np.asarray(out_l, dtype=np.int64), np.asarray(out_b, dtype=np.float64)


def best_label(labels, belongings) -> int:
    """Maximum-belonging label; ties break to the smallest label id (ref `copra.py:327-338`)."""
    labs = np.asarray(labels, dtype=np.int64)
    bels = np.asarray(belongings, dtype=np.float64)
    if labs.size == 0:
        raise ValueError("empty label set")
    top = bels.max()
    return int(labs[bels == top].min())
