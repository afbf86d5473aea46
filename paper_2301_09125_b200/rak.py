"""RAK / label propagation, single label per vertex, on the B200.

Drop-in for the reference's ``labelprop.rak`` (`pkg/src/labelprop/rak.py`):
``RakParams`` keeps the reference's fields, defaults and validation
(`rak.py:40-54`) and adds three defaulted fields; ``rak_detect`` keeps the
signature and return contract (`rak.py:161-194`); ``choose_max_label``
keeps the helper semantics (`rak.py:197-218`).

The hot loop -- the sweep of ``_rak_seq`` / ``_rak_par`` (`rak.py:87-158`)
-- is one call into ``liblabelprop_cuda.so`` (``lp_rak_run``).  Nothing sits
between this module and the CUDA kernels but ctypes; there is no CPU
fallback.

Schedules (``RakParams.batches``):

* ``0`` (default) -- the reference's own visit: vertices in the seeded
  order ``shuffled_indices(n, seed)`` (`rak.py:171`), each reading its
  neighbours' freshest labels.  With ``strict=True`` this reproduces
  ``_rak_seq`` (the reference's deterministic mode, `SPEC.md:256`) label for
  label and iteration for iteration, computed on the GPU as the fixed
  point of the sweep's dependency system;
* ``1`` -- synchronous sweep: every vertex reads the labels of the previous
  sweep;
* ``B`` -- B snapshot batches over the same order.

Tie rules (``RakParams.tie``): ``None`` follows the reference -- strict
means ``"scan-first"`` (first maximum in CSR scan order, `rak.py:61-70`),
non-strict means ``"random"`` (uniform among maxima; on the GPU the draw
is a counter hash of (seed, sweep, vertex, label) instead of the
reference's sequential xorshift stream, which a parallel sweep cannot
replay).  ``"min-label"`` picks the smallest tied label (BASELINE config-0
wording).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .graph import Graph, check_symmetric
from .prng import XorShift32, draw_bounded
from .quality import score
from .result import DetectionResult

# Vertices per parallel work unit in the reference's _rak_par (rak.py:36-37);
# kept for API compatibility (the CUDA engine has no chunking knob).
CHUNK = 1024


@dataclass(frozen=True)
class RakParams:
    tolerance: float = 0.05
    strict: bool = False
    max_iterations: int = 100
    workers: int = 1
    seed: int = 1
    # --- additions (defaults keep the reference signature valid) ---
    batches: int = 0              # 0 = reference visit order (exact async); 1 = synchronous
    tie: Optional[str] = None     # None: "scan-first" if strict else "random"
    backend: str = "cuda"

    def __post_init__(self):
        if not 0.0 < self.tolerance <= 1.0:
            raise ValueError("tolerance must be in (0, 1]")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.batches < 0:
            raise ValueError("batches must be >= 0")
        if self.tie is not None and self.tie not in _lib.TIE_NAMES:
            raise ValueError(f"tie must be one of {sorted(_lib.TIE_NAMES)} or None")
        if self.backend != "cuda":
            raise ValueError("only the 'cuda' backend exists (no CPU fallback)")

    @property
    def tie_rule(self) -> str:
        if self.tie is not None:
            return self.tie
        return "scan-first" if self.strict else "random"


def _opts(params: RakParams) -> _lib.RakOpts:
    o = _lib.RakOpts()
    o.tolerance = float(params.tolerance)
    o.max_iterations = int(params.max_iterations)
    o.tie = _lib.TIE_NAMES[params.tie_rule]
    o.batches = int(params.batches)
    o.seed = int(params.seed) & 0xFFFFFFFF
    return o


def rak_labels(graph: Graph, params: RakParams | None = None, *, order=None, labels=None, profile: bool = False,
               device_graph: "_lib.DeviceGraph | None" = None):
    """The detection call without validation or scoring.

    Returns ``(labels, iterations, stats, changed_per_sweep)``.  This is the
    timed body of ``rak_detect`` (the reference times the same span,
    `rak.py:172-193`); bench.py drives it for the end-to-end number.
    """
    if params is None:
        params = RakParams()
    n = graph.vertex_count
    if n == 0:
        return np.zeros(0, dtype=np.int64), 0, {}, np.zeros(0, dtype=np.int64)
    out = np.empty(n, dtype=np.int64)  # written by lp_rak_run
    dg = device_graph if device_graph is not None else _lib.device_graph(graph)
    opts = _opts(params)
    if profile:
        opts.flags |= _lib.RAK_PROFILE
    order_arr = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
    init = None if labels is None else np.ascontiguousarray(labels, dtype=np.int64)
    if order_arr is not None and order_arr.shape != (n,):
        raise ValueError("order must have one entry per vertex")
    if init is not None and init.shape != (n,):
        raise ValueError("labels must have one entry per vertex")
    changed = np.zeros(params.max_iterations, dtype=np.int64)
    stats = _lib.RunStats()
    _lib.check(_lib.lib().lp_rak_run(dg.handle, C.byref(opts), _lib.ptr(order_arr), _lib.ptr(init), _lib.ptr(out),
                                     _lib.ptr(changed), C.byref(stats)))
    return out, int(stats.iterations), stats.as_dict(), changed[: stats.iterations].copy()


def rak_detect(graph: Graph, params: RakParams | None = None, *, order=None, labels=None,
               changed_history: bool = False) -> DetectionResult:
    """Run RAK on a preprocessed graph (ref `rak.py:161-194`).

    ``order`` overrides the visit permutation (default
    ``shuffled_indices(n, seed)``); ``labels`` overrides the initial labels
    (default ``arange(n)``).  ``changed_history`` adds the per-sweep changed
    counts to ``result.stats``.
    """
    if params is None:
        params = RakParams()
    if __debug__:
        check_symmetric(graph)
    if graph.vertex_count == 0:
        return DetectionResult(np.zeros(0, dtype=np.int64), 0, 0.0, 0.0)
    start = time.perf_counter()
    out, iterations, st, changed = rak_labels(graph, params, order=order, labels=labels)
    elapsed = time.perf_counter() - start
    if changed_history:
        st["changed"] = changed
    return DetectionResult(out, iterations, elapsed, score(graph, out), st)


def _pick_from_tally(labels_in_order, weights_by_label, strict, states, slot):
    """Host restatement of `rak.py:57-84` for ``choose_max_label``."""
    best_w = -1.0
    best = -1
    for lab in labels_in_order:
        w = weights_by_label[lab]
        if w > best_w:
            best_w, best = w, lab
    if strict or len(labels_in_order) == 1:
        return best
    ties = [lab for lab in labels_in_order if weights_by_label[lab] == best_w]
    if len(ties) == 1:
        return best
    return ties[draw_bounded(states, slot, len(ties))]


def choose_max_label(labels, weights, strict: bool, rng: XorShift32) -> int:
    """Winning label of a tally given as parallel arrays (ref `rak.py:197-218`).

    Strict: the first maximum-weight label in scan order; non-strict: uniform
    among the tied maxima using ``rng`` (the reference's xorshift stream).
    """
    labs = np.asarray(labels, dtype=np.int64)
    wts = np.asarray(weights, dtype=np.float64)
    if labs.size == 0:
        raise ValueError("empty tally")
    if labs.size != wts.size:
        raise ValueError("labels and weights must have equal length")
    order, tally = [], {}
    for lab, w in zip(labs.tolist(), wts.tolist()):
        if lab not in tally:
            order.append(lab)
            tally[lab] = 0.0
        tally[lab] += w
    return int(_pick_from_tally(order, tally, strict, rng._state, 0))
