"""SLPA (speaker-listener label propagation) on the B200.

Drop-in for the reference's ``labelprop.slpa`` (`pkg/src/labelprop/
slpa.py`): ``SlpaParams`` keeps the reference's fields, defaults and
validation (`slpa.py:34-48`) and adds defaulted ``batches`` / ``tie`` /
``backend`` fields; ``slpa_detect`` keeps the signature and result contract
(`slpa.py:189-194`); ``most_popular_label`` keeps the helper
(`slpa.py:197-202`).

The speaking rounds and the projection (`slpa.py:91-150`) run in one call
into ``liblabelprop_cuda.so`` (``lp_slpa_run``): each round is the RAK
sweep machinery with a phase-1 gather that draws every speaker's spoken
label from its memory.  Schedules as in RAK (index visit
order, `slpa.py:99`): ``batches=0`` is the reference's in-place sweep
(every listener hears the freshest memories), ``1`` synchronous rounds.

Randomness: the reference draws speakers' slots (and non-strict ties) from
one sequential xorshift stream (`slpa.py:76`), which a parallel round cannot
replay; here slot ``j = speak_hash(seed, t, v, k) mod filled[u]`` for the
k-th speaking neighbour of listener v in round t, and ties use the RAK
counter hash.  The oracle (`oracle/lp_oracle.c` ``or_slpa``) implements the
same rule, so GPU runs match it exactly; against the reference's own
draws, parity is statistical (modularity / community counts).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .graph import Graph, check_symmetric
from .quality import score
from .result import DetectionResult

CHUNK = 1024  # the reference's parallel work unit (slpa.py:31); no CUDA counterpart


@dataclass(frozen=True)
class SlpaParams:
    memory_size: int = 20
    tolerance: float = 0.05
    strict: bool = False
    workers: int = 1
    seed: int = 1
    # --- additions (defaults keep the reference signature valid) ---
    batches: int = 0              # 0 = reference visit (in-place, index order); 1 = synchronous
    tie: Optional[str] = None     # None: "scan-first" if strict else "random"
    backend: str = "cuda"

    def __post_init__(self):
        if self.memory_size < 2:
            raise ValueError("memory_size must be >= 2")
        if not 0.0 < self.tolerance <= 1.0:
            raise ValueError("tolerance must be in (0, 1]")
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


def _opts(params: SlpaParams) -> _lib.SlpaOpts:
    o = _lib.SlpaOpts()
    o.tolerance = float(params.tolerance)
    o.memory_size = int(params.memory_size)
    o.tie = _lib.TIE_NAMES[params.tie_rule]
    o.batches = int(params.batches)
    o.seed = int(params.seed) & 0xFFFFFFFF
    return o


def slpa_run(graph: Graph, params: SlpaParams | None = None, *, want_slots: bool = True, profile: bool = False,
             device_graph: "_lib.DeviceGraph | None" = None):
    """One SLPA run on the GPU.

    Returns ``(labels, iterations, slots, filled, stats, repeats_per_round)``
    -- ``slots``/``filled`` as the reference's ``_detect_full`` returns them
    (`slpa.py:154-186`; ``slots`` is None without ``want_slots``).
    """
    if params is None:
        params = SlpaParams()
    n = graph.vertex_count
    T = params.memory_size
    if n == 0:
        return (np.zeros(0, dtype=np.int64), 0, np.zeros((0, T), dtype=np.int64), np.zeros(0, dtype=np.int64),
                {}, np.zeros(0, dtype=np.int64))
    dg = device_graph if device_graph is not None else _lib.device_graph(graph)
    opts = _opts(params)
    if profile:
        opts.flags |= _lib.RAK_PROFILE
    labels = np.empty(n, dtype=np.int64)
    slots = np.empty((n, T), dtype=np.int64) if want_slots else None
    repeats = np.zeros(T - 1, dtype=np.int64)
    stats = _lib.RunStats()
    _lib.check(_lib.lib().lp_slpa_run(dg.handle, C.byref(opts), _lib.ptr(labels), _lib.ptr(slots),
                                      _lib.ptr(repeats), C.byref(stats)))
    it = int(stats.iterations)
    filled = np.full(n, it + 1, dtype=np.int64)
    return labels, it, slots, filled, stats.as_dict(), repeats[:it].copy()


def _detect_full(graph: Graph, params: SlpaParams):
    """Run SLPA and return (labels, iterations, elapsed, slots, filled) (ref `slpa.py:154-186`)."""
    if __debug__:
        check_symmetric(graph)
    start = time.perf_counter()
    labels, it, slots, filled, _, _ = slpa_run(graph, params)
    elapsed = time.perf_counter() - start
    return labels, it, elapsed, slots, filled


def slpa_detect(graph: Graph, params: SlpaParams | None = None) -> DetectionResult:
    """Run SLPA on a preprocessed graph; the assignment is each modal label (ref `slpa.py:189-194`)."""
    if params is None:
        params = SlpaParams()
    if __debug__:
        check_symmetric(graph)
    if graph.vertex_count == 0:
        return DetectionResult(np.zeros(0, dtype=np.int64), 0, 0.0, 0.0)
    start = time.perf_counter()
    labels, it, _, _, st, repeats = slpa_run(graph, params, want_slots=False)
    elapsed = time.perf_counter() - start
    st["repeats"] = repeats
    return DetectionResult(labels, it, elapsed, score(graph, labels), st)


def _modal(arr: np.ndarray) -> int:
    # slpa.py:51-66: most frequent label, frequency ties to the smallest id
    vals, counts = np.unique(arr, return_counts=True)
    return int(vals[np.argmax(counts)])  # np.unique sorts: the first max is the smallest id


def most_popular_label(memory) -> int:
    """Modal label of a memory; frequency ties break to the smallest id (ref `slpa.py:197-202`)."""
    arr = np.asarray(memory, dtype=np.int64)
    if arr.size == 0:
        raise ValueError("empty memory")
    return _modal(arr)
