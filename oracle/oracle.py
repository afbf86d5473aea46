"""ctypes front end of the CPU oracle (``lp_oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke``
and ``bench.py``'s CPU-baseline leg, never by the product package.  See the
header of ``lp_oracle.c`` for what each function restates (reference
file:line) and how the restatement is pinned to the reference.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblp_oracle.so")

TIE_SCAN_FIRST = 0
TIE_RANDOM = 1
TIE_MIN_LABEL = 2
TIE_XORSHIFT = 3

_lib = None

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build() -> str:
    """Compile the oracle with its Makefile (system gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
            os.path.join(HERE, "lp_oracle.c")
        ):
            build()
        L = C.CDLL(LIB_PATH)
        L.or_xs32_next.argtypes = [C.c_uint32]
        L.or_xs32_next.restype = C.c_uint32
        L.or_mix_seed.argtypes = [C.c_uint32, C.c_uint32]
        L.or_mix_seed.restype = C.c_uint32
        L.or_tie_hash.argtypes = [C.c_uint32] * 4
        L.or_tie_hash.restype = C.c_uint32
        L.or_shuffled_indices.argtypes = [C.c_int64, C.c_uint32, _i64p]
        L.or_shuffled_indices.restype = None
        L.or_rak.argtypes = [C.c_int64, _i64p, _i64p, C.c_void_p, _i64p, C.c_int64, C.c_int,
                             C.c_uint32, C.c_double, C.c_int, _i64p, C.c_void_p, C.c_void_p]
        L.or_rak.restype = C.c_int
        L.or_rak_par.argtypes = [C.c_int64, _i64p, _i64p, C.c_void_p, _i64p, C.c_int, C.c_uint32,
                                 C.c_double, C.c_int, C.c_int, C.c_int64, _i64p]
        L.or_rak_par.restype = C.c_int
        L.or_max_threads.restype = C.c_int
        L.or_copra.argtypes = [C.c_int64, _i64p, _i64p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                               C.c_uint32, C.c_double, C.c_int, _i64p, _f64p, _i64p, _i64p]
        L.or_copra.restype = C.c_int
        L.or_slpa.argtypes = [C.c_int64, _i64p, _i64p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                              C.c_int, C.c_uint32, C.c_double, _i64p, _i64p, _i64p, _i64p]
        L.or_slpa.restype = C.c_int
        L.or_modularity.argtypes = [C.c_int64, _i64p, _i64p, C.c_void_p, _i64p, C.c_double]
        L.or_modularity.restype = C.c_double
        _lib = L
    return _lib


class Prepared:
    """A graph's CSR converted once to the oracle's argument types (int64
    offsets / neighbours, float64 weights, the all-unit test done), so timed
    loops pay only the kernel, as the reference's ``elapsed`` does
    (rak.py:171-172 prepare ``order`` and the scratch before the clock)."""

    def __init__(self, g):
        self.vertex_count = int(g.vertex_count)
        self.edge_count = int(g.edge_count)
        self.total_weight = float(g.total_weight)
        self.csr = _csr(g)
        self.offsets, self.neighbors, self.weights = self.csr[:3]


def prepare(g) -> Prepared:
    return g if isinstance(g, Prepared) else Prepared(g)


def _csr(g):
    if isinstance(g, Prepared):
        return g.csr
    off = np.ascontiguousarray(g.offsets, dtype=np.int64)
    nbr = np.ascontiguousarray(g.neighbors, dtype=np.int64)
    w = np.ascontiguousarray(g.weights, dtype=np.float64)
    unit = bool(np.all(w == 1.0))
    return off, nbr, w, unit


def _wptr(w, unit):
    return None if unit else w.ctypes.data_as(C.c_void_p)


def shuffled_indices(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    lib().or_shuffled_indices(n, seed & 0xFFFFFFFF, out)
    return out


def tie_hash(seed, sweep, vertex, label) -> int:
    return int(lib().or_tie_hash(seed & 0xFFFFFFFF, sweep, vertex, label))


def rak(g, *, batches=0, tie=TIE_SCAN_FIRST, seed=1, tolerance=0.05, max_iterations=100,
        order=None, labels=None, per_iteration=False):
    """Batched RAK restatement.  batches=0 means n (the reference order).

    Returns (labels, iterations, changed_per_iteration[, labels_per_iteration]).
    """
    n = g.vertex_count
    off, nbr, w, unit = _csr(g)
    if order is None:
        order = shuffled_indices(n, seed)
    order = np.ascontiguousarray(order, dtype=np.int64)
    lab = np.arange(n, dtype=np.int64) if labels is None else np.array(labels, dtype=np.int64)
    changed = np.zeros(max_iterations, dtype=np.int64)
    per = np.zeros((max_iterations, n), dtype=np.int64) if per_iteration else None
    it = lib().or_rak(n, off, nbr, _wptr(w, unit), order, int(batches), int(tie), seed & 0xFFFFFFFF,
                      float(tolerance), int(max_iterations), lab, changed.ctypes.data_as(C.c_void_p),
                      per.ctypes.data_as(C.c_void_p) if per is not None else None)
    if it < 0:
        raise MemoryError("oracle allocation failed")
    if per_iteration:
        return lab, it, changed[:it], per[:it]
    return lab, it, changed[:it]


def rak_par(g, *, strict=True, seed=1, tolerance=0.05, max_iterations=100, threads=None, chunk=1024,
            order=None):
    """OpenMP port of the reference's ``_rak_par`` (the bench CPU arm)."""
    n = g.vertex_count
    off, nbr, w, unit = _csr(g)
    if order is None:
        order = shuffled_indices(n, seed)
    order = np.ascontiguousarray(order, dtype=np.int64)
    lab = np.arange(n, dtype=np.int64)
    threads = threads or lib().or_max_threads()
    it = lib().or_rak_par(n, off, nbr, _wptr(w, unit), order,
                          TIE_SCAN_FIRST if strict else TIE_XORSHIFT, seed & 0xFFFFFFFF,
                          float(tolerance), int(max_iterations), int(threads), int(chunk), lab)
    if it < 0:
        raise MemoryError("oracle allocation failed")
    return lab, it


def copra(g, *, max_labels=8, batches=0, tie=TIE_XORSHIFT, seed=1, tolerance=0.01, max_iterations=100):
    """Batched COPRA restatement (index order).  Returns (best, iterations, labs, bels, sizes)."""
    n = g.vertex_count
    off, nbr, w, unit = _csr(g)
    L = int(max_labels)
    labs = np.zeros((n, L), dtype=np.int64)
    bels = np.zeros((n, L), dtype=np.float64)
    labs[:, 0] = np.arange(n)
    bels[:, 0] = 1.0
    sizes = np.ones(n, dtype=np.int64)
    best = np.arange(n, dtype=np.int64)
    it = lib().or_copra(n, off, nbr, _wptr(w, unit), L, int(batches), int(tie), seed & 0xFFFFFFFF,
                        float(tolerance), int(max_iterations), labs.reshape(-1), bels.reshape(-1), sizes,
                        best)
    return best, it, labs, bels, sizes


def slpa(g, *, memory_size=20, batches=0, tie=TIE_XORSHIFT, speaker_rng=0, seed=1, tolerance=0.05):
    """Batched SLPA restatement (index order).  Returns (labels, iterations, slots, filled)."""
    n = g.vertex_count
    off, nbr, w, unit = _csr(g)
    T = int(memory_size)
    slots = np.zeros((n, T), dtype=np.int64)
    slots[:, 0] = np.arange(n)
    filled = np.ones(n, dtype=np.int64)
    prev = np.full(n, -1, dtype=np.int64)
    labels = np.empty(n, dtype=np.int64)
    it = lib().or_slpa(n, off, nbr, _wptr(w, unit), T, int(batches), int(tie), int(speaker_rng),
                       seed & 0xFFFFFFFF, float(tolerance), slots.reshape(-1), filled, prev, labels)
    return labels, it, slots, filled


def modularity(g, labels) -> float:
    off, nbr, w, unit = _csr(g)
    lab = np.ascontiguousarray(labels, dtype=np.int64)
    return float(lib().or_modularity(g.vertex_count, off, nbr, _wptr(w, unit), lab, float(g.total_weight)))
