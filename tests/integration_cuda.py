# labelprop/_cuda.py -- the binding a maintainer would add to the reference
# package (Option B; kept verbatim there and checked by
# tests/test_integration_binding.py).  It replaces the numba kernel calls
# _rak_seq/_rak_par (rak.py:177-192), _copra_seq/_copra_par
# (copra.py:262-284) and _slpa_seq/_slpa_par + _project (slpa.py:169-184).
import ctypes as C
import os
import weakref

import numpy as np

_L = C.CDLL(os.environ.get("LABELPROP_CUDA_LIB", "liblabelprop_cuda.so"))


class RakOpts(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("max_iterations", C.c_int32), ("tie", C.c_int32),
                ("batches", C.c_int64), ("seed", C.c_uint32), ("flags", C.c_int32),
                ("reserved", C.c_int64 * 6)]


class CopraOpts(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("max_labels", C.c_int32), ("max_iterations", C.c_int32),
                ("batches", C.c_int64), ("seed", C.c_uint32), ("flags", C.c_int32),
                ("reserved", C.c_int64 * 6)]


class SlpaOpts(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("memory_size", C.c_int32), ("tie", C.c_int32),
                ("batches", C.c_int64), ("seed", C.c_uint32), ("flags", C.c_int32),
                ("reserved", C.c_int64 * 6)]


_L.lp_graph_create.argtypes = [C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_int32, C.POINTER(C.c_void_p)]
_L.lp_graph_destroy.argtypes = [C.c_void_p]
_L.lp_rak_run.argtypes = [C.c_void_p, C.POINTER(RakOpts)] + [C.c_void_p] * 5
_L.lp_copra_run.argtypes = [C.c_void_p, C.POINTER(CopraOpts)] + [C.c_void_p] * 6
_L.lp_slpa_run.argtypes = [C.c_void_p, C.POINTER(SlpaOpts)] + [C.c_void_p] * 4
_L.lp_last_error.restype = C.c_char_p


def _check(rc):
    if rc == -1:
        raise ValueError(_L.lp_last_error().decode())
    if rc != 0:
        raise RuntimeError(_L.lp_last_error().decode())


# device copies of the (immutable) Graph objects, uploaded once; kept outside
# the Graph so it stays picklable, freed when the Graph is collected
_HANDLES = {}


def _drop(key):
    h = _HANDLES.pop(key, None)
    if h is not None:
        _L.lp_graph_destroy(h)


def _handle(graph):
    key = id(graph)
    if key not in _HANDLES:
        h = C.c_void_p()
        w = graph.weights
        _check(_L.lp_graph_create(graph.vertex_count, graph.edge_count,
                                  graph.offsets.ctypes.data, graph.neighbors.ctypes.data,
                                  None if np.all(w == 1.0) else w.ctypes.data, -1, C.byref(h)))
        _HANDLES[key] = h
        weakref.finalize(graph, _drop, key)
    return _HANDLES[key]


def _iterations(stats):
    return int(C.cast(stats, C.POINTER(C.c_int32))[0])


def rak_cuda(graph, labels, order, strict, tolerance, max_iterations, seed):
    """Drop-in for _rak_seq: mutates `labels` (int64[n]) and returns iterations."""
    o = RakOpts(tolerance=tolerance, max_iterations=max_iterations, tie=0 if strict else 1,
                batches=0, seed=seed & 0xFFFFFFFF)
    out = np.empty_like(labels)
    stats = (C.c_int64 * 32)()
    _check(_L.lp_rak_run(_handle(graph), C.byref(o), order.ctypes.data, labels.ctypes.data,
                         out.ctypes.data, None, C.byref(stats)))
    labels[:] = out
    return _iterations(stats)


def copra_cuda(graph, params):
    """-> best, iterations, labs, bels, sizes (rows sorted by label, as _copra_seq leaves them)."""
    n, L = graph.vertex_count, params.max_labels
    best = np.empty(n, np.int64)
    labs = np.empty((n, L), np.int64)
    bels = np.empty((n, L), np.float64)
    sizes = np.empty(n, np.int64)
    o = CopraOpts(tolerance=params.tolerance, max_labels=L, max_iterations=params.max_iterations,
                  batches=0, seed=params.seed & 0xFFFFFFFF)
    stats = (C.c_int64 * 32)()
    _check(_L.lp_copra_run(_handle(graph), C.byref(o), labs.ctypes.data, bels.ctypes.data,
                           sizes.ctypes.data, best.ctypes.data, None, C.byref(stats)))
    return best, _iterations(stats), labs, bels, sizes


def slpa_cuda(graph, params):
    """-> labels (modal projection), iterations, slots, filled."""
    n, T = graph.vertex_count, params.memory_size
    labels = np.empty(n, np.int64)
    slots = np.empty((n, T), np.int64)
    o = SlpaOpts(tolerance=params.tolerance, memory_size=T, tie=0 if params.strict else 1,
                 batches=0, seed=params.seed & 0xFFFFFFFF)
    stats = (C.c_int64 * 32)()
    _check(_L.lp_slpa_run(_handle(graph), C.byref(o), labels.ctypes.data, slots.ctypes.data,
                          None, C.byref(stats)))
    it = _iterations(stats)
    return labels, it, slots, np.full(n, it + 1, np.int64)
