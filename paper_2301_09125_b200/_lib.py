"""ctypes binding of ``liblabelprop_cuda.so`` (the C-ABI in
``include/labelprop_cuda.h``).

This module takes the place of the reference's ``_backend.py``
(`pkg/src/labelprop/_backend.py:19-52`): there, the compile backend is
numba's ``njit``/``prange`` and the hot loops run as numba-compiled
functions; here the hot loops are sm_100a CUDA kernels reached through one
ctypes call per detection run.  There is no CPU fallback: if the library is
missing or no GPU is present, the detectors raise.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import weakref

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# (LP_LIB_PATH: an alternative build of the same library, for A/B timing)
LIB_PATH = os.environ.get("LP_LIB_PATH") or os.path.join(HERE, "liblabelprop_cuda.so")
CSRC = os.path.join(HERE, "csrc")

LP_OK = 0
LP_ERR_INVALID = -1
LP_ERR_CUDA = -2
LP_ERR_NOMEM = -3
LP_ERR_UNSUPPORTED = -4

TIE_SCAN_FIRST = 0
TIE_RANDOM = 1
TIE_MIN_LABEL = 2
TIE_NAMES = {"scan-first": TIE_SCAN_FIRST, "random": TIE_RANDOM, "min-label": TIE_MIN_LABEL}

WEIGHT_MODES = {0: "unit", 1: "fixed", 2: "float"}


class GraphInfo(C.Structure):
    _fields_ = [
        ("vertex_count", C.c_int64),
        ("edge_count", C.c_int64),
        ("weight_mode", C.c_int32),
        ("fixed_shift", C.c_int32),
        ("max_degree", C.c_int64),
        ("device_bytes", C.c_int64),
        ("device", C.c_int32),
        ("reserved", C.c_int32 * 7),
    ]


class RakOpts(C.Structure):
    _fields_ = [
        ("tolerance", C.c_double),
        ("max_iterations", C.c_int32),
        ("tie", C.c_int32),
        ("batches", C.c_int64),
        ("seed", C.c_uint32),
        ("flags", C.c_int32),
        ("reserved", C.c_int64 * 6),
    ]


class SlpaOpts(C.Structure):
    _fields_ = [
        ("tolerance", C.c_double),
        ("memory_size", C.c_int32),
        ("tie", C.c_int32),
        ("batches", C.c_int64),
        ("seed", C.c_uint32),
        ("flags", C.c_int32),
        ("reserved", C.c_int64 * 6),
    ]


class CopraOpts(C.Structure):
    _fields_ = [
        ("tolerance", C.c_double),
        ("max_labels", C.c_int32),
        ("max_iterations", C.c_int32),
        ("batches", C.c_int64),
        ("seed", C.c_uint32),
        ("flags", C.c_int32),
        ("reserved", C.c_int64 * 6),
    ]


RAK_PROFILE = 1
STATS_FUSED = 1  # lp_run_stats.flags: labels gathered inside the tally kernels
BIN_NAMES = ("hub", "team", "warp", "small")


class RunStats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("rounds", C.c_int32),
        ("kernel_ms", C.c_double),
        ("plan_ms", C.c_double),
        ("arcs_scanned", C.c_int64),
        ("arcs_dense", C.c_int64),
        ("launches", C.c_int32),
        ("reserved0", C.c_int32),
        ("bin_ms", C.c_double * 4),
        ("bin_launches", C.c_int64 * 4),
        ("bin_arcs", C.c_int64 * 4),
        ("bin_vertices", C.c_int64 * 4),
        ("aux_ms", C.c_double),
        ("gather_ms", C.c_double),
        ("arcs_gathered", C.c_int64),
        ("gather_launches", C.c_int64),
        ("flags", C.c_int64),
    ]

    def as_dict(self) -> dict:
        d = {}
        for k, _ in self._fields_:
            if k.startswith("reserved"):
                continue
            v = getattr(self, k)
            d[k] = list(v) if k.startswith("bin_") else v
        return d


# every symbol include/labelprop_cuda.h declares (checked by tests/test_host_abi.py)
EXPORTS = (
    "lp_graph_create",
    "lp_graph_destroy",
    "lp_graph_get_info",
    "lp_graph_stream",
    "lp_rak_run",
    "lp_rak_run_resident",
    "lp_labels_download",
    "lp_slpa_run",
    "lp_copra_run",
    "lp_modularity",
    "lp_calibrate",
    "lp_shuffled_indices",
    "lp_gen_rmat",
    "lp_csr_build_undirected",
    "lp_gen_rmat_csr",
    "lp_csr_build_undirected_gpu",
    "lp_host_register",
    "lp_host_unregister",
    "lp_last_error",
    "lp_version",
    "lp_device_count",
)

_lib = None
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


def build(verbose: bool = False) -> str:
    """Compile the CUDA library in-tree (nvcc, sm_100a)."""
    out = subprocess.run(["make", "-s", "-C", CSRC], capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"building liblabelprop_cuda.so failed:\n{out.stdout}\n{out.stderr}")
    return LIB_PATH


def lib():
    """Load the library (no GPU needed to load; compute calls need one)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C {CSRC}` or "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)"
        )
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.lp_graph_create.argtypes = [C.c_int64, C.c_int64, vp, vp, vp, C.c_int32, C.POINTER(vp)]
    L.lp_graph_destroy.argtypes = [vp]
    L.lp_graph_get_info.argtypes = [vp, C.POINTER(GraphInfo)]
    L.lp_graph_stream.argtypes = [vp]
    L.lp_graph_stream.restype = vp
    L.lp_rak_run.argtypes = [vp, C.POINTER(RakOpts), vp, vp, vp, vp, C.POINTER(RunStats)]
    L.lp_rak_run_resident.argtypes = [vp, C.POINTER(RakOpts), vp, C.POINTER(RunStats)]
    L.lp_labels_download.argtypes = [vp, vp]
    L.lp_modularity.argtypes = [vp, vp, C.c_double, C.POINTER(C.c_double)]
    L.lp_copra_run.argtypes = [vp, C.POINTER(CopraOpts), vp, vp, vp, vp, vp, C.POINTER(RunStats)]
    L.lp_slpa_run.argtypes = [vp, C.POINTER(SlpaOpts), vp, vp, vp, C.POINTER(RunStats)]
    L.lp_calibrate.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
    L.lp_shuffled_indices.argtypes = [C.c_int64, C.c_uint32, _i64p]
    L.lp_gen_rmat.argtypes = [C.c_int32, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_uint64, _i64p, _i64p]
    L.lp_csr_build_undirected.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _i64p, _i64p, C.POINTER(C.c_int64)]
    L.lp_gen_rmat_csr.argtypes = [C.c_int32, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int32,
                                  _i64p, _i64p, C.c_int64, C.POINTER(C.c_int64)]
    L.lp_csr_build_undirected_gpu.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, C.c_int32, _i64p, _i64p, C.c_int64,
                                              C.POINTER(C.c_int64)]
    L.lp_host_register.argtypes = [vp, C.c_int64]
    L.lp_host_unregister.argtypes = [vp]
    L.lp_last_error.restype = C.c_char_p
    L.lp_version.restype = C.c_char_p
    L.lp_device_count.argtypes = [C.POINTER(C.c_int32)]
    for name in EXPORTS:
        if name not in ("lp_graph_stream", "lp_last_error", "lp_version"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exceptions."""
    if rc == LP_OK:
        return
    msg = lib().lp_last_error().decode(errors="replace")
    if rc == LP_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"liblabelprop_cuda: {msg} (code {rc})")


def device_count() -> int:
    c = C.c_int32(0)
    lib().lp_device_count(C.byref(c))
    return int(c.value)


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class DeviceGraph:
    """An uploaded CSR graph (``lp_graph`` handle); freed with the object."""

    def __init__(self, graph, device: int = -1, unit: bool | None = None):
        self.n = int(graph.vertex_count)
        self.m = int(graph.edge_count)
        off = np.ascontiguousarray(graph.offsets, dtype=np.int64)
        nbr = np.ascontiguousarray(graph.neighbors, dtype=np.int64)
        w = np.ascontiguousarray(graph.weights, dtype=np.float64)
        if unit is None:  # the device re-checks; this only skips uploading all-ones weights
            unit = bool(w.size == 0 or np.all(w == 1.0))
        h = C.c_void_p()
        check(lib().lp_graph_create(self.n, self.m, ptr(off), ptr(nbr), None if unit else ptr(w), device,
                                    C.byref(h)))
        self.handle = h

    def info(self) -> dict:
        gi = GraphInfo()
        check(lib().lp_graph_get_info(self.handle, C.byref(gi)))
        d = {k: getattr(gi, k) for k, _ in gi._fields_ if k != "reserved"}
        d["weight_mode"] = WEIGHT_MODES.get(d["weight_mode"], d["weight_mode"])
        return d

    @property
    def stream(self) -> int:
        return int(lib().lp_graph_stream(self.handle) or 0)

    def close(self):
        if getattr(self, "handle", None):
            lib().lp_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# Device copies of immutable ``Graph`` objects, keyed by id() and dropped when
# the Graph is collected (weakref.finalize) or released explicitly.  Kept
# outside the Graph so Graph objects stay picklable / deep-copyable like the
# reference's (graph.py:34-50) and carry no GPU state.
_DEVICE_CACHE: dict = {}


def _drop(key: int) -> None:
    dg = _DEVICE_CACHE.pop(key, None)
    if dg is not None:
        dg.close()


def device_graph(graph) -> DeviceGraph:
    """The cached device copy of an immutable ``Graph`` (uploaded once)."""
    key = id(graph)
    dg = _DEVICE_CACHE.get(key)
    if dg is None or dg.handle is None or dg.owner() is not graph:
        dg = DeviceGraph(graph)
        dg.owner = weakref.ref(graph)
        _DEVICE_CACHE[key] = dg
        weakref.finalize(graph, _drop, key)
    return dg


def release_device_graph(graph) -> bool:
    """Free the device copy of ``graph`` (CSR, plans, route buffers) now
    instead of when the Graph is collected.  Returns whether one existed."""
    key = id(graph)
    dg = _DEVICE_CACHE.get(key)
    if dg is None or dg.owner() is not graph:
        return False
    _drop(key)
    return True
