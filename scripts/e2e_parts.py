"""Where the end-to-end step goes (bench.py e2e): graph upload, plan build,
sweeps, label download, for R-MAT-22 from pinned int64 host arrays."""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2301_09125_b200 as lp  # noqa: E402
from paper_2301_09125_b200 import _lib  # noqa: E402

g = bench.make_graph(sys.argv[1] if len(sys.argv) > 1 else "rmat22")
L = _lib.lib()
arrays = [np.ascontiguousarray(g.offsets), np.ascontiguousarray(g.neighbors)]
for a in arrays:
    _lib.check(L.lp_host_register(_lib.ptr(a), a.nbytes))
p = lp.RakParams(strict=True, tolerance=0.05, max_iterations=20)
for step in range(4):
    t0 = time.perf_counter()
    fresh = lp.Graph(g.vertex_count, g.edge_count, arrays[0], arrays[1], g.weights, g.total_weight)
    dg = _lib.DeviceGraph(fresh, unit=True)
    t1 = time.perf_counter()
    out = np.empty(g.vertex_count, dtype=np.int64)
    st = _lib.RunStats()
    _lib.check(L.lp_rak_run(dg.handle, C.byref(lp.rak._opts(p)), None, None, _lib.ptr(out), None, C.byref(st)))
    t2 = time.perf_counter()
    dg.close()
    t3 = time.perf_counter()
    print(f"step {step}: create {1e3*(t1-t0):.1f} ms, run {1e3*(t2-t1):.1f} ms (plan {st.plan_ms:.1f}, sweeps "
          f"{st.kernel_ms:.1f}, rest {1e3*(t2-t1)-st.plan_ms-st.kernel_ms:.1f}), destroy {1e3*(t3-t2):.1f} ms, "
          f"total {1e3*(t3-t0):.1f} ms", flush=True)
