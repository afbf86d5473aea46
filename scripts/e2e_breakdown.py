"""Where the end-to-end time of bench.py's e2e leg goes (R-MAT-22)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2301_09125_b200 as lp  # noqa: E402
from paper_2301_09125_b200 import _lib  # noqa: E402

g = bench.make_graph("rmat22")
L = _lib.lib()
arrays = [np.ascontiguousarray(g.offsets), np.ascontiguousarray(g.neighbors)]
for a in arrays:
    _lib.check(L.lp_host_register(_lib.ptr(a), a.nbytes))
p = lp.RakParams(strict=True, tolerance=0.05, max_iterations=20)
import torch  # noqa: E402

for r in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fresh = lp.Graph(g.vertex_count, g.edge_count, arrays[0], arrays[1], g.weights, g.total_weight)
    dg = _lib.DeviceGraph(fresh, unit=True)
    t1 = time.perf_counter()
    labels, it, st, _ = lp.rak_labels(fresh, p, device_graph=dg)
    t2 = time.perf_counter()
    dg.close()
    t3 = time.perf_counter()
    print(f"run {r}: create {1e3 * (t1 - t0):.1f} ms, detect {1e3 * (t2 - t1):.1f} ms (plan {st['plan_ms']:.1f}, "
          f"sweeps {st['kernel_ms']:.1f}), close {1e3 * (t3 - t2):.1f} ms, total {1e3 * (t3 - t0):.1f}", flush=True)
