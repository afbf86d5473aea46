"""Experiment: gather / tally cost with the R-MAT vertex ids relabelled by
descending degree (hubs' labels packed together)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2301_09125_b200 as lp  # noqa: E402
from paper_2301_09125_b200 import _lib  # noqa: E402


def relabel(g, perm):
    # perm[old] = new
    n = g.vertex_count
    deg = np.diff(g.offsets)
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    ndeg = deg[inv]
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(ndeg, out=off[1:])
    rows = np.repeat(np.arange(n), deg)
    nr = perm[rows]
    nc = perm[g.neighbors]
    order = np.lexsort((nc, nr))
    nbr = nc[order]
    return lp.Graph(n, g.edge_count, off, nbr, np.ones(g.edge_count), g.total_weight)


g = bench.make_graph("rmat22")
deg = np.diff(g.offsets)
perm = np.empty(g.vertex_count, dtype=np.int64)
perm[np.argsort(-deg, kind="stable")] = np.arange(g.vertex_count)
gr = relabel(g, perm)
for name, gg in (("orig", g), ("degree-sorted", gr)):
    for batches in (0, 1):
        p = lp.RakParams(strict=True, batches=batches, tolerance=0.05, max_iterations=20)
        dg = _lib.DeviceGraph(gg)
        for r in range(2):
            labels, it, st, ch = lp.rak_labels(gg, p, device_graph=dg, profile=True)
        print(f"{name} B={batches}: it {it} rounds {st['rounds']} kernel_ms {st['kernel_ms']:.2f} bin_ms "
              f"{[round(x, 2) for x in st['bin_ms']]} gather {st['gather_ms']:.2f} aux {st['aux_ms']:.2f}", flush=True)
        for mode in (2, 3):
            ms = C.c_double(0)
            _lib.check(_lib.lib().lp_calibrate(dg.handle, mode, 10, C.byref(ms)))
            print(f"   calibrate {mode}: {ms.value * 1e3:.1f} us")
        dg.close()
