"""One RAK detection on a benchmark graph, for ncu / compute-sanitizer runs.

    python scripts/prof_run.py [--config rmat22] [--batches 0] [--non-strict] [--runs 1]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2301_09125_b200 as lp  # noqa: E402
from paper_2301_09125_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="rmat22")
ap.add_argument("--batches", type=int, default=0)
ap.add_argument("--non-strict", action="store_true")
ap.add_argument("--runs", type=int, default=1)
ap.add_argument("--no-calibrate", action="store_true")
args = ap.parse_args()
g = bench.make_graph(args.config)
cfg = bench.CONFIGS[args.config]
p = lp.RakParams(strict=not args.non_strict, batches=args.batches, tolerance=cfg["tolerance"],
                 max_iterations=cfg["max_iterations"])
dg = _lib.DeviceGraph(g)
for r in range(args.runs):
    t = time.perf_counter()
    labels, it, st, changed = lp.rak_labels(g, p, device_graph=dg, profile=True)
    print(f"run {r}: iterations {it} rounds {st['rounds']} kernel_ms {st['kernel_ms']:.3f} plan_ms {st['plan_ms']:.3f} "
          f"bin_ms {[round(x, 3) for x in st['bin_ms']]} gather_ms {st['gather_ms']:.3f} route_ms {st['aux_ms']:.3f} gathered {st['arcs_gathered']/1e6:.1f}M bin_launches {st['bin_launches']} changed {changed.tolist()} "
          f"wall {time.perf_counter() - t:.3f}s", flush=True)

import ctypes as C
for mode in (() if args.no_calibrate else (0, 1, 2, 3, 4, 5)):
    ms = C.c_double(0)
    _lib.check(_lib.lib().lp_calibrate(dg.handle, mode, 10, C.byref(ms)))
    print(f"calibrate mode {mode}: {ms.value * 1e3:.1f} us per pass over the active rows")
