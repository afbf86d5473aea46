"""Device ms per detection (median of N runs, inputs resident) for A/B builds.

    LP_LIB_PATH=build/x.so python scripts/ab_time.py [--config rmat22] [--runs 7] [--batches 0 1] [--non-strict]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2301_09125_b200 as lp  # noqa: E402
from paper_2301_09125_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="rmat22")
ap.add_argument("--runs", type=int, default=7)
ap.add_argument("--batches", type=int, nargs="+", default=[0, 1])
ap.add_argument("--non-strict", action="store_true")
ap.add_argument("--tag", default=os.environ.get("LP_LIB_PATH", "in-tree"))
args = ap.parse_args()
g = bench.make_graph(args.config)
cfg = bench.CONFIGS[args.config]
dg = _lib.DeviceGraph(g)
for b in args.batches:
    p = lp.RakParams(strict=not args.non_strict, batches=b, tolerance=cfg["tolerance"],
                     max_iterations=cfg["max_iterations"])
    ms, labels = [], None
    for r in range(args.runs + 1):
        labels, it, st, changed = lp.rak_labels(g, p, device_graph=dg)
        if r:
            ms.append(st["kernel_ms"])
    print(f"{args.tag} {args.config} batches={b} {'non-strict' if args.non_strict else 'strict'}: mean {np.mean(ms):.3f} "
          f"median {np.median(ms):.3f} ms min {min(ms):.3f} it {it} rounds {st['rounds']} "
          f"changed {changed.tolist()} labels_hash {hash(labels.tobytes()) & 0xffffffff:08x}", flush=True)
