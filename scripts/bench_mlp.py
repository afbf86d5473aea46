"""COPRA / SLPA throughput on the BASELINE configs 3 and 4 (one JSON line each).

    python scripts/bench_mlp.py [--algo copra|slpa|all] [--steps 3] [--warmup 3] [--no-cpu]

COPRA: R-MAT scale 20, edge factor 16, unit weights, k = 1, 4, 8, 16,
tolerance 0.01, max 20 sweeps, the reference's in-place index-order sweep
(batches=0) and the synchronous sweep.  SLPA: planted partition n = 1e6
(10,000 x 100, 16 intra + 4 random), T = 10, 20, 50, tolerance 0.05.
value = dense-equivalent GTEPS = edge_count x sweeps / device time (CUDA
events of the library's stream, inputs resident).  cpu = the oracle's
sequential restatement (one core) of the same run, for scale.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2301_09125_b200 as lp  # noqa: E402
from paper_2301_09125_b200 import _lib  # noqa: E402
from paper_2301_09125_b200.copra import copra_run  # noqa: E402
from paper_2301_09125_b200.slpa import slpa_run  # noqa: E402


def _peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


PEAK = _peak()


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    ms, its = [], []
    for _ in range(steps):
        it, kms = fn()
        ms.append(kms)
        its.append(it)
    return float(np.median(ms)), its[-1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", default="all", choices=["copra", "slpa", "all"])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    from oracle import oracle as O

    if args.algo in ("copra", "all"):
        g = lp.rmat(20, seed=1)
        dg = _lib.DeviceGraph(g)
        for batches in (0, 1):
            for K in (1, 4, 8, 16):
                p = lp.CopraParams(max_labels=K, max_iterations=20, seed=1, batches=batches)

                def run():
                    best, it, _, _, _, st, _ = copra_run(g, p, want_sets=False, device_graph=dg)
                    run.best = best
                    return it, st["kernel_ms"]

                ms, it = timed(run, args.steps, args.warmup)
                # roofline: per dense sweep 4 B index + (4 B label + 8 B belonging) per entry of
                # the neighbour's label set per arc, the row's set written (12 B per entry + size)
                _, _, _, _, sizes, _, _ = copra_run(g, p, want_sets=True, device_graph=dg)
                sbar = float(np.mean(sizes))
                sweep_bytes = g.edge_count * (4 + 12 * sbar) + g.vertex_count * (12 * sbar + 8)
                gbs = sweep_bytes * it / (ms * 1e-3) / 1e9
                line = {"algo": "copra", "metric": "COPRA GTEPS on R-MAT-20 (edge_count x sweeps / time)",
                        "value": g.edge_count * it / (ms * 1e-3) / 1e9, "unit": "GTEPS", "ms_per_run": ms,
                        "iterations": it, "config": {"workload": "rmat20", "max_labels": K, "batches": batches,
                                                     "tolerance": 0.01, "vertices": g.vertex_count,
                                                     "arcs": g.edge_count},
                        "modularity": O.modularity(g, run.best),
                        "communities": int(len(np.unique(run.best))),
                        "roofline": {"bound": "hbm", "achieved": gbs, "peak": PEAK, "unit": "GB/s", "frac": gbs / PEAK,
                                     "bytes_model": "per sweep m (4 + 12 s) + n (12 s + 8), s = mean label-set size "
                                                    f"{sbar:.3f}"}}
                if not args.no_cpu and batches == 0 and K in (1, 8):
                    t0 = time.perf_counter()
                    best, cit, _, _, _ = O.copra(g, max_labels=K, batches=0, tie=1, seed=1, tolerance=0.01,
                                                 max_iterations=20)
                    dt = time.perf_counter() - t0
                    line["cpu"] = {"value": g.edge_count * cit / dt / 1e9, "unit": "GTEPS", "cores": 1,
                                   "kind": "port", "seconds": dt, "same_result": bool(np.array_equal(best, run.best))}
                print(json.dumps(line), flush=True)
        dg.close()
    if args.algo in ("slpa", "all"):
        g = lp.planted_partition(1_000_000, 10_000, seed=1)
        dg = _lib.DeviceGraph(g)
        for batches in (0, 1):
            for T in (10, 20, 50):
                p = lp.SlpaParams(memory_size=T, seed=1, batches=batches)

                def run():
                    labels, it, _, _, st, _ = slpa_run(g, p, want_slots=False, device_graph=dg)
                    run.labels = labels
                    return it, st["kernel_ms"]

                ms, it = timed(run, args.steps, args.warmup)
                # roofline: per speaking round 4 B index + 4 B spoken label per arc, 8 B per vertex
                gbs = (8 * g.edge_count + 8 * g.vertex_count) * it / (ms * 1e-3) / 1e9
                line = {"algo": "slpa", "metric": "SLPA GTEPS on planted-1M (edge_count x rounds / time)",
                        "value": g.edge_count * it / (ms * 1e-3) / 1e9, "unit": "GTEPS", "ms_per_run": ms,
                        "iterations": it, "config": {"workload": "planted1m", "memory_size": T, "batches": batches,
                                                     "tolerance": 0.05, "vertices": g.vertex_count,
                                                     "arcs": g.edge_count},
                        "modularity": O.modularity(g, run.labels),
                        "communities": int(len(np.unique(run.labels))),
                        "roofline": {"bound": "hbm", "achieved": gbs, "peak": PEAK, "unit": "GB/s", "frac": gbs / PEAK,
                                     "bytes_model": "per round 8 m + 8 n (index + spoken label per arc)"}}
                if not args.no_cpu and batches == 0 and T == 20:
                    t0 = time.perf_counter()
                    labels, cit, _, _ = O.slpa(g, memory_size=T, batches=0, tie=1, speaker_rng=1, seed=1,
                                               tolerance=0.05)
                    dt = time.perf_counter() - t0
                    line["cpu"] = {"value": g.edge_count * cit / dt / 1e9, "unit": "GTEPS", "cores": 1,
                                   "kind": "port", "seconds": dt,
                                   "same_result": bool(np.array_equal(labels, run.labels))}
                print(json.dumps(line), flush=True)
        dg.close()


if __name__ == "__main__":
    main()
