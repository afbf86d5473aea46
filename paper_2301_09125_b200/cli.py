"""Command-line front end: detect, sweep, info.

Mirrors the reference's `labelprop detect / sweep / info` (`labelprop/cli.py:
74-249`) on the CUDA detectors.  File loaders (MatrixMarket, edge lists) are
out of scope here, so a graph is named by a spec:

    rmat:SCALE[:SEED]          seeded R-MAT (a,b,c,d = .57,.19,.19,.05), unit weights
    rmatw:SCALE[:SEED]         the same with float32 weights U[1,2)
    planted:N:COMMUNITIES[:SEED]
    grid:SIDE[:SEED]           road-like grid (BASELINE config 2)
    PATH.npz                   a CSR saved with offsets / neighbors [/ weights] arrays

`detect` writes `vertex<TAB>community` (stdout or --output) and the
reference's one-line summary on stderr; `sweep` streams the reference's CSV
(`--extended` adds batches, edges scanned and GTEPS).  `--batches` selects
the schedule (0 = the reference's visit order, 1 = synchronous).
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from . import synth
from .graph import Graph, undirected_csr
from .sweep import (CSV_HEADER, CSV_HEADER_EXTENDED, DEFAULT_MAX_LABELS, DEFAULT_MEMORY_SIZES, DEFAULT_TOLERANCES,
                    ALGORITHMS, SweepSpec, run_one, run_sweep)


def load_spec(spec: str) -> Graph:
    """A graph from a generator spec or an .npz CSR (see the module doc)."""
    if spec.endswith(".npz"):
        z = np.load(spec)
        off, nbr = z["offsets"].astype(np.int64), z["neighbors"].astype(np.int64)
        n = len(off) - 1
        u = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
        w = z["weights"] if "weights" in z else None
        return undirected_csr(n, u, nbr, w)
    kind, *rest = spec.split(":")
    nums = [int(x) for x in rest]
    if kind in ("rmat", "rmatw") and 1 <= len(nums) <= 2:
        return synth.rmat(nums[0], seed=nums[1] if len(nums) > 1 else 1, weighted=kind == "rmatw")
    if kind == "planted" and 2 <= len(nums) <= 3:
        return synth.planted_partition(nums[0], nums[1], seed=nums[2] if len(nums) > 2 else 1)
    if kind == "grid" and 1 <= len(nums) <= 2:
        return synth.road_grid(nums[0], seed=nums[1] if len(nums) > 1 else 1)
    raise ValueError(f"unknown graph spec {spec!r}")


def _tuple(cast):
    return lambda text: tuple(cast(x) for x in text.split(",") if x)


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2301_09125_b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="command", required=True)
    d = sub.add_parser("detect", help="one detection; vertex<TAB>community out")
    d.add_argument("--graph", required=True)
    d.add_argument("--algorithm", choices=ALGORITHMS, required=True)
    d.add_argument("--strict", action="store_true", help="scan-first ties (default: random ties)")
    d.add_argument("--tolerance", type=float, default=None)
    d.add_argument("--max-labels", type=int, default=8)
    d.add_argument("--memory-size", type=int, default=20)
    d.add_argument("--max-iterations", type=int, default=100)
    d.add_argument("--batches", type=int, default=0)
    d.add_argument("--seed", type=int, default=1)
    d.add_argument("--output", default="-")
    s = sub.add_parser("sweep", help="parameter sweep; CSV out")
    s.add_argument("--algorithm", choices=ALGORITHMS, required=True)
    s.add_argument("--graph", nargs="+", required=True)
    s.add_argument("--tolerances", type=_tuple(float), default=DEFAULT_TOLERANCES)
    s.add_argument("--max-labels-grid", type=_tuple(int), default=DEFAULT_MAX_LABELS)
    s.add_argument("--memory-sizes", type=_tuple(int), default=DEFAULT_MEMORY_SIZES)
    s.add_argument("--modes", type=_tuple(str), default=("strict", "non-strict"))
    s.add_argument("--batches-grid", type=_tuple(int), default=(0,))
    s.add_argument("--repetitions", type=int, default=1)
    s.add_argument("--seed", type=int, default=1)
    s.add_argument("--extended", action="store_true", help="add batches, edges_scanned, gteps columns")
    s.add_argument("--output", default="-")
    i = sub.add_parser("info", help="vertices / edges / average degree per graph")
    i.add_argument("graph", nargs="+")
    return ap


def _open(path):
    return sys.stdout if path == "-" else open(path, "w")


def cmd_detect(args) -> int:
    g = load_spec(args.graph)
    res = run_one(args.algorithm, g, mode="strict" if args.strict else "non-strict", tolerance=args.tolerance,
                  max_labels=args.max_labels, memory_size=args.memory_size, max_iterations=args.max_iterations,
                  seed=args.seed, batches=args.batches)
    out = _open(args.output)
    try:
        out.write("".join(f"{v}\t{c}\n" for v, c in enumerate(np.asarray(res.assignment).tolist())))
    finally:
        if out is not sys.stdout:
            out.close()
    print(f"vertices={g.vertex_count} iterations={res.iterations} elapsed_ms={res.elapsed * 1e3:.3f} "
          f"modularity={res.modularity:.6f}", file=sys.stderr)
    return 0


def cmd_sweep(args) -> int:
    spec = SweepSpec(args.algorithm, tolerances=args.tolerances, max_labels=args.max_labels_grid,
                     memory_sizes=args.memory_sizes, modes=args.modes, repetitions=args.repetitions, seed=args.seed,
                     batches=args.batches_grid)
    out = _open(args.output)
    try:
        print(CSV_HEADER_EXTENDED if args.extended else CSV_HEADER, file=out, flush=True)
        for rec in run_sweep(spec, [(name, load_spec(name)) for name in args.graph]):
            print(rec.csv_row(extended=args.extended), file=out, flush=True)
    finally:
        if out is not sys.stdout:
            out.close()
    return 0


def cmd_info(args) -> int:
    print("graph\tvertices\tedges\tavg_degree")
    for name in args.graph:
        g = load_spec(name)
        print(f"{name}\t{g.vertex_count}\t{g.edge_count}\t{g.edge_count / max(g.vertex_count, 1):.2f}")
    return 0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return {"detect": cmd_detect, "sweep": cmd_sweep, "info": cmd_info}[args.command](args)
    except ValueError as exc:
        print(f"paper_2301_09125_b200: {exc}", file=sys.stderr)
        return 2
