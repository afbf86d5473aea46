"""Per-kernel time split of one COPRA / SLPA run (LP_RAK_PROFILE).

    python scripts/prof_mlp.py copra|slpa [K|T] [batches] [scale]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2301_09125_b200 as lp  # noqa: E402
from paper_2301_09125_b200 import _lib  # noqa: E402
from paper_2301_09125_b200.copra import copra_run  # noqa: E402
from paper_2301_09125_b200.slpa import slpa_run  # noqa: E402

algo = sys.argv[1]
par = int(sys.argv[2]) if len(sys.argv) > 2 else 8
batches = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if algo == "copra":
    g = lp.rmat(int(sys.argv[4]) if len(sys.argv) > 4 else 20, seed=1)
    dg = _lib.DeviceGraph(g)
    for r in range(2):
        best, it, _, _, _, st, ch = copra_run(g, lp.CopraParams(max_labels=par, max_iterations=20, seed=1,
                                                                 batches=batches), want_sets=False, profile=True,
                                              device_graph=dg)
        print(f"copra K={par} B={batches}: it {it} rounds {st['rounds']} kernel_ms {st['kernel_ms']:.2f} "
              f"tier0_ms {st['bin_ms'][2]:.2f} tier1_ms {st['bin_ms'][1]:.2f} team_ms {st['bin_ms'][0]:.2f} aux_ms {st['aux_ms']:.2f} "
              f"launches {st['bin_launches']} changed {ch.tolist()}")
else:
    g = lp.planted_partition(1_000_000, 10_000, seed=1)
    dg = _lib.DeviceGraph(g)
    for r in range(2):
        labels, it, _, _, st, rep = slpa_run(g, lp.SlpaParams(memory_size=par, seed=1, batches=batches),
                                             want_slots=False, profile=True, device_graph=dg)
        print(f"slpa T={par} B={batches}: it {it} rounds {st['rounds']} kernel_ms {st['kernel_ms']:.2f} "
              f"bin_ms {[round(x, 2) for x in st['bin_ms']]} gather_ms {st['gather_ms']:.2f} aux {st['aux_ms']:.2f} "
              f"repeats {rep.tolist()}")
