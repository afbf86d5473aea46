import sys, os
sys.path.insert(0, "/root/repo")
import paper_2301_09125_b200 as lp
from paper_2301_09125_b200 import _lib
from paper_2301_09125_b200.copra import copra_run
g = lp.rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 20, seed=1)
dg = _lib.DeviceGraph(g)
for K in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["16"])]:
    best, it, _, _, _, st, _ = copra_run(g, lp.CopraParams(max_labels=K, max_iterations=20, seed=1), want_sets=False, device_graph=dg)
    print("K", K, "it", it, "ms", st["kernel_ms"], flush=True)
