"""Key metrics per kernel from `ncu -i rep --page details --csv` output.

    python scripts/ncu_summary.py details.csv
"""
import csv
import sys
from collections import OrderedDict

WANT = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "Memory Throughput"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("GPU Speed Of Light Throughput", "L2 Cache Throughput"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Memory Workload Analysis", "L1/TEX Hit Rate"),
    ("Memory Workload Analysis", "Mem Busy"),
    ("GPU Speed Of Light Throughput", "L1/TEX Cache Throughput"),
    ("Scheduler Statistics", "Eligible Warps Per Scheduler"),
    ("Scheduler Statistics", "Active Warps Per Scheduler"),
    ("Scheduler Statistics", "No Eligible"),
    ("Occupancy", "Achieved Occupancy"),
    ("Occupancy", "Theoretical Occupancy"),
    ("Compute Workload Analysis", "Issue Slots Busy"),
    ("Compute Workload Analysis", "Executed Ipc Active"),
    ("Warp State Statistics", "Avg. Active Threads Per Warp"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Block Size"),
]
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
ker = OrderedDict()
for r in rows[1:]:
    if len(r) < 15:
        continue
    d = dict(zip(hdr, r))
    k = (d["ID"], d["Kernel Name"].split("(")[0].replace("void ", "").replace("lp::", ""))
    d["Section Name"] = d["Section Name"].strip()
    ker.setdefault(k, {})[(d["Section Name"], d["Metric Name"])] = (d["Metric Value"], d["Metric Unit"])
for (kid, name), m in ker.items():
    print(f"== launch {kid}: {name}")
    for key in WANT:
        if key in m:
            v, u = m[key]
            print(f"   {key[1]:<38} {v:>12} {u}")
