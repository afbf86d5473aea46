"""SURVEY §8 d6 table from ncu_summary.py outputs: per tally / gather kernel
(= degree bin) the duration, DRAM throughput, L2 hit rate, achieved occupancy
and active threads per warp (warp execution efficiency = threads / 32).

    python scripts/degree_bins.py profiles/r2b_ncu_full_summary_rmat22.txt [...]
"""
import re
import sys

BIN = {"k_first_round": "first round (all rows)", "k_small<0, 0, 16>": "d 9-16 (thread/row)",
       "k_small<0, 0, 8>": "d 5-8 (thread/row)", "k_small<0, 0, 4>": "d 2-4 (thread/row)",
       "k_midh": "d 17-64 (thread/row hash)", "k_gather_dense": "phase-1 gather (d > 16)",
       "k_warp<0, 0, 0": "d 65-2048 (warp/row)", "k_warp<0, 0, 1": "d <= 8192 (warp/row, big table)",
       "k_team<0, 0, 256": "team 8 warps (d <= 16K)", "k_team<0, 0, 512": "team 16 warps",
       "k_team<0, 0, 1024": "hubs (32 warps / partition)"}
KEYS = ["Duration", "DRAM Throughput", "L2 Hit Rate", "Achieved Occupancy", "Avg. Active Threads Per Warp"]
for path in sys.argv[1:]:
    print(f"== {path}")
    print(f"{'kernel':34s} {'bin':32s} {'us':>8s} {'DRAM%':>6s} {'L2hit%':>7s} {'occ%':>6s} {'thr/warp':>8s} {'eff':>5s}")
    cur, vals = None, {}

    def flush():
        if cur is None:
            return
        b = next((v for k, v in BIN.items() if cur.startswith(k)), "")
        dur = vals.get("Duration", "")
        thr = vals.get("Avg. Active Threads Per Warp", "0")
        try:
            eff = f"{float(thr) / 32:.2f}"
        except ValueError:
            eff = ""
        print(f"{cur[:34]:34s} {b:32s} {dur:>8s} {vals.get('DRAM Throughput', ''):>6s} "
              f"{vals.get('L2 Hit Rate', ''):>7s} {vals.get('Achieved Occupancy', ''):>6s} {thr:>8s} {eff:>5s}")

    for line in open(path):
        m = re.match(r"== launch \d+: (.*)", line)
        if m:
            flush()
            cur, vals = m.group(1).strip(), {}
            continue
        for k in KEYS:
            if line.strip().startswith(k):
                parts = line.split()
                num = parts[len(k.split())]
                unit = parts[len(k.split()) + 1] if len(parts) > len(k.split()) + 1 else ""
                if k == "Duration" and unit == "ms":
                    num = f"{float(num) * 1e3:.1f}"
                vals[k] = num
    flush()
