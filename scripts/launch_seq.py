"""Per-round kernel durations from an ncu --csv launch list of one RAK
detection: sweep kernels in launch order, grouped at each phase-1 gather.

    python scripts/launch_seq.py launches.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
seq = []
for r in rows:
    if "Kernel Name" in r and "Metric Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("lp::", "")
        us = float(d["Metric Value"].replace(",", "")) / (1000.0 if d["Metric Unit"] == "nsecond" else 1.0)
        seq.append((name, us))
# keep from the first k_first_round on
start = next((i for i, (n, _) in enumerate(seq) if n.startswith("k_first_round")), 0)
seq = seq[start:]
groups, cur = [], []
for n, us in seq:
    if n.startswith("k_gather") and cur:
        groups.append(cur)
        cur = []
    cur.append((n, us))
groups.append(cur)
tot = 0.0
for g in groups:
    t = sum(us for _, us in g)
    tot += t
    big = sorted(g, key=lambda x: -x[1])[:6]
    print(f"{t:8.1f} us | " + "  ".join(f"{n[:22]} {us:.0f}" for n, us in big))
print(f"total {tot:.1f} us over {len(seq)} launches")
