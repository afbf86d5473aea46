"""Per-launch listing of the last detection in an ncu --csv launch list
(gpu__time_duration.sum, dram bytes, L2 hit rate; serialised, cold-cache).

    python scripts/launch_rounds.py launches.csv [marker-kernel]
"""
import collections
import csv
import sys

path = sys.argv[1]
marker = sys.argv[2] if len(sys.argv) > 2 else "k_init_labels"
hdr, L = None, collections.OrderedDict()
for r in csv.reader(open(path)):
    if "Kernel Name" in r and "Metric Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        rec = L.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0].replace("void ", "").replace("lp::", "")})
        try:
            rec[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            pass
recs = list(L.values())
starts = [i for i, r in enumerate(recs) if r["name"].startswith(marker)]
last = recs[starts[-1]:] if starts else recs
tot_us = tot_mb = 0.0
for r in last:
    t = r.get("gpu__time_duration.sum", 0) / 1e3
    mb = (r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)) / 1e6
    tot_us += t
    tot_mb += mb
    print(f"{t:8.1f} us {mb:8.1f} MB  L2 hit {r.get('lts__t_sector_hit_rate.pct', 0):5.1f}%  {r['name'][:70]}")
print(f"total {tot_us:.1f} us, {tot_mb:.1f} MB DRAM, {len(last)} launches")
