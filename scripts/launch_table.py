"""Summarise an ncu --csv launch list (gpu__time_duration.sum, optionally
dram__bytes_read/write.sum and lts__t_sector_hit_rate.pct) per kernel.

    python scripts/launch_table.py launches.csv [all]
"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
launch = OrderedDict()  # (id) -> {name, metrics}
for r in rows:
    if "Kernel Name" in r and "Metric Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = d.get("ID")
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("lp::", "")
        rec = launch.setdefault(key, {"name": name})
        try:
            rec[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            pass

tot = OrderedDict()
for rec in launch.values():
    t = tot.setdefault(rec["name"], {"n": 0, "us": 0.0, "bytes": 0.0, "hit": 0.0})
    t["n"] += 1
    t["us"] += rec.get("gpu__time_duration.sum", 0.0) / 1000.0
    t["bytes"] += rec.get("dram__bytes_read.sum", 0.0) + rec.get("dram__bytes_write.sum", 0.0)
    t["hit"] += rec.get("lts__t_sector_hit_rate.pct", 0.0)
total_us = sum(t["us"] for t in tot.values())
print(f"launches {len(launch)} total_us {total_us:.1f}")
print(f"{'us':>10} {'share':>6} {'n':>5} {'us/launch':>10} {'DRAM MB/launch':>15} {'DRAM GB/s':>10} {'L2 hit%':>8}  kernel")
for name, t in sorted(tot.items(), key=lambda kv: -kv[1]["us"]):
    mb = t["bytes"] / t["n"] / 1e6
    gbs = t["bytes"] / (t["us"] * 1e-6) / 1e9 if t["us"] > 0 else 0.0
    print(f"{t['us']:10.1f} {t['us'] / max(total_us, 1e-9):6.3f} {t['n']:5d} {t['us'] / t['n']:10.1f} {mb:15.2f} "
          f"{gbs:10.1f} {t['hit'] / t['n']:8.1f}  {name}")
if len(sys.argv) > 2:
    for key, rec in launch.items():
        print(f"{rec.get('gpu__time_duration.sum', 0.0) / 1000.0:9.1f}  {rec['name']}")
