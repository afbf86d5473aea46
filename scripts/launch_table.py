"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
seq = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("lp::", "")
            seq.append((name, float(d["Metric Value"].replace(",", "")) / 1000.0))
tot = OrderedDict()
for name, us in seq:
    tot[name] = tot.get(name, 0.0) + us
print("launches", len(seq), "total_us", round(sum(us for _, us in seq), 1))
for name, us in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{us:10.1f} us  {name}")
if len(sys.argv) > 2:
    for name, us in seq:
        print(f"{us:9.1f}  {name}")
