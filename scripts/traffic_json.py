"""profiles/ncu_traffic.json from an ncu --csv launch list (dram__bytes_read.sum
+ dram__bytes_write.sum per launch, averaged per bench.py kernel group).

    python scripts/traffic_json.py launches.csv [config] > profiles/ncu_traffic.json
"""
import csv
import json
import sys
from collections import OrderedDict, defaultdict


def group(name):
    if name.startswith("k_warp"):
        return "tally_warp"
    if name.startswith("k_team"):
        return "tally_hub" if "1024" in name else "tally_team"
    if name.startswith("k_small") or name.startswith("k_first_round") or name.startswith("k_mid"):
        return "tally_small"
    if name.startswith("k_gather"):
        return "k_gather"
    return None


rows = list(csv.reader(open(sys.argv[1])))
cfg = sys.argv[2] if len(sys.argv) > 2 else "rmat22"
hdr = None
launch = OrderedDict()
for r in rows:
    if "Kernel Name" in r and "Metric Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("lp::", "")
        rec = launch.setdefault(d["ID"], {"name": name})
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        if d["Metric Name"].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            rec["dram"] = rec.get("dram", 0.0) + v
acc = defaultdict(list)
for rec in launch.values():
    g = group(rec["name"])
    if g and "dram" in rec:
        acc[g].append(rec["dram"])
out = {"_note": "DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch, averaged over the launches "
                "of one bench run under ncu (cold-cache serialised launches, " + sys.argv[1].split("/")[-1] +
                "); keys = bench.py kernel_table names",
       cfg: {k: sum(v) / len(v) for k, v in acc.items()}}
print(json.dumps(out, indent=1))
