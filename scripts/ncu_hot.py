"""Hot SASS lines of an ncu report: python scripts/ncu_hot.py rep.ncu-rep [kernel_index] [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
blk = blocks[idx + 1] if len(blocks) > idx + 1 else blocks[-1]
lines = list(csv.reader(io.StringIO('"Kernel Name"' + blk)))
print(lines[0][:2])
hdr = lines[1]
data = [dict(zip(hdr, r)) for r in lines[2:] if len(r) == len(hdr)]
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(d.get(key) or 0) for d in data) or 1
inst = sum(float(d.get("Instructions Executed") or 0) for d in data)
print("samples", tot, "warp-instructions", inst)
for d in sorted(data, key=lambda d: -float(d.get(key) or 0))[:top]:
    print(f"{float(d[key]) / tot * 100:5.1f}% ex={d.get('Instructions Executed'):>10} {d.get('Source', '')[:100]}")
