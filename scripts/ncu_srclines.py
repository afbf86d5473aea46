"""Hot CUDA source lines (warp-stall samples) per kernel of an ncu report.

    python scripts/ncu_srclines.py rep.ncu-rep [function-substring] [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
path, func, hdr = None, None, None
acc = defaultdict(lambda: [0.0, 0.0, ""])
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        path = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        func = row[1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0].strip().isdigit():
        continue
    if want and want not in (func or ""):
        continue
    d = dict(zip(hdr[:5], row[:5]))
    try:
        samples = float(row[4])
        inst = float(row[7]) if row[7] not in ("-", "") else 0.0
    except (ValueError, IndexError):
        continue
    key = (func, path, int(row[0]))
    acc[key][0] += samples
    acc[key][1] += inst
    acc[key][2] = row[1]
by_func = defaultdict(list)
for (f, p, ln), (smp, inst, src) in acc.items():
    by_func[f].append((smp, inst, p, ln, src))
for f, rows in by_func.items():
    tot = sum(r[0] for r in rows) or 1.0
    print(f"== {f}: {int(tot)} samples")
    for smp, inst, p, ln, src in sorted(rows, reverse=True)[:top]:
        print(f"{100 * smp / tot:5.1f}% inst={int(inst):>11} {p}:{ln}  {src.strip()[:90]}")
