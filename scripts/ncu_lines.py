"""Per-CUDA-source-line stall attribution of an ncu report (needs -lineinfo).
python scripts/ncu_lines.py rep.ncu-rep [top] [kernel-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ksub = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
recs = []
cur_file, cur_fn, hdr = None, None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        cur_fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].strip().isdigit():
        d = dict(zip(hdr, r))
        d["file"] = cur_file
        d["fn"] = cur_fn
        recs.append(d)
key = "Warp Stall Sampling (All Samples)"
fns = []
for d in recs:
    if d["fn"] not in fns:
        fns.append(d["fn"])
for fn in fns:
    if ksub and ksub not in (fn or ""):
        continue
    sel = [d for d in recs if d["fn"] == fn]
    tot = sum(float(d.get(key) or 0) for d in sel) or 1
    inst = sum(float(d.get("Instructions Executed") or 0) for d in sel)
    print("==", (fn or "?")[:90], "samples", tot, "warp-inst", inst)
    for d in sorted(sel, key=lambda d: -float(d.get(key) or 0))[:top]:
        print(f"{float(d[key]) / tot * 100:5.1f}% inst={float(d.get('Instructions Executed') or 0) / max(inst, 1) * 100:5.1f}% "
              f"{d['file']}:{d['Line No']:>5} {d['Source'].strip()[:90]}")

if "--by-inst" in sys.argv:
    for fn in fns:
        if ksub and ksub not in (fn or ""):
            continue
        sel = [d for d in recs if d["fn"] == fn]
        inst = sum(float(d.get("Instructions Executed") or 0) for d in sel)
        print("== by instructions", (fn or "?")[:80])
        for d in sorted(sel, key=lambda d: -float(d.get("Instructions Executed") or 0))[:top]:
            print(f"inst={float(d.get('Instructions Executed') or 0) / max(inst, 1) * 100:5.1f}% "
                  f"{d['file']}:{d['Line No']:>5}")
