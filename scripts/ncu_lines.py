#!/usr/bin/env python
"""Per-source-line instruction / stall-sample attribution of one ncu report:
    python scripts/ncu_lines.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
hdr = None
agg = defaultdict(lambda: [0, 0])
src = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    key = (cur, r[0])
    agg[key][0] += ie
    agg[key][1] += ss
    src[key] = r[1][:100]
tot = sum(v[0] for v in agg.values()) or 1
st = sum(v[1] for v in agg.values()) or 1
print(f"total instructions {tot}, stall samples {st}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]:10s}:{k[1]:5s} inst {v[0]/tot*100:5.1f}% stall {v[1]/st*100:5.1f}%  {src[k]}")
