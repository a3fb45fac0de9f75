#!/usr/bin/env python
"""Hottest SASS lines (warp-stall samples) of one kernel in an ncu report.

    python scripts/ncu_sass_hot.py <report.ncu-rep> <kernel-regex> [N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
h = rows[hi]
ia, iss, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = [r for r in rows[hi + 1:] if len(r) > ie and r[iss].isdigit()]
tot = sum(int(r[iss]) for r in body) or 1
print(f"{len(body)} SASS lines, {tot} stall samples")
for r in sorted(body, key=lambda r: -int(r[iss]))[:n]:
    print(f"{int(r[iss]) / tot * 100:5.1f}%  {r[0]:>6s}  exec {r[ie]:>8s}  {r[ia][:90]}")
