#!/usr/bin/env python
"""Per-source-line instruction counts of one kernel: an ncu `--page source --csv
--print-source sass` export joined with `nvdisasm --print-line-info` of the same build.

    python scripts/ncu_line_profile.py <sass.csv> <cubin> <mangled kernel name> [top]
"""
import collections
import csv
import re
import subprocess
import sys

sass_csv, cubin, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4].isdigit() else 30
rows = list(csv.reader(open(sass_csv)))
h = rows[1]
iA, iE, iT = h.index("Address"), h.index("Instructions Executed"), h.index("Thread Instructions Executed")
iW = h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) > iT]
a0 = int(data[0][iA], 16)
execd = {int(r[iA], 16) - a0: (float(r[iE] or 0), float(r[iT] or 0), float(r[iW] or 0)) for r in data}
dis = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
sec = re.search(r"\.text\.%s:(.*?)(?:\n\s*\.section|\Z)" % re.escape(kname), dis, re.S).group(1)
cur = "?"
per = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for line in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', line)
    if m:
        f = m.group(1).split("/")[-1]
        cur = f"{f}:{m.group(2)}" + (f" <- {m.group(3).split('/')[-1]}:{m.group(4)}" if m.group(3) else "")
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m:
        off = int(m.group(1), 16)
        if off in execd:
            per[cur][0] += execd[off][0]
            per[cur][1] += execd[off][1]
            per[cur][2] += execd[off][2]
tot = sum(v[0] for v in per.values())
totw = sum(v[2] for v in per.values()) or 1.0
key = 2 if "--stalls" in sys.argv else 0
print(f"total warp instructions {tot:.0f}, stall samples {totw:.0f}")
print(" inst%  stall%   instructions  thr/inst  line")
for k, (e, t, w) in sorted(per.items(), key=lambda kv: -kv[1][key])[:top]:
    print(f"{e / tot * 100:5.1f}%  {w / totw * 100:5.1f}%  {e:12.0f}  {t / max(e, 1):5.1f}  {k}")
