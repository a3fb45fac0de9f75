#!/usr/bin/env python
"""Summarise gpurun_out/ profiler output into tracked files under profiles/.

    python scripts/summarize_profiles.py launches <launches.csv> <out.txt> [--title T]
    python scripts/summarize_profiles.py full <kernel.ncu-rep> <out.txt> [--traffic-key NAME]
    python scripts/summarize_profiles.py csv <raw.csv> <sass.csv> <out.txt> [--traffic-key NAME]

`launches`: the `ncu --metrics gpu__time_duration.sum --clock-control none` launch list
-> per-kernel count / mean / share of the per-sweep kernel time.
`csv`: the same from the `--page raw --csv` / `--page source --csv --print-source sass`
exports of a capture (scripts/gpu_round_profile.sh reduces reports to these on the box).
`full`: one `ncu --set full` capture -> the metrics the roofline and DESIGN.md cite
(duration, dram bytes, L2/L1 throughput, occupancy, issue, stall reasons, top SASS
opcodes); with --traffic-key, dram read+write bytes per launch are also written to
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name: str) -> str:
    name = re.sub(r"\(.*\)$", "", name.strip())
    name = name.replace("bnmc_gpu::<unnamed>::", "").replace("void ", "")
    return name


def launches(src, dst, title):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    h = rows[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = collections.OrderedDict()
    for r in rows[1:]:
        v = float(r[iv].replace(",", ""))
        v = v / 1e3 if r[iu] == "ns" else (v if r[iu] == "us" else v * 1e3)
        per.setdefault(short(r[ik]), []).append(v)
    tot = sum(sum(v) for v in per.values())
    lines = [f"# {title}", "# count  mean_us  total_us  share  kernel"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{len(v):7d} {sum(v)/len(v):8.2f} {sum(v):9.1f} {sum(v)/tot*100:5.1f}%  {k}")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__t_bytes.sum",
    "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
]


def to_bytes(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit)
    return float(v) * f if f else None


def to_us(v, unit):
    f = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
         "second": 1e6, "s": 1e6}.get(unit)
    try:
        return round(float(v) * f, 2) if f else None
    except (TypeError, ValueError):
        return None


def full(rep, dst, key, raw=None, src=None, source_name=None):
    if raw is None:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = []
    traffic = []
    for d in rows[2:]:
        m = dict(zip(h, d))
        un = dict(zip(h, u))
        out.append(f"kernel: {short(m.get('Kernel Name', '?'))}")
        for k in WANT:
            if k in m:
                out.append(f"  {k:62s} {m[k]:>16s} {un.get(k, '')}")
        stalls = {k.split("stalled_")[1].split("_per_issue")[0]: float(m[k]) for k in h
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                  and m.get(k)}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
        out.append("  stalls (warps per issue): " + ", ".join(f"{k} {v:.2f}" for k, v in top))
        rb = to_bytes(m.get("dram__bytes_read.sum", 0), un.get("dram__bytes_read.sum"))
        wb = to_bytes(m.get("dram__bytes_write.sum", 0), un.get("dram__bytes_write.sum"))
        if rb is not None and wb is not None:
            def pct(k):
                try:
                    return round(float(m[k]), 2)
                except (KeyError, ValueError):
                    return None
            traffic.append({"dram_bytes": rb + wb,
                            "l1tex_pct": pct("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                            "lts_pct": pct("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                            "issue_pct": pct("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
                            "dram_pct": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                            "kernel_us_ncu": to_us(m.get("gpu__time_duration.sum"), un.get("gpu__time_duration.sum")),
                            "source": os.path.relpath(dst, ROOT)})
            out.append(f"  dram read+write bytes per launch: {rb + wb:.4g}")
    # SASS opcode mix (instructions executed)
    if src is None:
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2 and "Source" in srows[1]:
        sh = srows[1]
        ia, ie = sh.index("Source"), sh.index("Instructions Executed")
        c = collections.Counter()
        for r in srows[2:]:
            if len(r) <= max(ia, ie) or not r[ie].isdigit():
                continue
            toks = r[ia].strip().split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            c[op.split(".")[0]] += int(r[ie] or 0)
        tot = sum(c.values())
        out.append(f"  SASS instructions executed: {tot}; top opcodes: " +
                   ", ".join(f"{k} {v/tot*100:.1f}%" for k, v in c.most_common(12)))
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))
    if key and traffic:
        p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        cur = {}
        if os.path.exists(p):
            cur = json.load(open(p))
        cur[key] = traffic[0]
        json.dump(cur, open(p, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "csv":
        key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
        full(None, sys.argv[4], key, raw=open(sys.argv[2]).read(), src=open(sys.argv[3]).read())
    elif mode == "launches":
        title = sys.argv[sys.argv.index("--title") + 1] if "--title" in sys.argv else "ncu launch list"
        launches(sys.argv[2], sys.argv[3], title)
    else:
        key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
        full(sys.argv[2], sys.argv[3], key)
