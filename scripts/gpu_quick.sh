#!/bin/bash
# Quick GPU iteration: NIPS bench (smem + regs theta variants) + one ncu --set full capture.
# usage (under gpurun): bash scripts/gpu_quick.sh TAG [kernel-regex]
mkdir -p gpurun_out
TAG=${1:-q}; KR=${2:-zscreen}
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bq_$TAG.json 2>&1
BNMC_ZSTEP_THETA=regs timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bq_regs_$TAG.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KR -s 4 -c 1 -o gpurun_out/q_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python - <<PY
import json
for f in ["gpurun_out/bq_$TAG.json", "gpurun_out/bq_regs_$TAG.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["phases_ms"])
    except Exception as e:
        print(f, "FAILED", open(f).read()[-2000:])
PY
