#!/bin/bash
# One `ncu --set full` capture of the small per-sweep kernels (NIPS workload).
# usage: bash scripts/gpu_ncu_small.sh TAG [kernel-regex]
set -x
TAG=${1:-small}
RE=${2:-"wterm|colsum|zfallback"}
CNT=${3:-3}
mkdir -p gpurun_out
python -m paper_1312_3613_b200.build >/dev/null
BNMC_PDL=0 ncu --set full --clock-control none --cache-control none --import-source on -k "regex:$RE" -c $CNT \
    -o gpurun_out/${TAG} -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}.log 2>&1
tail -3 gpurun_out/${TAG}.log
