#!/bin/bash
# One GPU round trip: parity tests, bench, launch list, full ncu captures.
# usage (under gpurun): bash scripts/gpu_check.sh [tag]
mkdir -p gpurun_out
TAG=${1:-run}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_$TAG.log
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_nips_$TAG.json 2> gpurun_out/bench_nips_$TAG.err
BNMC_ZSTEP_THETA=regs timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_nips_regs_$TAG.json 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --workload kos > gpurun_out/bench_kos_$TAG.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zscreen -s 4 -c 1 -o gpurun_out/zscreen_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
cat gpurun_out/pytest_gpu_$TAG.log; cat gpurun_out/bench_nips_$TAG.json gpurun_out/bench_nips_regs_$TAG.json gpurun_out/bench_kos_$TAG.json | cut -c1-900
