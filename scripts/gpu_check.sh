#!/bin/bash
# One GPU round trip: parity tests, bench (NIPS + KOS + 1B + GMM + logreg), launch list,
# full ncu captures of the z-step and phi-block kernels.
# usage (under gpurun): bash scripts/gpu_check.sh TAG
mkdir -p gpurun_out
TAG=${1:-run}
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu_$TAG.log
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_nips_$TAG.json 2> gpurun_out/bench_nips_$TAG.err
timeout 300 python bench.py --steps 50 --warmup 5 --workload kos > gpurun_out/bench_kos_$TAG.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --workload gmm > gpurun_out/bench_gmm_$TAG.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --workload logreg > gpurun_out/bench_logreg_$TAG.json 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --workload 1b --no-cpu-baseline > gpurun_out/bench_1b_$TAG.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 300 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zscreen -s 4 -c 1 -o gpurun_out/zstep_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:phi_gamma -s 4 -c 1 -o gpurun_out/phigamma_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full2_$TAG.log 2>&1
cat gpurun_out/pytest_gpu_$TAG.log
for w in nips kos gmm logreg 1b; do python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/bench_${w}_$TAG.json').read().strip().splitlines()[-1]); print('$w', d['ms_per_step'], d['value'], d.get('e2e',{}).get('value'))
except Exception as e: print('$w FAILED', e)"; done
