#!/bin/bash
# Compare library variants on the NIPS bench: bash scripts/gpu_variants.sh TAG lib1.so lib2.so ...
mkdir -p gpurun_out
TAG=$1; shift
for lib in "$@"; do
  n=$(basename $lib .so)
  BNMC_GPU_LIB=$PWD/$lib timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bv_${TAG}_$n.json 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/bv_${TAG}_$n.json').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],4), d['phases_ms'])" || tail -5 gpurun_out/bv_${TAG}_$n.json
done
