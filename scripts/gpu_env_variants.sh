#!/bin/bash
# Compare env-selected variants on a bench workload:
#   bash scripts/gpu_env_variants.sh TAG WORKLOAD SPEC SPEC ...
# SPEC = "-" (defaults) or comma-separated VAR=val assignments.
mkdir -p gpurun_out
TAG=$1; WL=$2; shift 2
for spec in "$@"; do
  n=$(echo "$spec" | tr '=/, ' '____')
  if [ "$spec" = "-" ]; then envs=""; else envs="${spec//,/ }"; fi
  env $envs timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --workload $WL > "gpurun_out/be_${TAG}_${WL}_$n.json" 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/be_${TAG}_${WL}_$n.json').read().strip().splitlines()[-1]); print('$spec', round(d['ms_per_step'],4), d['phases_ms'])" || tail -n 5 "gpurun_out/be_${TAG}_${WL}_$n.json"
done
