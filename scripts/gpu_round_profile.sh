# One GPU call: default bench line + reference arm + ncu captures for profiles/.
#   bash scripts/gpu_round_profile.sh TAG
# ncu reports are reduced to CSV pages on the box (gpurun returns <= 64 MiB).
T=${1:-r02}
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/${T}_ref.json 2> $O/${T}_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-1b > /dev/null 2>&1
cap() {  # name, regex, extra bench args
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$2 -s ${4:-5} -c 1 -o /tmp/${T}_$1 -f \
    python bench.py $3 --no-cpu-baseline --no-1b > /dev/null 2>&1
  ncu -i /tmp/${T}_$1.ncu-rep --page raw --csv > $O/${T}_$1_raw.csv 2>/dev/null
  ncu -i /tmp/${T}_$1.ncu-rep --page source --csv --print-source sass > $O/${T}_$1_sass.csv 2>/dev/null
  rm -f /tmp/${T}_$1.ncu-rep
}
for k in zscreen_t phi_pool phi_colsum2 wterm zfallback; do cap nips_$k $k "--steps 3 --warmup 3"; done
cap 1b_zscreen zscreen_kernel "--workload 1b --steps 1 --warmup 3" 1
du -sh $O
