# Bench lines of every workload (one GPU), for profiles/ and DESIGN.md section 5.
#   bash scripts/gpu_all_workloads.sh TAG
T=${1:-r02}
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/${T}_bench_nips.json 2> $O/${T}_bench_nips.err
for w in kos gmm logreg; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > $O/${T}_bench_$w.json 2> $O/${T}_bench_$w.err
done
timeout 900 python bench.py --workload 1b --steps 3 --warmup 3 --no-cpu-baseline > $O/${T}_bench_1b.json 2> $O/${T}_bench_1b.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/${T}_ref_nips.json 2> $O/${T}_ref_nips.err
