# compute-sanitizer over the small-corpus GPU parity tests (memcheck) and one LDA sweep test (racecheck).
#   bash scripts/gpu_sanitize.sh   -> gpurun_out/t15*.txt
export BNMC_SPECULATE=1
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --log-file gpurun_out/t15_memcheck.txt python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -q -x -k "lda_sweeps_vs_reference or layouts_vs_restatement and (K1- or K5- or K100- or K513-) or sharded_lda_vs_reference_goldens or zoo_sweeps or gmm_sweeps or mh_" > gpurun_out/t15.log 2>&1; echo "exit $?" >> gpurun_out/t15.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 --log-file gpurun_out/t15_racecheck.txt python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lda_sweeps_vs_reference and False-lda_desk" > gpurun_out/t15b.log 2>&1; echo "exit $?" >> gpurun_out/t15b.log
