# compute-sanitizer over the small-corpus GPU parity tests (memcheck) and small sweeps of the
# kernels with shared-memory handoffs (racecheck).
#   bash scripts/gpu_sanitize.sh   -> gpurun_out/t15*.txt, gpurun_out/t16*.txt
export BNMC_SPECULATE=1
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --log-file gpurun_out/t15_memcheck.txt python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -q -x -k "lda_sweeps_vs_reference or layouts_vs_restatement and (K1- or K5- or K100- or K513-) or sharded_lda_vs_reference_goldens or zoo_sweeps or gmm_sweeps or mh_" > gpurun_out/t15.log 2>&1; echo "exit $?" >> gpurun_out/t15.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 --log-file gpurun_out/t15_racecheck.txt python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lda_sweeps_vs_reference and False-lda_desk" > gpurun_out/t15b.log 2>&1; echo "exit $?" >> gpurun_out/t15b.log
# r02 additions: word-major z-step (sort, warp units, staged fallback), segmented prior rows,
# running-sum topic picks, chunked HMM scans
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --log-file gpurun_out/t16_memcheck.txt python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -q -x -k "word_major and (k150 or k300 or K300) or long_rows and v2048 or running_sums and k7 or hmm_prior_chain and s17 or hmm_chunked and s64 or exact_weights_screen and k300" > gpurun_out/t16.log 2>&1; echo "exit $?" >> gpurun_out/t16.log
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 9 --log-file gpurun_out/t16_racecheck.txt python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "word_major and (k150 or k300) or hmm_chunked and s64 or running_sums and k7 or exact_weights_screen and k100-all" > gpurun_out/t16b.log 2>&1; echo "exit $?" >> gpurun_out/t16b.log
