cd $GRAFT_REPO_ROOT
bash tools/gpu_round.sh r01r tests bench launches full
tail -3 gpurun_out/r01r_pytest_gpu.log; grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*\|"kernel": "[a-z]*"' gpurun_out/r01r_bench.json; tail -2 gpurun_out/r01r_bench.err; tail -2 gpurun_out/r01r_ncu_full.log
