cd $GRAFT_REPO_ROOT
bash tools/gpu_round.sh r01s tests bench launches full
tail -3 gpurun_out/r01s_pytest_gpu.log; grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*\|"kernel": "[a-z]*"' gpurun_out/r01s_bench.json; tail -2 gpurun_out/r01s_bench.err; tail -1 gpurun_out/r01s_ncu_full.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
