cd $GRAFT_REPO_ROOT
bash tools/gpu_round.sh r01n tests bench launches full
tail -3 gpurun_out/r01n_pytest_gpu.log; cat gpurun_out/r01n_bench.json | head -c 3000; tail -2 gpurun_out/r01n_bench.err
