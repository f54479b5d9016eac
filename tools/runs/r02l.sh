cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/r02l_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02l_pytest.log
timeout 600 python bench.py --mode sharded --steps 5 --warmup 3 > gpurun_out/r02l_bench_sharded.json 2> gpurun_out/r02l_bench_sharded.err
