cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02y_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r02y_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02y_pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err
timeout 600 python bench.py --mode ipsc --steps 3 --warmup 3 --no-cpu-baseline --no-gpu-baselines > gpurun_out/r02y_bench_ipsc.json 2>> gpurun_out/r02y_bench.err
timeout 600 python bench.py --mode inplace --steps 5 --warmup 3 --no-cpu-baseline --no-gpu-baselines > gpurun_out/r02y_bench_inplace.json 2>> gpurun_out/r02y_bench.err
