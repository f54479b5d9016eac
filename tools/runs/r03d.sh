cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "rank or alternate or shuffle_bit_exact" > gpurun_out/r03d_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r03d_pytest.log
for m in atomic match; do SHUF_RANK_MODE=$m timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-gpu-baselines --e2e-steps 0 > gpurun_out/r03d_bench_$m.json 2>> gpurun_out/r03d_bench.err; done
