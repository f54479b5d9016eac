cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ipsc.py -x -q > gpurun_out/r03g_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r03g_pytest.log
timeout 600 python tools/ipsc_run.py hot --reps 3 > gpurun_out/r03g_plain.log 2>&1
SHUF_DBG=128 timeout 600 python tools/ipsc_run.py hot --reps 1 >> gpurun_out/r03g_plain.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03g_launches.csv python tools/ipsc_run.py hot --reps 1 > gpurun_out/r03g_ncu.log 2>&1
