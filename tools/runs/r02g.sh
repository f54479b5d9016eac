cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02g_par.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02g_hot.json 2> gpurun_out/r02g_hot.err
SHUF_DBG=4 python tools/ktime.py hot > gpurun_out/r02g_dbg4.log 2>&1
SHUF_DBG=12 python tools/ktime.py hot > gpurun_out/r02g_dbg12.log 2>&1
