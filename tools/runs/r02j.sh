cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02j_par.log 2>&1
python tools/kprof.py 268435456 16 256 4096 > gpurun_out/r02j_kp16.log 2>&1
python tools/sweep.py 28 5 > gpurun_out/r02j_sweep.jsonl 2> gpurun_out/r02j_sweep.err
