cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_elemsize.py -x -q > gpurun_out/r02i_elem.log 2>&1
python tools/sweep.py 28 5 > gpurun_out/r02i_sweep.jsonl 2> gpurun_out/r02i_sweep.err
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02i_hot.json 2> gpurun_out/r02i_hot.err
