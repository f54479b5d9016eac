cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02d_par.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02d_hot.json 2> gpurun_out/r02d_hot.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "hot or c1 or c2" > gpurun_out/r02d_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_finish_fast" -c 1 \
      -o gpurun_out/r02d_fin python tools/prof_run.py hot > gpurun_out/r02d_ncu.log 2>&1
