cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02c_par.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02c_hot.json 2> gpurun_out/r02c_hot.err
python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02c_c3.json 2> gpurun_out/r02c_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter" -c 1 \
      -o gpurun_out/r02c_sc python tools/prof_run.py hot > gpurun_out/r02c_ncu.log 2>&1
