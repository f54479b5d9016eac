cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bl_plain.json 2>&1; echo plain $?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r01u_bench_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bl_ncu.log 2>&1; echo ncu $?
wc -l gpurun_out/r01u_bench_launches.csv
