cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python tools/ipsc_run.py hot --reps 3 > gpurun_out/r02n_ipsc_plain.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02n_ipsc_launches.csv python tools/ipsc_run.py hot --reps 1 > gpurun_out/r02n_ncu.log 2>&1
timeout 600 python bench.py --mode ipsc --steps 3 --warmup 3 --no-cpu-baseline --no-gpu-baselines > gpurun_out/r02n_bench_ipsc.json 2> gpurun_out/r02n_bench_ipsc.err
