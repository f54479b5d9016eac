cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for g in 1 2 4 8; do echo "grid $g/SM" >> gpurun_out/r02s_plain.log; SHUF_IPSC_RSGRID=$g timeout 600 python tools/ipsc_run.py hot --reps 2 >> gpurun_out/r02s_plain.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02s_launches.csv python tools/ipsc_run.py hot --reps 1 > gpurun_out/r02s_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_ipsc_small" -c 1 -o gpurun_out/r02s_small python tools/ipsc_run.py hot --n 4194304 --reps 1 >> gpurun_out/r02s_ncu.log 2>&1
