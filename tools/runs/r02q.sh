cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/ipsc_run.py hot --n 4194304 --reps 2 > gpurun_out/r02q_plain.log 2>&1
timeout 300 python tools/ipsc_run.py hot --reps 2 >> gpurun_out/r02q_plain.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_ipsc_small" -c 1 -o gpurun_out/r02q_small python tools/ipsc_run.py hot --n 4194304 --reps 1 > gpurun_out/r02q_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_ipsc_rs|k_ipsc_fine" -c 2 -o gpurun_out/r02q_rs python tools/ipsc_run.py hot --n 67108864 --reps 1 >> gpurun_out/r02q_ncu.log 2>&1
