cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_ipsc_small" -c 1 -o gpurun_out/r03f_small python tools/ipsc_run.py hot --n 4194304 --reps 1 > gpurun_out/r03f_ncu.log 2>&1
