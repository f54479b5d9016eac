cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/ipsc_run.py hot --n 4194304 --reps 2 > gpurun_out/r02p_plain.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_ipsc_small|k_ipsc_fine|k_ipsc_rs" -c 3 -o gpurun_out/r02p_full python tools/ipsc_run.py hot --n 4194304 --reps 1 > gpurun_out/r02p_ncu.log 2>&1
