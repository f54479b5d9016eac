cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_ipsc_rs_warp" -c 1 -o gpurun_out/r02w_rsw python tools/ipsc_run.py hot --reps 1 > gpurun_out/r02w_ncu.log 2>&1
