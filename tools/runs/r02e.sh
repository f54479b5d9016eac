cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_finish_fast" --launch-skip 1 -c 1 \
      -o gpurun_out/r02e_fin python tools/prof_run.py hot > gpurun_out/r02e_ncu.log 2>&1
