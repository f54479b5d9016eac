cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_run.py hot > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter_rx" -c 1 \
   -o gpurun_out/r01q_rx python tools/prof_run.py hot > gpurun_out/r01q_ncu.log 2>&1
echo "exit $?"; tail -3 gpurun_out/r01q_ncu.log
