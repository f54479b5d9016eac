cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_run.py hot > gpurun_out/r01m_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_leaf_items|k_finish_children" -c 3 \
   -o gpurun_out/r01m_leaf python tools/prof_run.py hot > gpurun_out/r01m_ncu.log 2>&1
echo "exit $?"
tail -5 gpurun_out/r01m_ncu.log
