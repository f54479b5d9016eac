cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/ip_prof.py > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ip_classify|k_ip_permute" -c 2 \
   -o gpurun_out/r01v_ip python tools/ip_prof.py > gpurun_out/r01v_ncu.log 2>&1
echo "exit $?"
