cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_inplace.py -x -q 2>&1 | tail -3
timeout 300 python tools/ktime.py hot --inplace
timeout 300 python tools/ktime.py c3 --inplace
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/ip_prof.py 2>/dev/null | grep -i "k_ip\|k_finish\|k_leaf" | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | head -30
