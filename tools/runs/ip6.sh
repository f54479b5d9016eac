cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_inplace.py -x -q 2>&1 | tail -2
timeout 300 python tools/ktime.py hot --inplace
timeout 300 python tools/ktime.py c2 --inplace
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/ip_prof.py 2>/dev/null | grep -i "k_ip_permute\|k_ip_classify" | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | head -30
