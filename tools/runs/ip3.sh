cd $GRAFT_REPO_ROOT
timeout 300 python tools/ktime.py hot --inplace
timeout 300 python tools/ktime.py c2 --inplace
timeout 300 python tools/ktime.py c3 --inplace
timeout 300 python tools/prof_run.py hot > /dev/null 2>&1; echo plain $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/ip_prof.py 2>/dev/null | grep -i "k_ip\|k_finish\|k_leaf" | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | head -40
