cd $GRAFT_REPO_ROOT
timeout 300 python tools/prof_run.py c3 > /dev/null 2>&1; echo plain $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_run.py c3 2>/dev/null | grep -i "k_finish\|k_leaf" | awk -F'","' '{print $5, $(NF)}' | sed 's/"//g' | head -20
