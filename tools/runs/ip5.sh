cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_inplace.py -x -q 2>&1 | tail -2
for c in "3000000 256 4096 11" "1048576 256 4096 1" "300001 1000 50 7" "900000 256 3000 5 8"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -1; done | sort | uniq -c
timeout 300 python tools/ktime.py hot --inplace
timeout 300 python tools/ktime.py hot | head -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/ip_prof.py 2>/dev/null | grep -i "k_ip\|k_finish\|k_leaf" | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | grep -v "stripes\|plan\|root\|leaf" | head -30
