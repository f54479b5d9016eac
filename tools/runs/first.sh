cd $GRAFT_REPO_ROOT
for c in "3000000 256 4096 11" "300001 1000 50 7" "900000 256 3000 5 8" "600000 64 1500 5 16" "200000 2 1 8" "777777 7 300 6" "1048576 256 4096 1"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -1; done | sort | uniq -c
for i in 1 2 3; do timeout 300 python tools/ktime.py hot 2>&1 | sed -n 1p; timeout 300 python tools/ktime.py hot 2>&1 | sed -n 6p; done
