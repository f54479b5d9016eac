cd $GRAFT_REPO_ROOT
for c in "100000 256 4096 1" "3000000 256 4096 11" "2000000 2 3000 4" "50000 8 3000 2" "900000 256 3000 5 8" "600000 64 1500 5 16" "8000 2 4096 3" "5000 16 4096 4" "1048576 256 4096 1" "3000000 256 64 5" "777777 7 300 6" "300001 1000 50 7" "200000 2 1 8"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -1; done | sort | uniq -c
for w in hot c2 c3 c5; do timeout 300 python tools/ktime.py $w 2>&1 | head -8 | tr '\n' ' ' | sed 's/  */ /g'; echo; done
