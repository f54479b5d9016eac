cd $GRAFT_REPO_ROOT
for c in "100000 256 4096 1" "3000000 256 4096 11" "3000000 256 64 5" "50000 8 3 2" "2000000 16 100 4" "3000000 256 64 5 8" "3000000 128 200 5 16" "200000 2 1 8" "777777 64 300 6" "999999 32 50 3"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -1; done
timeout 300 python tools/ktime.py hot 2>&1 | head -9
