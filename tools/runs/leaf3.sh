cd $GRAFT_REPO_ROOT
for c in "100000 256 4096 1" "3000000 256 64 5" "50000 7 3 2" "5000 256 4096 3" "2000000 16 100 4" "3000000 256 64 5 8" "3000000 100 200 5 16" "20000 256 16 3"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -1; done
timeout 300 python tools/ktime.py hot 2>&1 | head -9
SHUF_DEFER=0 timeout 300 python tools/ktime.py hot 2>&1 | head -9
timeout 60 tools/mb_fy
