cd $GRAFT_REPO_ROOT
export SHUF_FAST_FINISH=1
for c in "100000 256 4096 1" "3000000 256 4096 11" "3000000 256 64 5" "50000 7 3 2" "2000000 16 100 4" "3000000 256 64 5 8" "3000000 100 200 5 16" "20000 256 16 3" "1048576 256 4096 1"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -1; done
SHUF_DBG=4 timeout 300 python tools/ktime.py hot 2>&1 | tail -40
SHUF_RANK_MODE=match timeout 300 python tools/ktime.py hot 2>&1 | head -9
