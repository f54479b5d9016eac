cd $GRAFT_REPO_ROOT
for c in "100000 256 4096 1" "3000000 256 4096 11" "2000000 2 3000 4" "50000 8 3000 2" "900000 256 3000 5 8" "600000 64 1500 5 16" "1048576 256 4096 1" "3000000 256 64 5" "777777 7 300 6" "300001 1000 50 7" "200000 2 1 8"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -1; done | sort | uniq -c
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "raw or segmented" 2>&1 | tail -1
SHUF_DBG=4 timeout 300 python tools/ktime.py hot 2>&1 | sed -n 1,8p
SHUF_DBG=4 timeout 300 python tools/ktime.py hot 2>&1 | tail -30 | sed -n 1,12p
for w in c2 c3 c5; do timeout 300 python tools/ktime.py $w 2>&1 | head -1; done
