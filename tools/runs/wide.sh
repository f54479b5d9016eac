cd $GRAFT_REPO_ROOT
for c in "3000000 256 4096 11" "900000 256 3000 5 8" "300001 1000 50 7"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -1; done | sort | uniq -c
timeout 300 python tools/ktime.py hot 2>&1 | sed -n 1p
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c4" 2>&1 | tail -2
