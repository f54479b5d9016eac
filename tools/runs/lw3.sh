cd $GRAFT_REPO_ROOT
for c in "2000000 2 3000 4" "50000 8 3000 2" "900000 256 3000 5 8" "600000 64 1500 5 16" "8000 2 4096 3" "5000 16 4096 4" "100000 256 4096 1"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -1; done | sort | uniq -c
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "segmented" 2>&1 | tail -1
for w in c2 c5 c3 hot; do timeout 300 python tools/ktime.py $w 2>&1 | sed -n 1p; done
