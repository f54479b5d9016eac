cd $GRAFT_REPO_ROOT
for c in "100000 256 4096 1" "3000000 256 4096 11" "2000000 2 3000 4" "50000 8 3000 2" "900000 256 3000 5 8" "600000 64 1500 5 16" "8000 2 4096 3" "5000 16 4096 4" "1048576 256 4096 1"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "segmented or bit_exact" 2>&1 | tail -2
timeout 300 python tools/ktime.py c2 2>&1 | head -9
timeout 300 python tools/ktime.py c5 2>&1 | head -9
timeout 300 python tools/ktime.py hot 2>&1 | head -2
