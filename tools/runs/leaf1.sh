set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in "100000 256 4096 1" "3000000 256 64 5" "50000 7 3 2" "1000 2 1 9" "5000 256 4096 3" "2000000 16 100 4"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -2; done
for c in "3000000 256 64 5 8" "3000000 100 200 5 16"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -2; done
timeout 300 python tools/ktime.py hot 2>&1 | head -12
SHUF_LEAF=0 timeout 300 python tools/ktime.py hot 2>&1 | head -12
SHUF_SFUSE=4096 timeout 300 python tools/ktime.py hot 2>&1 | head -12
timeout 300 python tools/ktime.py c2 2>&1 | head -12
SHUF_LEAF=0 timeout 300 python tools/ktime.py c2 2>&1 | head -12
timeout 300 python tools/ktime.py c5 2>&1 | head -12
SHUF_LEAF=0 timeout 300 python tools/ktime.py c5 2>&1 | head -12
