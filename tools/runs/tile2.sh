cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for i in 1 2 3; do timeout 300 python tools/ktime.py hot 2>&1 | sed -n 1p; done
for w in c2 c3; do timeout 300 python tools/ktime.py $w 2>&1 | sed -n 1p; done
