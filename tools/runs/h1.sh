cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/ktime.py hot 2>&1 | sed -n 1,3p; done
timeout 300 python tools/ktime.py c3 2>&1 | sed -n 1,3p
