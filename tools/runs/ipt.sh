cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_inplace.py -x -q 2>&1 | tail -2
timeout 600 python tools/ktime.py hot --inplace 2>&1 | head -1
timeout 600 python tools/ktime.py c2 --inplace 2>&1 | head -1
timeout 600 python tools/ktime.py c3 --inplace 2>&1 | head -1
