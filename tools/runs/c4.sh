cd $GRAFT_REPO_ROOT
timeout 600 python tools/ktime.py c4 2>&1 | head -9
timeout 600 python tools/ktime.py c4 --inplace 2>&1 | head -2
timeout 600 python tools/ktime.py c3 --inplace 2>&1 | head -2
timeout 600 python tools/ktime.py c5 2>&1 | head -1
