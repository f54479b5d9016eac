cd $GRAFT_REPO_ROOT
timeout 600 python tools/ktime.py c3 --inplace 2>&1 | tail -8
