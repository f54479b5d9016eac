cd $GRAFT_REPO_ROOT
SHUF_FAST_FINISH=0 timeout 300 python tools/ktime.py c3 2>&1 | head -9
SHUF_DBG=2 SHUF_FAST_FINISH=0 timeout 300 python tools/ktime.py c3 2>&1 | tail -12
