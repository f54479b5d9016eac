cd $GRAFT_REPO_ROOT
SHUF_DBG=2 timeout 300 python tools/ktime.py hot 2>&1 | tail -32
timeout 300 python tools/ktime.py hot 2>&1 | head -9
