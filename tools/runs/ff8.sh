cd $GRAFT_REPO_ROOT
export SHUF_FAST_FINISH=1
echo "== FY skipped (S-bound)"; SHUF_DBG=12 timeout 300 python tools/ktime.py hot 2>&1 | tail -40 | sed -n 9,20p
echo "== S idle (F alone)"; SHUF_DBG=20 timeout 300 python tools/ktime.py hot 2>&1 | tail -40 | sed -n 9,20p
