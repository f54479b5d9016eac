cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SHUF_FAST_FINISH=1 timeout 300 python tools/ktime.py hot 2>&1 | head -30
timeout 300 python tools/ktime.py c5 2>&1 | head -12
SHUF_LEAF=0 timeout 300 python tools/ktime.py c5 2>&1 | head -12
timeout 300 python tools/ktime.py c3 2>&1 | head -12
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
