cd $GRAFT_REPO_ROOT
for w in 16 64 256 100000; do echo "wpr $w"; SHUF_IP_WPR=$w timeout 300 python tools/ktime.py hot --inplace 2>&1 | head -1; done
