cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bit_exact" 2>&1 | tail -2
SHUF_FAST_FINISH=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "shuffle_bit_exact" 2>&1 | tail -1
