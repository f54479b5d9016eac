cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
T=r05h
for e in 1 0; do
  python -c "import paper_2302_03317_b200._build as b; b.build(force=True, extra=['-DSHUF_LEAF_EARLY=$e'])" > gpurun_out/${T}_build$e.log 2>&1
  for wl in c5 c2; do
    echo "== $wl early=$e" >> gpurun_out/${T}_ktime.log
    timeout 300 python tools/ktime.py $wl >> gpurun_out/${T}_ktime.log 2>&1
  done
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "c2 or c5 or c1 or leaf or segment or seg" > gpurun_out/${T}_parity$e.log 2>&1; echo "exit $?" >> gpurun_out/${T}_parity$e.log
done
