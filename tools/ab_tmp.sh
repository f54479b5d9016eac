cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
T=r05c
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${T}_parity.log 2>&1; echo "exit $?" >> gpurun_out/${T}_parity.log
for wl in hot c2 c5 c3; do for b in 1 0; do
  echo "== $wl lanes=$b" >> gpurun_out/${T}_ktime.log
  SHUF_HIST_LANES=$b timeout 300 python tools/ktime.py $wl >> gpurun_out/${T}_ktime.log 2>&1
done; done
for b in 1 0; do
SHUF_HIST_LANES=$b timeout 600 ncu --clock-control none -k regex:k_hist -c 1 --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active python tools/prof_run.py hot > gpurun_out/${T}_ncu_hist_lanes$b.log 2>&1
done
