#!/bin/bash
# One gpurun call: GPU tests, bench line, launch list and a full ncu capture
# of the scatter + finish kernels on the hot workload.  Usage (under gpurun):
#   bash tools/gpu_round.sh TAG [what...]   what in {tests bench launches full}
TAG=${1:-r}; shift
WHAT=${*:-tests bench launches full}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
for w in $WHAT; do
case $w in
tests)
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_gpu.log ;;
bench)
  timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
  echo "bench exit $?" >> gpurun_out/${TAG}_bench.err ;;
launches)
  timeout 600 python tools/prof_run.py hot --reps 2 > gpurun_out/${TAG}_plain.log 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches.csv python tools/prof_run.py hot --reps 2 > gpurun_out/${TAG}_ncu_launches.log 2>&1
  echo "launches exit $?" >> gpurun_out/${TAG}_ncu_launches.log ;;
full)
  timeout 600 python tools/prof_run.py hot > gpurun_out/${TAG}_plain1.log 2>&1 &&
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_finish_fast|k_hist" -c 7 \
      -o gpurun_out/${TAG}_full python tools/prof_run.py hot > gpurun_out/${TAG}_ncu_full.log 2>&1
  echo "full exit $?" >> gpurun_out/${TAG}_ncu_full.log ;;
esac
done
ls -la gpurun_out
