#!/bin/bash
# One gpurun call: a pytest selection, then bench lines of the given workloads.
# Usage (under gpurun): bash tools/gpu_round_d.sh TAG "<pytest args>" c2 c5 ...
TAG=${1:-r}; SEL=$2; shift; shift
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest $SEL -m gpu -x -q > gpurun_out/${TAG}_pytest_sel.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_sel.log
for c in "$@"; do
  timeout 900 python bench.py --workload $c --steps 10 --warmup 3 --no-gpu-baselines --e2e-steps 0 --no-cpu-baseline \
      > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "bench $c exit $?" >> gpurun_out/${TAG}_bench_$c.err
  SHUF_LEAF_SIGMA=-1 timeout 900 python bench.py --workload $c --steps 10 --warmup 3 --no-gpu-baselines --e2e-steps 0 --no-cpu-baseline \
      > gpurun_out/${TAG}_bench_${c}_onepass.json 2>> gpurun_out/${TAG}_bench_$c.err
done
ls -la gpurun_out | grep ${TAG}
