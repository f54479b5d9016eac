#!/bin/bash
# One gpurun call: parity + full-size GPU tests, then bench lines of the given
# workloads.  Usage (under gpurun): bash tools/gpu_round_c.sh TAG c2 c5 c4 ...
TAG=${1:-r}; shift
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/${TAG}_pytest_leaf.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_leaf.log
for c in "$@"; do
  steps=10; [ $c = c4 ] && steps=3
  timeout 1500 python bench.py --workload $c --steps $steps --warmup 3 --no-gpu-baselines \
      > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "bench $c exit $?" >> gpurun_out/${TAG}_bench_$c.err
done
ls -la gpurun_out | grep ${TAG}
