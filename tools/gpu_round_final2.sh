#!/bin/bash
# Round-end check plus the C2 / C5 bench lines of the same build.
TAG=${1:-r}
cd "${GRAFT_REPO_ROOT:-.}"
bash tools/gpu_round_final.sh $TAG
for c in c5 c2; do
  timeout 900 python bench.py --workload $c --steps 10 --warmup 3 --no-gpu-baselines > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "bench $c exit $?" >> gpurun_out/${TAG}_bench_$c.err
done
ls gpurun_out | grep $TAG
