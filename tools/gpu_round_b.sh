#!/bin/bash
# One gpurun call: per-config bench lines (C1..C5, HOT in-place) and full ncu
# captures of the kernels that dominate the other configs -- the leaf kernel
# on C2 / C5 and the in-place kernels on HOT.  Usage (under gpurun):
#   bash tools/gpu_round_b.sh TAG [what...]   what in {configs c4 leaf inplace}
TAG=${1:-r}; shift
WHAT=${*:-configs leaf inplace c4}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for w in $WHAT; do
case $w in
configs)
  for c in c1 c2 c3 c5; do
    timeout 900 python bench.py --workload $c --steps 10 --warmup 3 --no-gpu-baselines \
        > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
    echo "bench $c exit $?" >> gpurun_out/${TAG}_bench_$c.err
  done
  timeout 900 python bench.py --mode inplace --steps 10 --warmup 3 --no-gpu-baselines --no-cpu-baseline \
      > gpurun_out/${TAG}_bench_inplace.json 2> gpurun_out/${TAG}_bench_inplace.err ;;
c4)
  timeout 1500 python bench.py --workload c4 --steps 3 --warmup 3 --no-gpu-baselines \
      > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
  echo "bench c4 exit $?" >> gpurun_out/${TAG}_bench_c4.err ;;
leaf)
  for c in c2 c5; do
    timeout 300 python tools/prof_run.py $c > gpurun_out/${TAG}_plain_$c.log 2>&1 &&
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_leaf" -c 3 \
        -o gpurun_out/${TAG}_leaf_$c python tools/prof_run.py $c > gpurun_out/${TAG}_ncu_leaf_$c.log 2>&1
    echo "leaf $c exit $?" >> gpurun_out/${TAG}_ncu_leaf_$c.log
  done ;;
inplace)
  timeout 300 python tools/ip_prof.py hot > gpurun_out/${TAG}_plain_ip.log 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling node --csv \
      --log-file gpurun_out/${TAG}_ip_launches.csv python tools/ip_prof.py hot > gpurun_out/${TAG}_ncu_ip_launches.log 2>&1
  echo "ip launches exit $?" >> gpurun_out/${TAG}_ncu_ip_launches.log
  timeout 1200 ncu --set full --clock-control none --import-source on --graph-profiling node \
      -k regex:"k_ip_classify|k_ip_permute" -c 4 \
      -o gpurun_out/${TAG}_ip python tools/ip_prof.py hot > gpurun_out/${TAG}_ncu_ip.log 2>&1
  echo "ip full exit $?" >> gpurun_out/${TAG}_ncu_ip.log ;;
esac
done
ls -la gpurun_out
