cd $GRAFT_REPO_ROOT
bash tools/gpu_round.sh r02a tests bench launches full
for w in c1 c2 c3 c5; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02a_$w.json 2> gpurun_out/r02a_$w.err
done
python bench.py --workload hot --mode inplace --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02a_ip_hot.json 2> gpurun_out/r02a_ip_hot.err
