cd $GRAFT_REPO_ROOT
for w in c1 c2 c3 c5 hot; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02n_$w.json 2> gpurun_out/r02n_$w.err
done
python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02n_c4.json 2> gpurun_out/r02n_c4.err
for w in hot c2 c3; do
  python bench.py --workload $w --mode inplace --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02n_ip_$w.json 2> gpurun_out/r02n_ip_$w.err
done
