cd $GRAFT_REPO_ROOT
for w in c1 c2 c3 c5; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02b_$w.json 2> gpurun_out/r02b_$w.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02b_par.log 2>&1
