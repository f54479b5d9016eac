cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02o_par.log 2>&1
for w in c1 c2 c5; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02o_$w.json 2> gpurun_out/r02o_$w.err
done
