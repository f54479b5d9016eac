cd $GRAFT_REPO_ROOT
for v in 1 4 5 6; do
  SHUF_SCV=$v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02f_scv$v.json 2>&1
done
for v in 1 4 5 6; do
  SHUF_SCV=$v python -m pytest tests/test_gpu_parity.py -x -q -k "shuffle_bit_exact or level_limited" > gpurun_out/r02f_par$v.log 2>&1
done
