cd $GRAFT_REPO_ROOT
for v in 0 1 2 3; do
  SHUF_SCV=$v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02e_scv$v.json 2>&1
done
SHUF_SCV=0 python -m pytest tests/test_gpu_parity.py -x -q -k "bit_exact and not alternate" > gpurun_out/r02e_par0.log 2>&1
SHUF_SCV=2 python -m pytest tests/test_gpu_parity.py -x -q -k "bit_exact and not alternate" > gpurun_out/r02e_par2.log 2>&1
