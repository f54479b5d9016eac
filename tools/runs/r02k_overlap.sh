cd $GRAFT_REPO_ROOT
for lib in libshuf.so libshuf_m3.so; do for ov in 0 1; do
  SHUF_LIB_PATH=$PWD/paper_2302_03317_b200/$lib SHUF_HIST_OVERLAP=$ov python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02k_${lib}_$ov.json 2>&1
done; done
python -m pytest tests/test_gpu_parity.py -x -q -k "shuffle_bit_exact or level_limited or invariance or depth" > gpurun_out/r02k_par.log 2>&1
