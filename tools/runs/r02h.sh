cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_inplace.py -x -q > gpurun_out/r02h_ip.log 2>&1
for w in hot c2 c3; do
python bench.py --workload $w --mode inplace --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02h_ip_$w.json 2> gpurun_out/r02h_ip_$w.err
done
