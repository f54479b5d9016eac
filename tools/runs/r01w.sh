cd $GRAFT_REPO_ROOT
bash tools/gpu_round.sh r01w tests bench launches full
tail -3 gpurun_out/r01w_pytest_gpu.log; python -c "
import json; b=json.load(open('gpurun_out/r01w_bench.json')); print(b['ms_per_step'], b['value']/1e9, b['eff_GBps'], b['frac_of_8TBps'], b['roofline']['achieved'], b['roofline']['frac'], b['roofline']['avg_launch_ms'], b['e2e']['ms_per_step'], b['kernels']['finish'], b['kernels']['scatter'], b['clocks'])"; tail -2 gpurun_out/r01w_bench.err; tail -1 gpurun_out/r01w_ncu_full.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
