cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench $?
python -c "
import json; b=json.load(open('gpurun_out/final_bench.json')); print(b['ms_per_step'], round(b['value']/1e9,2), round(b['eff_GBps']), round(b['frac_of_8TBps'],4), b['roofline']['achieved'], b['roofline']['frac'], b['e2e']['ms_per_step'], b['cpu_baseline']['value'], b['clocks'])"
