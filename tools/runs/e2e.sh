cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/e2e_bench.json 2> gpurun_out/e2e_bench.err; echo exit $?
python -c "import json; b=json.load(open('gpurun_out/e2e_bench.json')); print(b['ms_per_step'], b['e2e'])"
tail -3 gpurun_out/e2e_bench.err
