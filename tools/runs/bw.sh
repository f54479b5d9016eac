cd $GRAFT_REPO_ROOT
for w in c5 c2 c3; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; b=json.loads(sys.stdin.read()); print(b['config']['workload'][:40], round(b['ms_per_step'],3), round(b['frac_of_8TBps'],3), b['roofline']['kernel'], b['roofline']['frac'], round(b['e2e']['ms_per_step'],2))"; done
