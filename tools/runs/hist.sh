cd $GRAFT_REPO_ROOT
for c in "3000000 256 4096 11" "1048576 128 4096 1" "2000000 16 100 4" "200000 2 1 8"; do timeout 120 python tools/repro_case.py $c 2>&1 | tail -1; done | sort | uniq -c
for i in 1 2; do timeout 300 python tools/ktime.py hot 2>&1 | sed -n 1,3p; done
