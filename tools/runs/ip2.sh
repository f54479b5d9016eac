cd $GRAFT_REPO_ROOT
SHUF_SFUSE=1 timeout 900 python tools/ip_census.py 300 6000 5000
SHUF_SFUSE=1 timeout 900 python tools/ip_census.py 300 6000 20000
SHUF_SFUSE=1 timeout 900 python tools/ip_census.py 160 8000 777
