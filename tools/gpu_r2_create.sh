cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not fullsize" 2>&1 | tail -2
EZLDA_CREATE_TIMING=1 python tools/create_time.py pubmed 2>&1 | tail -13
timeout 900 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --curve-iters 0 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value']/1e9,3), round(j['ms_per_step'],2), 'e2e', round(j['e2e']['value']/1e9,3), j['setup_s'])"
