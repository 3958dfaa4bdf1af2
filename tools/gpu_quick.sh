# quick GPU check: parity tests + PubMed/NYTimes bench lines (no CPU baseline / e2e)
# usage: bash tools/gpu_quick.sh [cfgs] [steps]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -4
for c in ${1:-pubmed nytimes}; do
  timeout 600 python bench.py --config $c --steps ${2:-10} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['config']['workload'][:8], round(j['value']/1e9,3), 'Gtok/s', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phases_ms_per_step'].items()}, 'frac', round(j['roofline']['frac'],3), 'redraw', j.get('exact_redraw_frac'))"
done
