# NEXT-3 ablations on the current code (iterations 4-11 unless noted): W storage, g, split, H4 schedule, exact draws
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for c in pubmed nytimes_k10k; do
for a in "" "--w-mode 1" "--w-mode 2" "--g 1" "--g 3" "--split 2000" "--split 100000" "--schedule 1" "--exact-draws"; do
  timeout 900 python bench.py --config $c --steps 8 --warmup 3 --curve-iters 0 --no-cpu-baseline --no-e2e $a 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print(json.dumps({'config': '$c', 'args': '$a' or 'default', 'gtok_s': round(j['value']/1e9,3), 'ms_per_step': round(j['ms_per_step'],2), 'phases': {k: round(v,2) for k,v in j['phases_ms_per_step'].items()}, 'skip_S': round(j['skip_S_frac'],4), 'redraw': j.get('exact_redraw_frac')}))"
done
done
