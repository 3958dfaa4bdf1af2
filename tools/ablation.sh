# NEXT-3 ablations on the PubMed-shaped config: W storage, S_est depth g,
# large-word split, exact fp64 draws.  usage: bash tools/ablation.sh [config] [steps]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
c=${1:-pubmed}; st=${2:-8}
for a in "" "--w-mode 1" "--w-mode 2" "--g 1" "--g 3" "--split 2000" "--split 100000" "--exact-draws"; do
  timeout 900 python bench.py --config $c --steps $st --warmup ${WARM:-3} --no-cpu-baseline --no-e2e $a 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print(json.dumps({'args': '$a' or 'default', 'gtok_s': round(j['value']/1e9,3), 'ms_per_step': round(j['ms_per_step'],2), 'phases': {k: round(v,2) for k,v in j['phases_ms_per_step'].items()}, 'skip_S': round(j['skip_S_frac'],4), 'redraw': j.get('exact_redraw_frac')}))"
done
