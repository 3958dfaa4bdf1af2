# round-2 quick GPU check: GPU tests (optionally filtered) + PubMed bench line
# usage: bash tools/gpu_r2_quick.sh [pytest -k expr] [bench configs]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
K="${1:-}"
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=8 -k "$K" 2>&1 | tail -25 > gpurun_out/gputests.log
else
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=8 2>&1 | tail -25 > gpurun_out/gputests.log
fi
cat gpurun_out/gputests.log
for c in ${2:-pubmed}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err
  python -c "import json,sys; j=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(j['value']/1e9,3), 'Gtok/s', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phases_ms_per_step'].items()}, 'frac', round(j['roofline']['frac'] or 0,3), 'redraw', j.get('exact_redraw_frac'))" || tail -5 gpurun_out/bench_$c.err
done
