# bench lines only (no tests): usage bash tools/gpu_r2_bench.sh "cfgs" [steps] [extra args]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for c in ${1:-pubmed}; do
  timeout 900 python bench.py --config $c --steps ${2:-8} --warmup 3 --curve-iters 0 --no-cpu-baseline --no-e2e ${3:-} > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err
  python -c "import json,sys; j=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); r=j['roofline']; print('$c', round(j['value']/1e9,3), 'Gtok/s', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phases_ms_per_step'].items()}, 'smp_kernel_ms', round(r['ms_per_launch'],2), 'frac', round(r['frac'] or 0,3), 'redraw', j.get('exact_redraw_frac'))" || tail -5 gpurun_out/bench_$c.err
done
