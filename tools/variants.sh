#!/bin/bash
# usage: tools/variants.sh "cfg1 cfg2" lib1 lib2 ...  (runs bench.py with EZLDA_LIB=each variant)
cfgs="$1"; shift
for lib in "$@"; do
  for c in $cfgs; do
    EZLDA_LIB=$lib timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup ${WARMUP:-3} --no-cpu-baseline --no-e2e ${EXTRA} 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$(basename $lib)', j['config']['workload'][:8], round(j['value']/1e9,3), 'Gtok/s', round(j['ms_per_step'],2), {k: round(v,2) for k,v in j['phases_ms_per_step'].items()}, round(j['roofline']['frac'],3))" 2>&1 | tail -1
  done
done
