# create time and e2e per library variant (PubMed-shaped): tools/create_time.py + bench.py e2e
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for v in "$@"; do
  echo "== $v"
  EZLDA_LIB=$PWD/_variants/lib_$v.so timeout 600 python tools/create_time.py pubmed 2>&1 | grep "^create"
  EZLDA_LIB=$PWD/_variants/lib_$v.so timeout 900 python bench.py --steps 30 --warmup 3 --curve-iters 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('value', round(j['value']/1e9,3), 'e2e', round(j['e2e']['value']/1e9,3))"
done
