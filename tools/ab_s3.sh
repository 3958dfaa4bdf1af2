# A/B of library variants in _variants/: GPU parity tests on the variant named by $TESTV, then bench lines
# usage: TESTV=name bash tools/ab_s3.sh "cfgs" base v1 v2 ...
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
cfgs="$1"; shift
for v in $TESTV; do
  echo "== gpu tests $v"; EZLDA_LIB=$PWD/_variants/lib_$v.so timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
done
libs=""; for v in "$@"; do libs="$libs $PWD/_variants/lib_$v.so"; done
STEPS=${STEPS:-8} WARMUP=3 EXTRA="--curve-iters 0" bash tools/variants.sh "$cfgs" $libs
