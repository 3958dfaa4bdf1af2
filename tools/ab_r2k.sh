cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
EZLDA_LIB=$PWD/_variants/lib_du1.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "tiny or small or long_docs or parity_g" 2>&1 | tail -1
STEPS=8 WARMUP=3 EXTRA="--curve-iters 0" bash tools/variants.sh "pubmed nytimes" $PWD/_variants/lib_du0.so $PWD/_variants/lib_du1.so $PWD/_variants/lib_du1m3.so
