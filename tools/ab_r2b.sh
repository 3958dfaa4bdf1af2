cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not fullsize" 2>&1 | tail -3
STEPS=8 WARMUP=3 EXTRA="--curve-iters 0" bash tools/variants.sh "pubmed nytimes_k5k nytimes_k10k" $PWD/paper_2007_08725_b200/libezlda.so $PWD/_variants/lib_g8.so $PWD/_variants/lib_g16.so
