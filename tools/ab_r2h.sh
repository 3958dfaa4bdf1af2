cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
EZLDA_LIB=$PWD/_variants/lib_mg8.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "large_K or wide_segment or two_branch or rare_paths" 2>&1 | tail -1
STEPS=6 WARMUP=3 EXTRA="--curve-iters 0" bash tools/variants.sh "nytimes_k5k nytimes_k10k" $PWD/_variants/lib_head.so $PWD/_variants/lib_mg128.so $PWD/_variants/lib_mg32.so $PWD/_variants/lib_mg8.so
