cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "large_K or wide_segment or two_branch or rare_paths or multi_rank or one_rank" 2>&1 | tail -2
bash tools/gpu_r2_bench.sh "nytimes_k5k nytimes_k10k nytimes_k32k clueweb_shard8" 4
