cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "large_K or wide_segment or rare_paths or exact or tiny" 2>&1 | tail -2
for a in "" "--w-mode 1"; do
  bash tools/gpu_r2_bench.sh "nytimes_k5k nytimes_k10k" 8 "$a"
done
bash tools/gpu_r2_bench.sh "pubmed" 8
