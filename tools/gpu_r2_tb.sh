# GPU tests (optionally -k filtered) then bench lines: bash tools/gpu_r2_tb.sh "<-k expr or empty>" "cfgs"
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
if [ -n "$1" ]; then timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$1" 2>&1 | tail -3
else timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3; fi
bash tools/gpu_r2_bench.sh "${2:-pubmed}" ${3:-8}
