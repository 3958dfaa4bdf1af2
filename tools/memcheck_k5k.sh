cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "large_K_paths and 5000" > gpurun_out/memcheck_k5k.log 2>&1
grep -v "Host Frame" gpurun_out/memcheck_k5k.log | head -30
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
