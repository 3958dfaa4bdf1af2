cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
free -g | head -2; nproc
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 2>&1 | tail -30 > gpurun_out/gputests.log
cat gpurun_out/gputests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_pubmed.json 2>gpurun_out/bench.err; tail -c 3000 gpurun_out/bench_pubmed.json
