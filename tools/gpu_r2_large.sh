cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=6 -k "large_K or two_branch or invalid" 2>&1 | tail -12
bash tools/gpu_prof.sh nytimes_k10k r2a k_sampler 3
python tools/ncu_summary.py gpurun_out/prof_nytimes_k10k_r2a.ncu-rep > gpurun_out/prof_nytimes_k10k_r2a.txt 2>&1; head -30 gpurun_out/prof_nytimes_k10k_r2a.txt
timeout 900 python bench.py --config nytimes_k32k --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_k32k.json 2>gpurun_out/bench_k32k.err; tail -c 1500 gpurun_out/bench_k32k.json; tail -3 gpurun_out/bench_k32k.err
