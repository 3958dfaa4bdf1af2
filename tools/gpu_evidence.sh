# Round evidence run on one B200: GPU tests, smoke, bench lines, ncu launch list + one full capture.
# usage: bash tools/gpu_evidence.sh <tag>
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
tag=${1:-x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_pubmed_${tag}.json 2> gpurun_out/bench_pubmed_${tag}.err; tail -c 600 gpurun_out/bench_pubmed_${tag}.json
timeout 600 python bench.py --config nytimes --no-cpu-baseline > gpurun_out/bench_nytimes_${tag}.json 2>gpurun_out/bench_nytimes_${tag}.err; tail -c 300 gpurun_out/bench_nytimes_${tag}.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${tag}.json 2>&1; tail -c 300 gpurun_out/bench_ref_${tag}.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${tag}.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_${tag}.log 2>&1; tail -2 gpurun_out/launches_${tag}.log
bash tools/gpu_prof.sh pubmed ${tag} k_sampler 3
