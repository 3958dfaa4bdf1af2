# Round evidence run on one B200: GPU tests, smoke, bench lines, ncu launch list + full captures.
# usage: bash tools/gpu_evidence.sh <tag>
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
tag=${1:-x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_pubmed_${tag}.json 2> gpurun_out/bench_pubmed_${tag}.err; tail -c 300 gpurun_out/bench_pubmed_${tag}.json
timeout 600 python bench.py --config nytimes --no-cpu-baseline > gpurun_out/bench_nytimes_${tag}.json 2>gpurun_out/bench_nytimes_${tag}.err; tail -c 200 gpurun_out/bench_nytimes_${tag}.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${tag}.json 2>&1; tail -c 200 gpurun_out/bench_ref_${tag}.json
# launch list of the library's kernels over the bench command (2 timed + 3 warm-up iterations)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 200 --csv --log-file gpurun_out/launches_${tag}.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_${tag}.log 2>&1; tail -1 gpurun_out/launches_${tag}.log
bash tools/gpu_prof.sh pubmed ${tag} k_sampler 3
bash tools/gpu_prof.sh pubmed ${tag}doc k_doc_hist 3
timeout 600 python tools/curve.py --config pubmed --iters 200 --llpt-every 20 --csv gpurun_out/curve_pubmed_${tag}.csv 2>&1 | tail -1
timeout 600 python tools/curve.py --config nytimes --iters 200 --llpt-every 20 --csv gpurun_out/curve_nytimes_${tag}.csv 2>&1 | tail -1
for c in nytimes_k5k nytimes_k10k; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_${tag}.json 2>/dev/null; tail -c 120 gpurun_out/bench_${c}_${tag}.json
done
for c in pubmed nytimes; do
  timeout 600 python bench.py --config $c --sampler 2 --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_two_branch_${c}_${tag}.json 2>/dev/null; tail -c 120 gpurun_out/bench_two_branch_${c}_${tag}.json
done
