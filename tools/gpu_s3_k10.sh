cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 200 --csv --log-file gpurun_out/launches_k10.csv \
  python bench.py --config nytimes_k10k --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --curve-iters 0 > gpurun_out/launches_k10.log 2>&1; echo "launches rc=$?"
bash tools/gpu_s3_prof.sh s3k10b k_sampler nytimes_k10k
