# round-2 (session 3) final evidence on one B200: GPU tests, smoke, the driver's bench line + reference arm,
# ncu launch list, K sweep / ClueWeb-shaped shard / two-branch / schedule-ablation lines
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
T=${1:-f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2 | tee gpurun_out/gputests_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_pubmed_$T.json 2> gpurun_out/bench_pubmed_$T.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 300 --csv --log-file gpurun_out/launches_$T.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --curve-iters 0 > gpurun_out/launches_$T.log 2>&1; echo "launches rc=$?"
for c in nytimes nytimes_k5k nytimes_k10k; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --curve-iters 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_$T.json 2>/dev/null; echo "$c rc=$?"
done
timeout 900 python bench.py --config nytimes_k32k --steps 3 --warmup 2 --curve-iters 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_nytimes_k32k_$T.json 2>/dev/null; echo "k32k rc=$?"
timeout 1200 python bench.py --config clueweb_shard8 --steps 3 --warmup 3 --curve-iters 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_clueweb_shard8_$T.json 2>/dev/null; echo "clueweb rc=$?"
timeout 900 python bench.py --sampler 2 --steps 5 --warmup 3 --curve-iters 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_two_branch_pubmed_$T.json 2>/dev/null; echo "tb rc=$?"
for sc in 1 2; do
  timeout 900 python bench.py --schedule $sc --steps 10 --warmup 3 --curve-iters 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_pubmed_sched${sc}_$T.json 2>/dev/null; echo "sched$sc rc=$?"
done
for f in gpurun_out/bench_*_$T.json; do
  python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    j = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "ERR", e); sys.exit()
r = j.get("roofline") or {}
pm = (j.get("paper_metric") or {}).get("mean_tokens_per_s")
print(f.split("/")[-1], round(j["value"] / 1e9, 3), "Gtok/s", round(j["ms_per_step"], 2), "frac", r.get("frac") and round(r["frac"], 3),
      "paper", pm and round(pm / 1e9, 3), "e2e", (j.get("e2e") or {}).get("value"), "phases", j.get("phases_ms_per_step"))
PY
done
