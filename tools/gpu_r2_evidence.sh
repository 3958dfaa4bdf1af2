# round-2 evidence: driver-style bench lines, reference arm, K sweep / ClueWeb shard / two-branch lines
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
T=${1:-e1}
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_pubmed_$T.json 2> gpurun_out/bench_pubmed_$T.err; echo "pubmed rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; echo "ref rc=$?"
for c in nytimes nytimes_k5k nytimes_k10k; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_$T.json 2> gpurun_out/bench_${c}_$T.err; echo "$c rc=$?"
done
timeout 900 python bench.py --config nytimes_k32k --steps 3 --warmup 2 --curve-iters 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_nytimes_k32k_$T.json 2> gpurun_out/bench_nytimes_k32k_$T.err; echo "k32k rc=$?"
timeout 900 python bench.py --config clueweb_shard8 --steps 3 --warmup 2 --curve-iters 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_clueweb_shard8_$T.json 2> gpurun_out/bench_clueweb_shard8_$T.err; echo "clueweb rc=$?"
timeout 900 python bench.py --sampler 2 --steps 5 --warmup 3 --curve-iters 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_two_branch_pubmed_$T.json 2> gpurun_out/bench_two_branch_pubmed_$T.err; echo "tb rc=$?"
for s in 1 2; do
  timeout 900 python bench.py --schedule $s --steps 10 --warmup 3 --curve-iters 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_pubmed_sched${s}_$T.json 2> gpurun_out/bench_pubmed_sched${s}_$T.err; echo "sched $s rc=$?"
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
ph = j.get("phases_ms_per_step") or {}
pm = (j.get("paper_metric") or {}).get("mean_tokens_per_s")
print(f.split("/")[-1], round(j["value"] / 1e9, 3), "Gtok/s", round(j["ms_per_step"], 2), {k: round(v, 2) for k, v in ph.items()},
      "frac", r.get("frac") and round(r["frac"], 3), "paper", pm and round(pm / 1e9, 3), "e2e", j.get("e2e", {}).get("value"))
PY
done
