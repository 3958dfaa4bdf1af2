# copy one evidence run (tools/gpu_evidence.sh <tag>) from gpurun_out/ into profiles/
# usage: bash tools/save_evidence.sh <tag>
T=$1
cp gpurun_out/bench_pubmed_$T.json profiles/r01_bench_${T}_pubmed.json
cp gpurun_out/bench_nytimes_$T.json profiles/r01_bench_${T}_nytimes.json
cp gpurun_out/bench_ref_$T.json profiles/r01_bench_${T}_reference.json
cp gpurun_out/curve_pubmed_$T.csv profiles/r01_curve_pubmed_$T.csv
cp gpurun_out/curve_nytimes_$T.csv profiles/r01_curve_nytimes_$T.csv
python tools/ncu_summary.py gpurun_out/prof_pubmed_$T.ncu-rep > profiles/r01_ncu_sampler_pubmed_$T.txt 2>&1
python tools/ncu_smem.py gpurun_out/prof_pubmed_$T.ncu-rep 20 >> profiles/r01_ncu_sampler_pubmed_$T.txt
python tools/phase_split.py gpurun_out/prof_pubmed_$T.ncu-rep >> profiles/r01_ncu_sampler_pubmed_$T.txt
python tools/ncu_summary.py gpurun_out/prof_pubmed_${T}doc.ncu-rep > profiles/r01_ncu_docpass_pubmed_$T.txt 2>&1
python - "$T" <<'PY' > profiles/r01_launches_$T.txt
import csv, collections, sys
T = sys.argv[1]
rows = list(csv.reader([l for l in open(f'gpurun_out/launches_{T}.csv') if l.startswith('"')]))
hdr = rows[0]; agg = collections.defaultdict(list)
print("ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 200 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline")
print("(cold-cache, serialised per-launch times; create() setup kernels + 5 iterations + 1 LLPT)")
for r in rows[1:]:
    d = dict(zip(hdr, r)); agg[d['Kernel Name'].split('(')[0]].append(float(d['Metric Value']))
it = ['k_den', 'k_word_prep', 'k_doc_hist<1>', 'k_doc_block<1>', 'k_sampler']
tot = sum(sum(v) for k, v in agg.items() if any(x in k for x in it))
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    share = f"{100 * sum(v) / tot:5.1f}%" if any(x in k for x in it) else "  (setup/LLPT)"
    print(f"{len(v):3d} launches {sum(v) / 1e6:9.2f} ms total {sum(v) / len(v) / 1e6:8.3f} ms/launch  iteration share {share}  {k}")
PY
grep -h "dram__bytes\|Duration" profiles/r01_ncu_sampler_pubmed_$T.txt profiles/r01_ncu_docpass_pubmed_$T.txt
for f in gpurun_out/bench_nytimes_k5k_$T.json gpurun_out/bench_nytimes_k10k_$T.json gpurun_out/bench_two_branch_pubmed_$T.json gpurun_out/bench_two_branch_nytimes_$T.json; do
  [ -f $f ] && cp $f profiles/r01_$(basename $f .json | sed "s/_$T\$//")_$T.json
done
