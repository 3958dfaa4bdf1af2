cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
bash tools/gpu_r2_prof.sh nytimes_k10k k10s k_sampler 3 > /dev/null 2>&1
head -45 gpurun_out/prof_nytimes_k10k_k10s.txt
timeout 900 ncu --clock-control none -k regex:"k_word|k_doc|k_den|k_nk|k_item" -s 12 -c 12 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --csv --log-file gpurun_out/ncu_k10k_small.csv python tools/profile_iter.py --config nytimes_k10k --warmup 3 --iters 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/ncu_k10k_small.csv')))
hdr=None
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); print(d['ID'], d['Kernel Name'][:40], d['Metric Name'], d['Metric Value'])
PY
