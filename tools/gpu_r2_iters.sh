# per-iteration evidence (PubMed-shaped): the live curve with model bytes / roofline per iteration,
# and ncu DRAM bytes + duration of the sampler and doc pass at iterations 1, 10, 50, 100, 200
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
T=${1:-i1}
timeout 900 python tools/curve.py --config pubmed --iters 200 --llpt-every 20 --csv gpurun_out/curve_pubmed_$T.csv 2>&1 | tail -3
for it in 1 10 50 100 200; do
  timeout 900 ncu --clock-control none -k regex:"k_sampler|k_doc_hist" -s $((2 * (it - 1))) -c 2 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed \
    --csv --log-file gpurun_out/ncu_iter${it}_$T.csv python tools/profile_iter.py --config pubmed --warmup $((it - 1)) --iters 1 > gpurun_out/ncu_iter${it}_$T.log 2>&1
  echo "iter $it rc=$?"; tail -1 gpurun_out/ncu_iter${it}_$T.log
done
