# per-iteration ncu metrics of the sampler and doc pass over 200 PubMed-shaped iterations
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 2400 ncu --clock-control none -k regex:"k_sampler|k_doc_hist" -c 420 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed,sm__inst_executed.sum \
  --csv --log-file gpurun_out/ncu_iters_pubmed.csv python tools/profile_iter.py --config pubmed --warmup 199 --iters 1 > gpurun_out/ncu_iters_pubmed.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_iters_pubmed.log; wc -l gpurun_out/ncu_iters_pubmed.csv
