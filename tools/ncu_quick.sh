# quick ncu metrics of one kernel per library variant (PubMed-shaped iteration 4 by default)
# usage: bash tools/ncu_quick.sh "v1 v2 ..." [kernel regex] [config]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
KRE=${2:-k_sampler}; CFG=${3:-pubmed}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed
for v in $1; do
  EZLDA_LIB=$PWD/_variants/lib_$v.so timeout 900 ncu --metrics $M --clock-control none -k regex:$KRE -s 3 -c 1 --csv \
    python tools/profile_iter.py --config $CFG --warmup 4 --iters 1 2>/dev/null | grep '^"' > gpurun_out/ncuq_${v}_${CFG}.csv
  echo "== $v"; python - gpurun_out/ncuq_${v}_${CFG}.csv <<'PY'
import csv, sys
for r in csv.reader(open(sys.argv[1])):
    if len(r) > 14 and r[0] != "ID": print(f"  {r[12]:60s} {r[13]:8s} {r[14]}")
PY
done
