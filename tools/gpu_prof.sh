# usage: bash tools/gpu_prof.sh <config> <tag> [kernel regex] [skip]
cd $GRAFT_REPO_ROOT
cfg=${1:-pubmed}; tag=${2:-x}; kre=${3:-k_sampler}; skip=${4:-3}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 \
  -o gpurun_out/prof_${cfg}_${tag} python tools/profile_iter.py --config $cfg --warmup 4 --iters 1 > gpurun_out/prof_${cfg}_${tag}.log 2>&1
tail -3 gpurun_out/prof_${cfg}_${tag}.log
