# usage: bash tools/gpu_r2_prof.sh <config> <tag> [kernel regex] [skip]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
bash tools/gpu_prof.sh "$@"
cfg=${1:-pubmed}; tag=${2:-x}
python tools/ncu_summary.py gpurun_out/prof_${cfg}_${tag}.ncu-rep > gpurun_out/prof_${cfg}_${tag}.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_${cfg}_${tag}.ncu-rep 30 >> gpurun_out/prof_${cfg}_${tag}.txt 2>&1
head -60 gpurun_out/prof_${cfg}_${tag}.txt
