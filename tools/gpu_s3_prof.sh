# full ncu capture of one kernel (PubMed-shaped iteration 4 by default) + per-line and per-region summaries
# usage: bash tools/gpu_s3_prof.sh TAG [kernel regex] [config]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
T=${1:-x}; KRE=${2:-k_sampler}; CFG=${3:-pubmed}
bash tools/gpu_prof.sh $CFG $T $KRE 3 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_${CFG}_${T}.ncu-rep > gpurun_out/prof_${CFG}_${T}.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_${CFG}_${T}.ncu-rep 40 >> gpurun_out/prof_${CFG}_${T}.txt 2>&1
python tools/ncu_smem.py gpurun_out/prof_${CFG}_${T}.ncu-rep >> gpurun_out/prof_${CFG}_${T}.txt 2>&1
python tools/ncu_phases.py gpurun_out/prof_${CFG}_${T}.ncu-rep > gpurun_out/phases_${CFG}_${T}.txt 2>&1
head -40 gpurun_out/phases_${CFG}_${T}.txt
