# fresh source-level ncu captures of the doc pass and sampler (PubMed-shaped, iteration 4) + sanitizer on tiny
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
T=${1:-p2}
bash tools/gpu_r2_prof.sh pubmed ${T}doc k_doc_hist 3 > /dev/null 2>&1
python tools/ncu_smem.py gpurun_out/prof_pubmed_${T}doc.ncu-rep >> gpurun_out/prof_pubmed_${T}doc.txt 2>&1
bash tools/gpu_r2_prof.sh pubmed ${T}smp k_sampler 3 > /dev/null 2>&1
python tools/ncu_smem.py gpurun_out/prof_pubmed_${T}smp.ncu-rep >> gpurun_out/prof_pubmed_${T}smp.txt 2>&1
head -30 gpurun_out/prof_pubmed_${T}doc.txt
head -30 gpurun_out/prof_pubmed_${T}smp.txt
bash tools/gpu_r2_sanitize.sh
