cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for v in quad quad12; do
  EZLDA_LIB=$PWD/_variants/lib_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "tiny or small or long_docs or rare_paths or knob" 2>&1 | tail -2
done
STEPS=10 WARMUP=3 bash tools/variants.sh "pubmed nytimes" $PWD/_variants/lib_base.so $PWD/_variants/lib_quad.so $PWD/_variants/lib_quad12.so
