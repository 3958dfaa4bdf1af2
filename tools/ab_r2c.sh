cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
STEPS=8 WARMUP=3 EXTRA="--curve-iters 0" bash tools/variants.sh "pubmed" $PWD/_variants/lib_base.so $PWD/_variants/lib_fakerow.so $PWD/_variants/lib_noconf.so $PWD/_variants/lib_both.so $PWD/_variants/lib_docnophx.so
