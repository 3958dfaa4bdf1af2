cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
STEPS=6 WARMUP=3 EXTRA="--curve-iters 0" bash tools/variants.sh "pubmed" $PWD/_variants/lib_dbase.so $PWD/_variants/lib_dnorec.so $PWD/_variants/lib_dnoflag.so $PWD/_variants/lib_dnowalk.so $PWD/_variants/lib_docnophx.so
