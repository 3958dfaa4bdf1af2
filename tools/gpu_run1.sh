cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15
KBS="0 32768 65536 131072" CFGS="pubmed nytimes" bash -c 'for kb in $KBS; do EXTRA="--doc-block-kb $kb" tools/variants.sh "$CFGS" paper_2007_08725_b200/libezlda.so | sed "s/^/kb=$kb /"; done'
