cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5
for kb in ${KBS:-0}; do EXTRA="--doc-block-kb $kb" tools/variants.sh "${CFGS:-pubmed}" ${LIBS:-paper_2007_08725_b200/libezlda.so} | sed "s/^/kb=$kb /"; done
