export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for kb in ${KBS:-0 8192 24576 49152 98304 393216}; do EXTRA="--doc-block-kb $kb" tools/variants.sh "${CFGS:-pubmed nytimes}" paper_2007_08725_b200/libezlda.so | sed "s/^/kb=$kb /"; done
