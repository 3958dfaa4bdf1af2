"""Build libezlda variants with -D defines into _variants/ (for tools/variants.sh A/B runs).

    python tools/build_variants.py name1:DEF=1,DEF2=3 name2:DEF=2 ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_08725_b200 import build as b  # noqa: E402

os.makedirs(os.path.join(b.ROOT, "_variants"), exist_ok=True)
for spec in sys.argv[1:]:
    name, _, defs = spec.partition(":")
    lib = os.path.join(b.ROOT, "_variants", f"lib_{name}.so")
    b.build(force=True, lib=lib, defines=tuple(x for x in defs.split(",") if x))
    print(lib)
