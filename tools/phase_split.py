"""Split an ncu report's per-line stall/instruction shares of k_sampler into phases.
    python tools/phase_split.py <rep>   (line ranges taken from the current kernels.cu markers)"""
import re
import subprocess
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = open(os.path.join(ROOT, "paper_2007_08725_b200", "csrc", "kernels.cu")).read().splitlines()


def find(pat):
    for i, l in enumerate(src, 1):
        if pat in l:
            return i
    return None


marks = [("entry/helpers", find("unsigned long long entry_mac(")), ("exact_draw", find("__device__ uint32_t exact_draw(")),
         ("A", find("// ---- A: lane per run")), ("B", find("// ---- B: lane per segment")),
         ("D", find("// ---- D: lane per token")), ("after batch", find("  return nb;")),
         ("arm/stage", find("// Tail-word row staged by one warp")), ("kernel", find("k_sampler(Dev d, Buf cur, Buf nxt, uint32_t iter,")),
         ("end", find("// W / n_k of one item from its topic histogram, block-wide"))]
out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), sys.argv[1], "2000"], capture_output=True,
                     text=True).stdout
agg = {}
for l in out.splitlines():
    m = re.match(r"(\S+):\s+(\d+) stall\s+([\d.]+)% inst\s+([\d.]+)%", l)
    if not m:
        continue
    f, n, st, ins = m.group(1), int(m.group(2)), float(m.group(3)), float(m.group(4))
    key = "other:" + f
    if f == "kernels.cu":
        key = "kernels.cu:other"
        for (name, a), (_, b) in zip(marks, marks[1:]):
            if a and b and a <= n < b:
                key = name
    s = agg.setdefault(key, [0.0, 0.0])
    s[0] += st
    s[1] += ins
for k, (st, ins) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:24s} stall {st:5.1f}%  inst {ins:5.1f}%")
