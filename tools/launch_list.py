"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel totals.

    python tools/launch_list.py gpurun_out/launches_TAG.csv "<command line>"
"""
import collections
import csv
import re
import sys


def main(path, cmd):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = re.sub(r"\(.*$", "", r[4]).strip()
        unit, val = r[13], float(r[14].replace(",", ""))
        ms = val / 1e6 if unit == "ns" else val / 1e3 if unit == "us" else val if unit == "ms" else val * 1e3
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(v[1] for v in agg.values())
    print("# ncu launch list (gpu__time_duration.sum, --clock-control none) of the library's kernels over")
    print(f"# `{cmd}`;")
    print("# cold-cache serialised per-launch times: the SHARE of an iteration is what compares with the live CUDA events")
    print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:70]:70s} {n:8d} {ms:10.2f} {ms / tot * 100:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "bench.py --steps 2 --warmup 3")
