"""Summarise an ncu report: key metrics, stall reasons, top SASS basic blocks."""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Compute (SM) Throughput",
        "Issue Slots Busy", "Executed Ipc Active", "Achieved Occupancy", "Registers Per Thread",
        "Avg. Active Threads Per Warp", "Executed Instructions", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "Branch Efficiency", "Grid Size", "Dynamic Shared Memory Per Block",
        "Theoretical Occupancy", "SM Frequency"]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep, nblocks=15):
    out = run([rep, "--page", "details", "--csv"])
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    kern = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if kern != d.get("Kernel Name"):
            kern = d.get("Kernel Name")
            print("==", kern[:100])
        if d.get("Metric Name") in KEYS:
            print(f"  {d['Metric Name']:38s} {d['Metric Value']} {d['Metric Unit']}")
    raw = run([rep, "--page", "raw", "--csv"])
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        h, u, v = rr[0], rr[1], rr[2]
        for i, name in enumerate(h):
            if re.match(r"dram__bytes_(read|write)\.sum$", name) or name in ("lts__t_sector_hit_rate.pct",):
                print(f"  {name:38s} {v[i]} {u[i]}")
    sass = run([rep, "--page", "source", "--csv", "--print-source", "sass"])
    rows = list(csv.reader(io.StringIO(sass)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    ie = idx["Instructions Executed"]
    tot = sum(float(r[ie] or 0) for r in data)
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    st = {c: sum(float(r[idx[c]] or 0) for r in data) for c in cols}
    s = sum(st.values()) or 1
    print("  stalls:", ", ".join(f"{c[6:]} {v / s * 100:.1f}%" for c, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
    blocks, cur = [], None
    for r in data:
        c = float(r[ie] or 0)
        samp = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        if cur and c == cur["c"]:
            cur["n"] += 1
            cur["ops"].append(r[idx["Source"]].strip())
            cur["samp"] += samp
        else:
            cur = {"addr": r[idx["Address"]], "c": c, "n": 1, "ops": [r[idx["Source"]].strip()], "samp": samp}
            blocks.append(cur)
    ssum = sum(b["samp"] for b in blocks) or 1
    print(f"  total executed warp-instructions {tot:.4g}")
    for b in sorted(blocks, key=lambda b: -b["samp"])[:nblocks]:
        print(f"  {b['addr'][-5:]} n={b['n']:3d} exec={b['c']:.3g} inst%={b['c'] * b['n'] / tot * 100:5.2f} "
              f"stall%={b['samp'] / ssum * 100:5.2f} | " + " ; ".join(o[:30] for o in b["ops"][:6]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 15)
