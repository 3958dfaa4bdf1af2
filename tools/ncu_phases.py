"""Executed instructions and stall samples of an ncu report aggregated by code region.

    python tools/ncu_phases.py prof.ncu-rep [path/to/kernels.cu]

Regions: every function of kernels.cu / device.cuh (a line belongs to the nearest preceding
function definition), with sample_batch split at its '// ---- X:' phase markers.  Inlined
helpers keep their own names (entry_mac is phase B's MAC and the S' walk's).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys

DEF = re.compile(r"^(?:template\s*<.*>\s*)?(?:static\s+)?(?:__global__|__device__|__host__)[^(;]*?\b(\w+)\s*\(")


def regions(path):
    out = []
    name = "<top>"
    with open(path) as f:
        for i, line in enumerate(f, 1):
            m = DEF.match(line)
            if m:
                name = m.group(1)
            if name == "sample_batch":
                p = re.match(r"\s*// ---- (\w+):", line)
                if p:
                    out.append((i, f"sample_batch.{p.group(1)}"))
                    continue
            if m:
                out.append((i, name))
    return out


def region_of(regs, ln):
    r = "<top>"
    for start, name in regs:
        if start > ln:
            break
        r = name
    return r


OUTER = {"arm_slot", "item_epilogue_warp", "stage_row_warp", "exact_draw", "mpt_token", "doc_tokens_skip_test",
         "flag_run", "item_epilogue"}


def main(rep, src_dir):
    regs = {fn: regions(os.path.join(src_dir, fn)) for fn in ("kernels.cu", "device.cuh")}
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur_file, hdr, line_no = None, None, None
    # an inlined SASS instruction is listed under every source line of its inline chain: keep one
    # attribution per address, preferring the outermost region (a phase, a kernel) over a helper
    occ = collections.defaultdict(list)
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].split("/")[-1]
            continue
        if row[0] in ("Function Name",):
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None:
            continue
        if row[0].strip():
            line_no = int(row[0])
        if len(row) > 7 and row[2].strip() and row[2] != "..." and row[2] != "-":
            try:
                st, ex = float(row[4] or 0), float(row[7] or 0)
            except ValueError:
                continue
            reg = region_of(regs[cur_file], line_no) if cur_file in regs else ""
            occ[row[2]].append((cur_file, reg, st, ex))
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    for addr, lst in occ.items():
        def pri(o):
            f, reg, _, _ = o
            if f == "kernels.cu" and (reg.startswith("sample_batch") or reg.startswith("k_") or reg in OUTER):
                return 0
            return 1 if f == "kernels.cu" else 2
        f, reg, st, ex = sorted(lst, key=pri)[0]
        agg[f"{f}:{reg}" if reg else f][0] += st
        agg[f"{f}:{reg}" if reg else f][1] += ex
    tst = sum(v[0] for v in agg.values()) or 1.0
    tex = sum(v[1] for v in agg.values()) or 1.0
    print(f"executed warp-instructions (source attribution) {tex:.4g}")
    for k, (st, ex) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if ex / tex < 0.002 and st / tst < 0.002:
            continue
        print(f"  {k:50s} inst {ex / tex * 100:5.1f}% ({ex:.3g})  stall {st / tst * 100:5.1f}%")


if __name__ == "__main__":
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else os.path.join(here, "paper_2007_08725_b200", "csrc"))
