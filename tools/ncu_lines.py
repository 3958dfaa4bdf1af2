"""Per-CUDA-source-line attribution (stall samples, executed instructions) from an ncu report."""
import collections
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur_file = None
    agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
    hdr = None
    line_no = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].split("/")[-1]
            continue
        if row[0] == "Function Name":
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None:
            continue
        d = dict(zip(hdr[:2], row[:2]))
        # cuda,sass rows: "Line No","Source" then sass columns; cuda-only rows have line numbers
        if row[0].strip():
            line_no = row[0]
            src = row[1]
            agg[(cur_file, line_no)][2] = src.strip()[:90]
        if len(row) > 4 and row[2].strip():
            try:
                st = float(row[4] or 0)
                ex = float(row[7] or 0)
            except ValueError:
                continue
            agg[(cur_file, line_no)][0] += st
            agg[(cur_file, line_no)][1] += ex
    tot_st = sum(v[0] for v in agg.values()) or 1
    tot_ex = sum(v[1] for v in agg.values()) or 1
    for (f, ln), (st, ex, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{f}:{ln:>5} stall {st / tot_st * 100:5.1f}% inst {ex / tot_ex * 100:5.1f}% | {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
