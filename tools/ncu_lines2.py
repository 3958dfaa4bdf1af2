"""Per-CUDA-source-line warp-instructions and stall samples of an ncu report (needs -lineinfo).
    python tools/ncu_lines2.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, data = "", []
hdr = None
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0]:
        try:
            data.append((fname, int(r[0]), float(r[7] or 0), float(r[4] or 0), r[1],
                         {hdr[i][6:]: float(r[i] or 0) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]}))
        except ValueError:
            pass
ti = sum(d[2] for d in data) or 1; ts = sum(d[3] for d in data) or 1
print(f"total warp-instr {ti:.4g}  stall samples {ts:.4g}")
for f, ln, i, s, src, st in sorted(data, key=lambda d: -d[3])[:top]:
    tops = ",".join(f"{k}{v/max(s,1)*100:.0f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:2])
    print(f"{f[:9]}:{ln:<4d} inst {i/ti*100:5.1f}% stall {s/ts*100:5.1f}% [{tops}] | {src.strip()[:95]}")
