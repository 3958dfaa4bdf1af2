"""Rank SASS instructions of an ncu report by shared-memory wavefronts; print LSU totals."""
import csv
import io
import subprocess
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))[1:]
    h = r[0]
    rows = [dict(zip(h, x)) for x in r[1:]]
    tot = sum(f(x["L1 Wavefronts Shared"]) for x in rows)
    ideal = sum(f(x["L1 Wavefronts Shared Ideal"]) for x in rows)
    print(f"shared wavefronts {tot:.4g} (ideal {ideal:.4g})")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    for a, b, c in zip(rr[0], rr[1], rr[2]):
        if a in ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
                 "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                 "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                 "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
                 "sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                 "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"):
            print(f"  {a} {c} {b}")
    rows.sort(key=lambda x: -f(x["L1 Wavefronts Shared"]))
    for x in rows[:top]:
        w = f(x["L1 Wavefronts Shared"])
        print(f"{100 * w / tot:6.2f}%  wf/exec {w / max(1.0, f(x['Instructions Executed'])):5.2f}  "
              f"exec {f(x['Instructions Executed']):.3g}  {x['Source'].strip()[:60]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
