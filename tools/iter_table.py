"""Per-iteration roofline table: ncu metrics of the sampler and the doc pass (one profiled chain,
tools/gpu_r2_itercurve.sh) beside the live CUDA-event curve of the same chain (tools/curve.py).

    python tools/iter_table.py ncu_iters.csv curve.csv [peak_gbs] > table.txt
"""
import csv
import re
import sys


def main(ncu_csv, curve_csv, peak=None):
    if peak is None:
        import json
        import os
        peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                           "MEASURED_PEAKS.json")))["hbm_gbs"]
    launches = {}  # launch id -> (kernel, {metric: value})
    for r in csv.reader(open(ncu_csv)):
        if len(r) < 15 or not r[0].isdigit():
            continue
        k = "k_sampler" if "k_sampler" in r[4] else "k_doc_hist" if "k_doc_hist" in r[4] else None
        if k is None:
            continue
        launches.setdefault(int(r[0]), (k, {}))[1][r[12]] = (r[13], float(r[14].replace(",", "")))
    seq = [launches[i] for i in sorted(launches)]
    # create launches the sampler once (count mode); then each iteration: doc pass, sampler
    if seq and seq[0][0] == "k_sampler":
        seq = seq[1:]
    it_of = {}
    for n, (k, m) in enumerate(seq):
        it_of[(n // 2 + 1, k)] = m
    curve = {int(r["iteration"]): r for r in csv.DictReader(open(curve_csv))}

    def v(m, name, scale=1.0):
        u, x = m[name]
        f = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6,
             "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(u, 1.0)
        return x * f * scale

    print(f"# peak {peak} GB/s")
    print(f"{'it':>4} {'kernel':12s} {'ncu_ms':>7} {'live_ms':>8} {'model_GB':>9} {'DRAM_GB':>8} {'frac':>6} {'L2hit%':>7}"
          f" {'LSU%':>6} {'Ginst':>7} {'skip_S':>7}")
    for it in (1, 10, 50, 100, 200):
        c = curve.get(it)
        for k in ("k_sampler", "k_doc_hist"):
            m = it_of.get((it, k))
            if m is None or c is None:
                continue
            ms = v(m, "gpu__time_duration.sum")
            dram = v(m, "dram__bytes_read.sum") + v(m, "dram__bytes_write.sum")
            live = float(c["ms_sampler_kernel"] if k == "k_sampler" else c["ms_docpass"])
            gb = float(c["sampler_model_GB"] if k == "k_sampler" else c["docpass_model_GB"])
            frac = gb / (live / 1e3) / peak
            l2 = m["lts__t_sector_hit_rate.pct"][1]
            lsu = m.get("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", ("", float("nan")))[1]
            gi = m["sm__inst_executed.sum"][1] / 1e9
            print(f"{it:4d} {k:12s} {ms:7.2f} {live:8.2f} {gb:9.2f} {dram:8.2f} {frac:6.3f} {l2:7.1f} {lsu:6.1f}"
                  f" {gi:7.2f} {float(c['skip_S']):7.4f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None)
