"""Per-iteration curve: ms/iteration, tokens/s, skip fractions, phase times, LLPT every --llpt-every.

    python tools/curve.py --config pubmed --iters 100 [--llpt-every 10] [--csv out.csv]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="pubmed")
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--llpt-every", type=int, default=10)
    ap.add_argument("--csv", default=None)
    args = ap.parse_args()
    import torch

    from paper_2007_08725_b200 import lda
    from paper_2007_08725_b200.synth import CONFIGS, SAMPLER_SEED, corpus

    cfg = CONFIGS[args.config]
    w, d = corpus(args.config, backend="torch")
    N = w.shape[0]
    ez = lda.EzLDA(w, d, cfg.n_docs, cfg.V, cfg.K, seed=SAMPLER_SEED)
    import json
    peak = None
    try:
        peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                 "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    rows = ["iteration,ms,tokens_per_s,skip_S,skip_final,ms_wordprep,ms_docpass,ms_sample,active_runs,llpt,"
            "ms_sampler_kernel,sampler_model_GB,sampler_frac,docpass_model_GB,docpass_frac"]
    tot_ms = 0.0
    for i in range(1, args.iters + 1):
        ez.iterate(1)
        st = ez.stats()
        ll = ez.loglik() if (args.llpt_every and i % args.llpt_every == 0) else float("nan")
        tot_ms += st["ms_total"]
        rows.append(f"{i},{st['ms_total']:.3f},{N / st['ms_total'] * 1e3:.4g},{st['skip_S'] / N:.4f},"
                    f"{st['skip_final'] / N:.4f},{st['ms_wordprep']:.3f},{st['ms_docpass']:.3f},{st['ms_sample']:.3f},"
                    f"{st['active_runs']},{ll:.6f},{st['ms_sampler_kernel']:.3f},{st['model_bytes_sample'] / 1e9:.3f},"
                    f"{(st['model_bytes_sample'] / st['ms_sampler_kernel'] / 1e6 / peak) if peak else float('nan'):.4f},"
                    f"{st['model_bytes_docpass'] / 1e9:.3f},"
                    f"{(st['model_bytes_docpass'] / st['ms_docpass'] / 1e6 / peak) if peak else float('nan'):.4f}")
        if i in (1, 2, 5, 10, 20, 30, 50, 75, 100, 150, 200) or i == args.iters:
            print(rows[-1], flush=True)
    print(f"mean tokens/s over iterations 1..{args.iters}: {N * args.iters / tot_ms * 1e3:.4g}")
    if args.csv:
        with open(args.csv, "w") as f:
            f.write("\n".join(rows) + "\n")


if __name__ == "__main__":
    main()
