"""Run create + W warm-up iterations + 1 profiled iteration (for ncu / compute-sanitizer).

    python tools/profile_iter.py --config pubmed --warmup 3
Kernel launch order: create launches k_init_topics, k_sampler<true> (count mode); each
iteration launches k_den, k_word_prep, k_doc_block (if long docs), k_doc_hist/k_doc_warp,
k_sampler<false>.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="pubmed")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--iters", type=int, default=1)
    ap.add_argument("--np", action="store_true", help="numpy generator (small configs)")
    args = ap.parse_args()
    import torch

    from paper_2007_08725_b200 import lda
    from paper_2007_08725_b200.synth import CONFIGS, SAMPLER_SEED, corpus

    cfg = CONFIGS[args.config]
    w, d = corpus(args.config, backend="np" if args.np else "torch")
    ez = lda.EzLDA(w, d, cfg.n_docs, cfg.V, cfg.K, seed=SAMPLER_SEED)
    ez.iterate(args.warmup)
    ez.stats_sum(reset=True)
    t = time.perf_counter()
    ez.iterate(args.iters)
    st = ez.stats_sum()
    print(f"{args.config}: iterations {args.warmup + 1}..{args.warmup + args.iters} "
          f"{(time.perf_counter() - t) * 1e3 / args.iters:.1f} ms/iter wall; phases ms "
          f"wordprep {st['ms_wordprep']:.2f} docpass {st['ms_docpass']:.2f} sample {st['ms_sample']:.2f}; "
          f"skip_S {st['skip_S'] / st['n_tokens']:.4f} active_runs {st['active_runs']}")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
