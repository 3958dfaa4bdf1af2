"""Small end-to-end run of the library for compute-sanitizer (memcheck / racecheck / synccheck):
tiny planted corpora at K = 16 (small-K kernels) and K = 5000 (large-K kernels, HBM slot
histograms, Q' table in HBM), create + 3 iterations + counts + set_topics + loglik, and the
two-branch mode.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2007_08725_b200 import lda  # noqa: E402
from paper_2007_08725_b200.synth import SAMPLER_SEED, planted_corpus_np  # noqa: E402


def run(n_docs, V, mean_len, K, **kw):
    w, d = planted_corpus_np(n_docs=n_docs, V=V, mean_len=mean_len, sigma=0.8, K_true=20, seed=3)
    g = lda.EzLDA(w, d, n_docs, V, K, seed=SAMPLER_SEED, **kw)
    g.iterate(3)
    z = g.topics()
    g.W_csr()
    g.D_csr()
    g.set_topics(z, 3)
    g.iterate(1)
    ll = g.loglik()
    st = g.stats()
    g.close()
    print(f"K={K} {kw}: {len(w)} tokens, llpt {ll:.6f}, sampled {st['sampled']}, exact {st['exact_redraws']}")


if __name__ == "__main__":
    run(60, 400, 80.0, 16)
    run(60, 400, 80.0, 16, sampler=2)
    run(20, 800, 700.0, 5000)
    run(60, 400, 80.0, 16, debug_flags=3)
    print("sanitize run done")
