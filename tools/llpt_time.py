"""Time ezlda_loglik (LLPT, Eq 5) on a config after a few iterations."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2007_08725_b200 import lda
from paper_2007_08725_b200.synth import CONFIGS, SAMPLER_SEED, corpus
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "pubmed"]
w, d = corpus(cfg.name, backend="torch")
ez = lda.EzLDA(w, d, cfg.n_docs, cfg.V, cfg.K, seed=SAMPLER_SEED)
ez.iterate(3)
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ll = ez.loglik()
    torch.cuda.synchronize()
    print(f"{cfg.name}: llpt {ll:.9f} in {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
