import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2007_08725_b200 import lda
from paper_2007_08725_b200.synth import CONFIGS, SAMPLER_SEED, corpus
cfg = CONFIGS["pubmed"]
w, d = corpus("pubmed", backend="torch")
hw = torch.empty(w.shape, dtype=w.dtype, pin_memory=True); hw.copy_(w)
hd = torch.empty(d.shape, dtype=d.dtype, pin_memory=True); hd.copy_(d)
del w, d
torch.cuda.empty_cache(); torch.cuda.synchronize()
for rep in range(4):
    t = time.perf_counter()
    ez = lda.EzLDA(hw, hd, cfg.n_docs, cfg.V, cfg.K, seed=SAMPLER_SEED)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ez.iterate(3)
    torch.cuda.synchronize()
    print(f"rep {rep}: create {t1 - t:.3f} s, 3 iterations {time.perf_counter() - t1:.3f} s", flush=True)
    del ez
