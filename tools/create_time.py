"""Time ezlda_create on the PubMed-shaped corpus (device input and pinned host input)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2007_08725_b200 import lda
    from paper_2007_08725_b200.synth import CONFIGS, SAMPLER_SEED, corpus

    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "pubmed"]
    w, d = corpus(cfg.name, backend="torch")
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ez = lda.EzLDA(w, d, cfg.n_docs, cfg.V, cfg.K, seed=SAMPLER_SEED)
        torch.cuda.synchronize()
        print(f"create (device input) {time.perf_counter() - t:.3f} s")
        del ez
    hw = torch.empty(w.shape, dtype=w.dtype, pin_memory=True)
    hd = torch.empty(d.shape, dtype=d.dtype, pin_memory=True)
    hw.copy_(w)
    hd.copy_(d)
    del w, d
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    t = time.perf_counter()
    ez = lda.EzLDA(hw, hd, cfg.n_docs, cfg.V, cfg.K, seed=SAMPLER_SEED)
    torch.cuda.synchronize()
    print(f"create (pinned host input) {time.perf_counter() - t:.3f} s")


if __name__ == "__main__":
    main()
