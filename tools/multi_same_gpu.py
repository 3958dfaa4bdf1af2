"""Run the library's doc-partitioned NCCL path with world = 2 on ONE GPU (both ranks on
device 0) and compare with the single-rank chain: topics (concatenated shards) and W must be
bit-identical.  NCCL may refuse two ranks on one device; then the reason is printed.

    python tools/multi_same_gpu.py
"""
import os
import sys

import numpy as np
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

N_DOCS, V, K, ITERS = 400, 3000, 64, 4


def corpus():
    from paper_2007_08725_b200.synth import planted_corpus_np

    return planted_corpus_np(N_DOCS, V, 90.0, 0.5, seed=13)


def worker(rank, world, nccl_id, q):
    try:
        import torch

        torch.cuda.set_device(0)
        from paper_2007_08725_b200 import lda
        from paper_2007_08725_b200.synth import SAMPLER_SEED

        w, d = corpus()
        L = np.bincount(d, minlength=N_DOCS)
        b = lda.partition_docs(L, world)
        cum = np.concatenate([[0], np.cumsum(L)])
        t0, t1 = int(cum[b[rank]]), int(cum[b[rank + 1]])
        ez = lda.EzLDA(w[t0:t1], d[t0:t1] - b[rank], b[rank + 1] - b[rank], V, K, seed=SAMPLER_SEED, rank=rank,
                       world=world, nccl_id=nccl_id, token_base=t0)
        ez.iterate(ITERS)
        q.put((rank, ez.topics(), lda.EzLDA.csr_to_dense(*ez.W_csr(), K), ez.loglik()))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, None, repr(e)))


def main():
    from paper_2007_08725_b200 import lda
    from paper_2007_08725_b200.synth import SAMPLER_SEED

    w, d = corpus()
    ref = lda.EzLDA(w, d, N_DOCS, V, K, seed=SAMPLER_SEED)
    ref.iterate(ITERS)
    z_ref, W_ref, ll_ref = ref.topics(), lda.EzLDA.csr_to_dense(*ref.W_csr(), K), ref.loglik()
    del ref
    nid = lda.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, nid, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r, z, W, ll = q.get(timeout=300)
        res[r] = (z, W, ll)
    for p in ps:
        p.join(timeout=60)
    if res[0][0] is None or res[1][0] is None:
        print("world=2 on one GPU not runnable:", res[0][2] if res[0][0] is None else res[1][2])
        return
    z = np.concatenate([res[0][0], res[1][0]])
    print("topics identical:", np.array_equal(z, z_ref), "W identical (rank 0, rank 1):",
          np.array_equal(res[0][1], W_ref), np.array_equal(res[1][1], W_ref),
          "loglik", res[0][2], res[1][2], ll_ref)


if __name__ == "__main__":
    main()
