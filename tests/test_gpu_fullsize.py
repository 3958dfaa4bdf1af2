"""Parity at the benchmarked sizes: the PubMed-shaped corpus (8.2 M docs, V = 141,043,
738 M tokens, K = 1000) in the launch configuration bench.py times (default options: hybrid
W, 10,000-token regions, 32 MiB doc windows -- about 94 windows, so hot-word items are cut
at window boundaries and the 3-slot pipeline runs over ~200k items).

Two iterations on the GPU.  For each, on sampled tokens the oracle can compute one by one:
the oracle's single-token draw (ezlda_oracle_draw_grid: the three-branch map of SURVEY 8(c),
pinned by Fig 2/4 and brute force) applied to the snapshot -- D[d] and W[v] recounted with
numpy from the GPU's z^{i-1}, What[v] by ezlda_oracle_what_row, u by ezlda_oracle_uniform --
must give the GPU's z^i bit for bit.  The sample is >= 10^5 tokens: every token of ~1,300
random documents, plus 2,000 tokens of the most frequent word spread over the whole corpus
(its items are cut at doc windows and every 10,000 tokens).  Integer state at full size: n_k
and the W rows of every sampled word equal the recount.
"""
import numpy as np
import pytest

from paper_2007_08725_b200.synth import CONFIGS, CORPUS_SEED, SAMPLER_SEED

pytestmark = pytest.mark.gpu


def _w_counts(w, z, V, K, chunk=1 << 26):
    """W[v][k] of (w, z) by chunked bincount (test-side recount, int32)."""
    W = np.zeros(V * K, np.int64)
    for s in range(0, len(w), chunk):
        W += np.bincount(w[s:s + chunk].astype(np.int64) * K + z[s:s + chunk], minlength=V * K)
    return W.reshape(V, K).astype(np.int32)


@pytest.mark.parametrize("config,n_sample_docs", [("pubmed", 1300), ("nytimes", 400)])
def test_full_size_sampled_parity(oracle_mod, config, n_sample_docs):
    """PubMed-shaped (short docs: topic-ordered D rows) and NYTimes-shaped (99.5 M tokens,
    332 tokens per doc: the sector-interleaved D rows, kernels.h d_phys) at full size."""
    import torch

    from paper_2007_08725_b200 import lda
    from paper_2007_08725_b200.synth import planted_corpus_torch

    cfg = CONFIGS[config]
    K, V = cfg.K, cfg.V
    w_t, d_t = planted_corpus_torch(cfg.n_docs, cfg.V, cfg.mean_len, cfg.sigma, cfg.K_true, cfg.zipf_s,
                                    seed=CORPUS_SEED, device="cuda")
    w = w_t.cpu().numpy().view(np.uint32)
    d = d_t.cpu().numpy().view(np.uint32)
    gpu = lda.EzLDA(w_t, d_t, cfg.n_docs, V, K, seed=SAMPLER_SEED)
    del w_t, d_t
    torch.cuda.empty_cache()
    N = len(w)
    assert N > (7e8 if config == "pubmed" else 9e7)
    L = np.bincount(d, minlength=cfg.n_docs)
    dofs = np.concatenate([[0], np.cumsum(L)])
    assert np.all(np.diff(d.astype(np.int64)) >= 0), "recipe emits doc-grouped tokens"

    rng = np.random.default_rng(2024)
    docs = np.sort(rng.choice(cfg.n_docs, size=n_sample_docs, replace=False))
    top = int(np.argmax(np.bincount(w, minlength=V)))
    top_pos = np.nonzero(w == top)[0]
    top_pick = np.sort(rng.choice(top_pos, size=2000, replace=False))
    top_docs = np.unique(d[top_pick])

    def token_index(doc):
        """t_g of the doc's tokens: rank in (doc, word, input position) order (reading #14)."""
        s, e = int(dofs[doc]), int(dofs[doc + 1])
        order = np.lexsort((np.arange(e - s), w[s:e]))
        tg = np.empty(e - s, np.int64)
        tg[order] = s + np.arange(e - s)
        return s, e, tg

    checked = 0
    for it in (1, 2):
        z_prev = gpu.topics()
        gpu.iterate(1)
        z_new = gpu.topics()
        Wc = _w_counts(w, z_prev, V, K)
        nk = Wc.sum(0).astype(np.int32)
        # the GPU's post-iteration integer state at full size
        assert np.array_equal(gpu.n_k(), np.bincount(z_new, minlength=K)), it
        whats = {}

        def what(v):
            if v not in whats:
                whats[v] = oracle_mod.what_row(Wc[v], nk, V, cfg.beta)
            return whats[v]

        mism = 0
        # (a) every token of random documents
        for doc in docs:
            s, e, tg = token_index(int(doc))
            Drow = np.bincount(z_prev[s:e], minlength=K).astype(np.int32)
            ws = w[s:e]
            for v in np.unique(ws):
                idx = np.nonzero(ws == v)[0]
                u = np.array([oracle_mod.uniform(SAMPLER_SEED, it, int(tg[i])) for i in idx])
                topics, _ = oracle_mod.draw_grid(Drow, what(int(v)), cfg.alpha, 2, u)
                mism += int(np.sum(topics != z_new[s + idx]))
                checked += len(idx)
        # (b) tokens of the most frequent word across all doc windows / regions
        pick = set(top_pick.tolist())
        for doc in top_docs:
            s, e, tg = token_index(int(doc))
            Drow = np.bincount(z_prev[s:e], minlength=K).astype(np.int32)
            idx = [i for i in range(e - s) if (s + i) in pick]
            u = np.array([oracle_mod.uniform(SAMPLER_SEED, it, int(tg[i])) for i in idx])
            topics, _ = oracle_mod.draw_grid(Drow, what(top), cfg.alpha, 2, u)
            mism += int(np.sum(topics != z_new[s + np.array(idx)]))
            checked += len(idx)
        assert mism == 0, (it, mism)
        # W rows of the sampled words after the iteration equal the recount of z^i
        Wn = _w_counts(w, z_new, V, K)
        rp, col, val = gpu.W_csr()
        for v in list(whats)[:3000]:
            row = np.zeros(K, np.int32)
            row[col[rp[v]:rp[v + 1]].astype(np.int64)] = val[rp[v]:rp[v + 1]]
            assert np.array_equal(row, Wn[v]), (it, v)
        del Wc, Wn
    print(f"full-size {config}-shaped: {checked} sampled draws over 2 iterations, 0 mismatches")
    assert checked >= 2 * 100_000
