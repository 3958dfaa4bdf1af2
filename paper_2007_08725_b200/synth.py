"""Seeded synthetic LDA corpora shaped like the paper's workloads.

This module holds NO arithmetic of the method (no sampling of topics for the
Gibbs chain, no counts, no Philox): it only draws the input token lists
(word id, doc id) that both the CUDA path and the CPU oracle consume.

Recipe:
  * planted LDA with K_true = 100 topics: phi_k ∝ zipf(s) ⊙ Gamma(0.3) over V
    words (Zipf word marginal, the paper's power law, Fig 8 / P:1086),
    theta_d ~ Dir(0.1), z ~ theta_d, w ~ phi_z;
  * document lengths lognormal(mu, sigma) with mu chosen so the mean is L̄,
    rounded and clipped to [1, 65535] (16-bit packing limit);
  * vocabulary ids randomly permuted so that word id order != frequency order
    (exercises the frequency relabelling of P:765);
  * tokens are emitted doc-grouped (doc ids non-decreasing), each doc's tokens
    in generation order.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

CORPUS_SEED = 20200717
SAMPLER_SEED = 1


@dataclass(frozen=True)
class CorpusConfig:
    name: str
    n_docs: int
    V: int
    mean_len: float
    sigma: float
    K: int
    K_true: int = 100
    zipf_s: float = 1.0

    @property
    def alpha(self) -> float:
        return 50.0 / self.K

    beta: float = 0.01


# BASELINE.json configs (token counts are approximate: n_docs * mean_len)
CONFIGS = {
    "tiny": CorpusConfig("tiny", 100, 500, 100.0, 0.5, 16),
    "small": CorpusConfig("small", 2000, 5000, 90.0, 0.5, 64),
    "nytimes": CorpusConfig("nytimes", 299_752, 101_636, 332.0, 1.0, 1000),
    "nytimes_k5k": CorpusConfig("nytimes_k5k", 299_752, 101_636, 332.0, 1.0, 5000),
    "nytimes_k10k": CorpusConfig("nytimes_k10k", 299_752, 101_636, 332.0, 1.0, 10000),
    "nytimes_k32k": CorpusConfig("nytimes_k32k", 299_752, 101_636, 332.0, 1.0, 32768),
    "pubmed": CorpusConfig("pubmed", 8_200_000, 141_043, 90.0, 0.5, 1000),
    "clueweb": CorpusConfig("clueweb", 6_000_000, 1_000_000, 500.0, 1.0, 10000),
    # one rank's shard of the ClueWeb-shaped corpus at P = 8 (750k docs, ~375 M tokens, the
    # global vocabulary): the per-GPU workload of the 8 x B200 configuration
    "clueweb_shard8": CorpusConfig("clueweb_shard8", 750_000, 1_000_000, 500.0, 1.0, 10000),
}


def doc_lengths(rng: np.random.Generator, n_docs: int, mean_len: float, sigma: float) -> np.ndarray:
    mu = math.log(mean_len) - 0.5 * sigma * sigma
    L = np.rint(rng.lognormal(mu, sigma, size=n_docs))
    return np.clip(L, 1, 65535).astype(np.int64)


def planted_corpus_np(n_docs: int, V: int, mean_len: float, sigma: float, K_true: int = 100,
                      zipf_s: float = 1.0, doc_alpha: float = 0.1, gamma_shape: float = 0.3,
                      seed: int = CORPUS_SEED, permute_vocab: bool = True):
    """numpy generator for small corpora (CPU tests, oracle).  Returns (word_ids u32, doc_ids u32)."""
    rng = np.random.default_rng(seed)
    zipf = 1.0 / np.arange(1, V + 1, dtype=np.float64) ** zipf_s
    phi = zipf[None, :] * rng.gamma(gamma_shape, 1.0, size=(K_true, V))
    phi /= phi.sum(axis=1, keepdims=True)
    L = doc_lengths(rng, n_docs, mean_len, sigma)
    theta = rng.dirichlet(np.full(K_true, doc_alpha), size=n_docs)
    n = int(L.sum())
    doc_ids = np.repeat(np.arange(n_docs, dtype=np.int64), L)
    # z ~ theta_d : inverse CDF per token
    cdf_t = np.cumsum(theta, axis=1)
    cdf_t[:, -1] = 1.0
    u = rng.random(n)
    z = np.empty(n, dtype=np.int64)
    for d0 in range(0, n_docs, 4096):  # chunked to bound memory
        d1 = min(n_docs, d0 + 4096)
        s, e = int(L[:d0].sum()) if d0 else 0, int(L[:d1].sum())
        rows = cdf_t[doc_ids[s:e]]
        z[s:e] = (rows < u[s:e, None]).sum(axis=1)
    z = np.minimum(z, K_true - 1)
    # w ~ phi_z
    cdf_w = np.cumsum(phi, axis=1)
    cdf_w[:, -1] = 1.0
    u2 = rng.random(n)
    w = np.empty(n, dtype=np.int64)
    for k in range(K_true):
        idx = np.nonzero(z == k)[0]
        if idx.size:
            w[idx] = np.searchsorted(cdf_w[k], u2[idx], side="right")
    w = np.minimum(w, V - 1)
    if permute_vocab:
        w = rng.permutation(V)[w]
    return w.astype(np.uint32), doc_ids.astype(np.uint32)


def planted_corpus_torch(n_docs: int, V: int, mean_len: float, sigma: float, K_true: int = 100,
                         zipf_s: float = 1.0, doc_alpha: float = 0.1, gamma_shape: float = 0.3,
                         seed: int = CORPUS_SEED, device: str = "cuda", permute_vocab: bool = True):
    """torch generator for the large configs (same recipe, drawn on `device`).

    Returns (word_ids, doc_ids) as int32 tensors on `device` (values < 2^31)."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    f64 = torch.float64
    zipf = 1.0 / torch.arange(1, V + 1, device=device, dtype=f64) ** zipf_s
    gam = torch._standard_gamma(torch.full((K_true, V), gamma_shape, device=device, dtype=torch.float32),
                                generator=gen).to(f64)
    phi = zipf[None, :] * gam
    cdf_w = torch.cumsum(phi / phi.sum(dim=1, keepdim=True), dim=1)
    cdf_w[:, -1] = 1.0
    mu = math.log(mean_len) - 0.5 * sigma * sigma
    normals = torch.randn(n_docs, device=device, dtype=f64, generator=gen)
    L = torch.clamp(torch.round(torch.exp(mu + sigma * normals)), 1, 65535).to(torch.int64)
    theta = torch._standard_gamma(torch.full((n_docs, K_true), doc_alpha, device=device, dtype=torch.float32),
                                  generator=gen)
    theta = theta / theta.sum(dim=1, keepdim=True).clamp_min(1e-30)
    cdf_t = torch.cumsum(theta, dim=1)
    cdf_t[:, -1] = 1.0
    n = int(L.sum().item())
    doc_ids = torch.repeat_interleave(torch.arange(n_docs, device=device, dtype=torch.int32), L)
    z = torch.empty(n, device=device, dtype=torch.int32)
    chunk = 1 << 22
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        d = doc_ids[s:e].long()
        u = torch.rand(e - s, device=device, dtype=torch.float32, generator=gen)
        z[s:e] = torch.searchsorted(cdf_t[d], u[:, None], right=True).squeeze(1).clamp_max(K_true - 1).int()
    del cdf_t, theta
    w = torch.empty(n, device=device, dtype=torch.int32)
    order = torch.argsort(z, stable=True)
    zs = z[order]
    bounds = torch.searchsorted(zs, torch.arange(K_true + 1, device=device, dtype=torch.int32))
    bounds = bounds.tolist()
    for k in range(K_true):
        s, e = bounds[k], bounds[k + 1]
        if e > s:
            u = torch.rand(e - s, device=device, dtype=f64, generator=gen)
            w[order[s:e]] = torch.searchsorted(cdf_w[k], u, right=True).clamp_max(V - 1).int()
    del order, zs, z
    if permute_vocab:
        perm = torch.randperm(V, device=device, generator=gen).int()
        w = perm[w.long()]
    return w, doc_ids


def corpus(name: str, backend: str = "np", device: str = "cuda", seed: int = CORPUS_SEED):
    c = CONFIGS[name]
    if backend == "np":
        return planted_corpus_np(c.n_docs, c.V, c.mean_len, c.sigma, c.K_true, c.zipf_s, seed=seed)
    return planted_corpus_torch(c.n_docs, c.V, c.mean_len, c.sigma, c.K_true, c.zipf_s, seed=seed, device=device)


def random_state(rng: np.random.Generator, K: int, density: float = 0.5, max_count: int = 5,
                 gamma_shape: float = 0.5):
    """A random (D row, What row) pair for sampler property tests: sparse integer D row,
    Gamma(0.5) What row."""
    D = rng.integers(1, max_count + 1, size=K) * (rng.random(K) < density)
    What = rng.gamma(gamma_shape, 1.0, size=K) + 1e-6
    return D.astype(np.int32), What.astype(np.float64)
