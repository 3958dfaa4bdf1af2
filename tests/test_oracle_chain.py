"""Oracle chain pinned by invariants, closed forms and brute force."""
import math

import numpy as np
import pytest

from paper_2007_08725_b200.synth import planted_corpus_np

TINY = dict(n_docs=100, V=500, mean_len=100.0, sigma=0.5)


@pytest.fixture(scope="module")
def tiny():
    return planted_corpus_np(**TINY)


def brute_counts(w, d, z, n_docs, V, K):
    D = np.zeros((n_docs, K), np.int64)
    W = np.zeros((V, K), np.int64)
    np.add.at(D, (d.astype(np.int64), z.astype(np.int64)), 1)
    np.add.at(W, (w.astype(np.int64), z.astype(np.int64)), 1)
    return D, W


def test_token_index_is_doc_word_position_rank(oracle_mod, tiny):
    w, d = tiny
    h = oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], 16, token_base=1000)
    tg = h.token_index()
    order = np.lexsort((np.arange(len(w)), w, d))  # (doc, word, position)
    expect = np.empty(len(w), np.uint64)
    expect[order] = 1000 + np.arange(len(w), dtype=np.uint64)
    assert np.array_equal(tg, expect)


def test_init_topics_follow_philox(oracle_mod, tiny):
    w, d = tiny
    K = 16
    h = oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], K, seed=77)
    tg = h.token_index()
    z = h.topics()
    for t in range(0, len(w), 97):
        r0 = oracle_mod.philox4x32_10([int(tg[t]) & 0xFFFFFFFF, int(tg[t]) >> 32, 0, 0], [77, 0])[0]
        assert z[t] == (r0 * K) >> 32


def test_count_invariants_and_brute_force(oracle_mod, tiny):
    w, d = tiny
    n_docs, V, K = TINY["n_docs"], TINY["V"], 16
    h = oracle_mod.OracleLDA(w, d, n_docs, V, K)
    h.iterate(3)
    z = h.topics()
    D, W, nk = h.counts()
    Db, Wb = brute_counts(w, d, z, n_docs, V, K)
    assert np.array_equal(D, Db) and np.array_equal(W, Wb)
    assert np.array_equal(D.sum(1), np.bincount(d, minlength=n_docs))
    assert np.array_equal(W.sum(1), np.bincount(w, minlength=V))
    assert np.array_equal(W.sum(0), nk) and np.array_equal(D.sum(0), nk)
    assert nk.sum() == len(w)


def test_chain_independent_of_g(oracle_mod, tiny):
    """T identical for g in {1,2,3} and the appendix bound (exact skipping)."""
    w, d = tiny
    ref = None
    for g in (2, 1, 3, 0):
        h = oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], 16, g=g)
        h.iterate(6)
        z = h.topics()
        if ref is None:
            ref = z
        else:
            assert np.array_equal(z, ref), g


def test_llpt_dense_equals_identity(oracle_mod, tiny):
    w, d = tiny
    h = oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], 16)
    for _ in range(3):
        h.iterate(2)
        a, b = h.loglik(0), h.loglik(1)
        assert abs(a - b) <= 1e-12 * abs(a)


def test_llpt_K1_unigram_closed_form(oracle_mod, tiny):
    w, d = tiny
    V, beta = TINY["V"], 0.01
    h = oracle_mod.OracleLDA(w, d, TINY["n_docs"], V, 1, alpha=50.0, beta=beta)
    h.iterate(1)
    assert np.all(h.topics() == 0)
    c = np.bincount(w, minlength=V).astype(np.float64)
    N = len(w)
    expect = np.mean(np.log2((c[w] + beta) / (N + V * beta)))
    assert abs(h.loglik(0) - expect) < 1e-12 * abs(expect)
    assert abs(h.loglik(1) - expect) < 1e-12 * abs(expect)


def test_llpt_single_token_is_zero(oracle_mod):
    h = oracle_mod.OracleLDA(np.array([0], np.uint32), np.array([0], np.uint32), 1, 1, 1, alpha=50.0)
    assert h.loglik(0) == 0.0 and h.loglik(1) == 0.0


def test_llpt_of_appendix_a_state(oracle_mod):
    """Derived value -1.963006 bits/token for the Fig 1/2 state."""
    app = [(0, 0, 2), (0, 2, 1), (1, 1, 1), (1, 2, 0), (2, 0, 1), (2, 2, 3), (3, 1, 0)]
    w = np.array([t[0] for t in app], np.uint32)
    d = np.array([t[1] for t in app], np.uint32)
    h = oracle_mod.OracleLDA(w, d, 3, 4, 4, alpha=16.7, beta=0.01)
    h.set_topics(np.array([t[2] for t in app], np.uint16), 0)
    assert abs(h.loglik(0) - (-1.963006)) < 1e-6


def test_convergence_qualitative(oracle_mod, tiny):
    """LLPT rises then flattens; skip fraction grows with iterations."""
    w, d = tiny
    h = oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], 16)
    ll, skip = [], []
    for _ in range(30):
        h.iterate(1)
        ll.append(h.loglik(1))
        skip.append(h.last_stats()["skip_final"] / len(w))
    assert ll[-1] > ll[0] + 0.1
    assert np.mean(skip[-5:]) > np.mean(skip[:3])
    st = h.last_stats()
    assert st["skip_S"] <= st["skip_final"] == st["branch_hist"][0] + st["branch_hist"][1]


def split_docs(d, n_docs, P):
    """Contiguous doc ranges balanced by tokens (the multi-GPU partition)."""
    L = np.bincount(d, minlength=n_docs)
    cum = np.concatenate([[0], np.cumsum(L)])
    bounds = [0]
    for r in range(1, P):
        bounds.append(int(np.searchsorted(cum, cum[-1] * r / P)))
    bounds.append(n_docs)
    return bounds, cum


@pytest.mark.parametrize("P", [2, 3])
def test_shard_emulation_equals_single(oracle_mod, tiny, P):
    """P doc shards + summed W snapshot reproduce the single-shard chain bit for bit."""
    w, d = tiny
    n_docs, V, K = TINY["n_docs"], TINY["V"], 16
    ref = oracle_mod.OracleLDA(w, d, n_docs, V, K)
    bounds, cum = split_docs(d, n_docs, P)
    shards = []
    for r in range(P):
        t0, t1 = int(cum[bounds[r]]), int(cum[bounds[r + 1]])
        shards.append(oracle_mod.OracleLDA(w[t0:t1], d[t0:t1] - bounds[r], bounds[r + 1] - bounds[r], V, K,
                                           token_base=t0))
    assert np.array_equal(np.concatenate([s.topics() for s in shards]), ref.topics())
    for _ in range(4):
        Wg = sum(s.counts()[1] for s in shards)
        ng = Wg.sum(0).astype(np.int32)
        for s in shards:
            s.iterate(1, Wg, ng)
        ref.iterate(1)
        assert np.array_equal(np.concatenate([s.topics() for s in shards]), ref.topics())


def test_two_branch_chain_invariants_and_convergence(oracle_mod, tiny):
    """Two-branch (ESCA) chain mode (Alg P:1481-1507): exact counts, no skipping,
    every token drawn in the S or Q branch, and the LLPT rises like the three-branch chain's."""
    w, d = tiny
    n_docs, V, K = TINY["n_docs"], TINY["V"], 16
    h = oracle_mod.OracleLDA(w, d, n_docs, V, K, branches=2)
    h3 = oracle_mod.OracleLDA(w, d, n_docs, V, K)
    assert np.array_equal(h.topics(), h3.topics())  # same iteration-0 state
    ll, ll3 = [], []
    for _ in range(20):
        h.iterate(1)
        h3.iterate(1)
        ll.append(h.loglik(1))
        ll3.append(h3.loglik(1))
        st = h.last_stats()
        assert st["skip_S"] == st["skip_final"] == 0
        assert st["branch_hist"][0] == st["branch_hist"][1] == 0
        assert st["branch_hist"][2] + st["branch_hist"][3] == len(w)
    z = h.topics()
    D, W, nk = h.counts()
    Db, Wb = brute_counts(w, d, z, n_docs, V, K)
    assert np.array_equal(D, Db) and np.array_equal(W, Wb)
    assert ll[-1] > ll[0] + 0.1
    # same conditional, different u -> topic maps: different chains, similar likelihood
    assert not np.array_equal(z, h3.topics())
    assert abs(np.mean(ll[-5:]) - np.mean(ll3[-5:])) < 0.1 * abs(np.mean(ll3[-5:]))


def test_two_branch_K1_all_zero(oracle_mod, tiny):
    w, d = tiny
    h = oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], 1, branches=2)
    h.iterate(2)
    assert not h.topics().any()
    with pytest.raises(ValueError):
        oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], 4, branches=1)


@pytest.mark.parametrize("branches, g", [(3, 2), (3, 1), (2, 2)])
def test_iterate_is_per_token_draw_on_recounted_snapshot(oracle_mod, tiny, branches, g):
    """Composition pin of the chain: every topic of one iterate() step equals the single-token
    draw (draw_three_branch / draw_two_branch, pinned by Fig 2/4 and the brute-force u-measure)
    applied to the recounted snapshot D[d], What[v] (numpy recount) with u = uniform(seed, i, t_g)
    -- the snapshot semantics of SURVEY 8(c) steps 1-4."""
    w, d = tiny
    n_docs, V, K = TINY["n_docs"], TINY["V"], 16
    seed = 5
    h = oracle_mod.OracleLDA(w, d, n_docs, V, K, seed=seed, g=g, branches=branches)
    h.iterate(2)
    z_prev = h.topics()
    i = h.iterations + 1
    Db, Wb = brute_counts(w, d, z_prev, n_docs, V, K)
    nk = Wb.sum(0)
    tg = h.token_index()
    h.iterate(1)
    z_new = h.topics()
    whats = {}
    for t in range(len(w)):
        v = int(w[t])
        if v not in whats:
            whats[v] = oracle_mod.what_row(Wb[v], nk, V, h.beta)
        u = oracle_mod.uniform(seed, i, int(tg[t]))
        if branches == 3:
            topic = oracle_mod.draw_three_branch(Db[d[t]], whats[v], h.alpha, g, u)["topic"]
        else:
            topic = oracle_mod.draw_two_branch(Db[d[t]], whats[v], h.alpha, u)["topic"]
        assert topic == z_new[t], (t, topic, z_new[t])


@pytest.mark.parametrize("branches", [3, 2])
def test_openmp_build_is_identical(oracle_mod, tiny, branches):
    """The OpenMP build of the oracle (bench.py's all-core CPU leg) splits the per-word loop
    over threads; every draw reads only the snapshot, so topics and counters are identical."""
    w, d = tiny
    a = oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], 16, branches=branches)
    b = oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], 16, branches=branches, omp=True)
    for _ in range(4):
        a.iterate(1)
        b.iterate(1)
        assert np.array_equal(a.topics(), b.topics())
        assert a.last_stats() == b.last_stats()
