"""GPU (CUDA path through the C ABI) vs the CPU oracle, element by element.

One-step parity (BASELINE.json north star): every iteration the oracle is fed the
GPU's z^{i-1}; both run iteration i with the same Philox stream, and the GPU's
integer D / W / n_k must equal a brute-force recount of its own topics bit for bit.
Topics: the north star's bar is >= 99.99% agreement with every disagreement at a bucket
boundary (checked: within 1e-12 Z).  The CUDA path is built to meet a stronger bar -- its
fast path sums exact 64-bit fixed-point products and keeps only decisions certified by an
error margin, redrawing the others with the oracle's fp64 operations and orders (DESIGN.md
section 2) -- so the tests also require ZERO disagreements (bit-identical topics).
"""
import numpy as np
import pytest

from paper_2007_08725_b200.synth import SAMPLER_SEED, planted_corpus_np

pytestmark = pytest.mark.gpu

TINY = dict(n_docs=100, V=500, mean_len=100.0, sigma=0.5)
SMALL = dict(n_docs=2000, V=5000, mean_len=90.0, sigma=0.5)


@pytest.fixture(scope="module")
def ez():
    from paper_2007_08725_b200 import lda

    lda.load()
    return lda


@pytest.fixture(scope="module")
def tiny():
    return planted_corpus_np(**TINY)


@pytest.fixture(scope="module")
def small():
    return planted_corpus_np(**SMALL)


def brute(w, d, z, n_docs, V, K):
    D = np.zeros((n_docs, K), np.int64)
    W = np.zeros((V, K), np.int64)
    np.add.at(D, (d.astype(np.int64), z.astype(np.int64)), 1)
    np.add.at(W, (w.astype(np.int64), z.astype(np.int64)), 1)
    return D, W


def check_counts(ez, g, w, d, n_docs, V, K, z=None):
    z = g.topics() if z is None else z
    D, W = brute(w, d, z, n_docs, V, K)
    Wg = ez.EzLDA.csr_to_dense(*g.W_csr(), K)
    Dg = ez.EzLDA.csr_to_dense(*g.D_csr(), K)
    assert np.array_equal(Wg, W), "W differs from recount"
    assert np.array_equal(Dg, D), "D differs from recount"
    assert np.array_equal(g.n_k(), W.sum(0)), "n_k differs from recount"
    # packed rows are sorted by topic (CSR columns ascending within a row)
    rp, col, _ = g.D_csr()
    for r in range(0, n_docs, max(1, n_docs // 50)):
        c = col[rp[r]:rp[r + 1]]
        assert np.all(np.diff(c.astype(np.int64)) > 0)


def oracle_chain(oracle_mod, w, d, n_docs, V, K, iters, sampler=3, **kw):
    """The oracle's own chain (independent of the GPU): topics / n_k / LLPT after `iters`."""
    orc = oracle_mod.OracleLDA(w, d, n_docs, V, K, seed=SAMPLER_SEED, branches=sampler, **kw)
    orc.iterate(iters)
    return orc


def boundary_distance(oracle_mod, orc, w, d, z_prev, t, K, alpha, g, it):
    """Distance (relative to Z) from the token's x = u Z to the nearest breakpoint of
    the [M | S' | Q'] layout, computed by the oracle on the snapshot z_prev."""
    D, _, _ = orc.counts()
    Drow = D[d[t]]
    What = orc.what(int(w[t]))
    u = oracle_mod.uniform(SAMPLER_SEED, it, int(orc.token_index()[t]))
    det = oracle_mod.draw_three_branch(Drow, What, alpha, g, u)
    K1 = det["K_sel"][0]
    thr_gap = abs(u - det["thr"])
    Wp = What.copy()
    Wp[K1] = 0.0
    Sp = np.cumsum(np.where(Drow > 0, Drow * Wp, 0.0))
    Z = det["M"] + Sp[-1] + det["Qp"]
    x = u * Z
    bps = np.concatenate([[det["M"]], det["M"] + Sp, det["M"] + Sp[-1] + alpha * np.cumsum(Wp)])
    return min(np.min(np.abs(bps - x)) / Z, thr_gap)


def run_one_step_parity(ez, oracle_mod, w, d, n_docs, V, K, iters, g=2, check_every=1, **kw):
    gpu = ez.EzLDA(w, d, n_docs, V, K, seed=SAMPLER_SEED, g=g, **kw)
    orc = oracle_mod.OracleLDA(w, d, n_docs, V, K, seed=SAMPLER_SEED, g=g)
    z = gpu.topics()
    assert np.array_equal(z, orc.topics()), "iteration-0 topics differ (Philox init)"
    check_counts(ez, gpu, w, d, n_docs, V, K, z)
    worst = 1.0
    total_mismatch = 0
    for i in range(1, iters + 1):
        orc.set_topics(z, i - 1)
        orc.iterate(1)
        gpu.iterate(1)
        zg, zo = gpu.topics(), orc.topics()
        mism = np.nonzero(zg != zo)[0]
        agree = 1.0 - len(mism) / len(zg)
        worst = min(worst, agree)
        total_mismatch += len(mism)
        assert agree >= 0.9999, (i, len(mism))
        if len(mism):
            ref = oracle_mod.OracleLDA(w, d, n_docs, V, K, seed=SAMPLER_SEED, g=g)
            ref.set_topics(z, i - 1)
            for t in mism[:20]:
                dist = boundary_distance(oracle_mod, ref, w, d, z, int(t), K, gpu.alpha, g, i)
                print(f"iteration {i} token {t}: gpu {zg[t]} oracle {zo[t]} boundary distance {dist:.3e} Z")
                assert dist <= 1e-12, (i, t, dist)
        st = gpu.stats()
        so = orc.last_stats()
        assert st["iteration"] == i
        if not len(mism):
            assert st["skip_S"] == so["skip_S"], (i, st["skip_S"], so["skip_S"])
            assert st["skip_final"] == so["skip_final"], (i, st["skip_final"], so["skip_final"])
            assert st["sampled"] == len(zg) - so["skip_S"]
        if i % check_every == 0 or i == iters:
            check_counts(ez, gpu, w, d, n_docs, V, K, zg)
        z = zg
    print(f"worst per-iteration agreement {worst:.6f}, total mismatches {total_mismatch}, "
          f"exact redraws (last iteration) {gpu.stats()['exact_redraws']}")
    assert total_mismatch == 0, "certified fast path + exact redraw must reproduce the oracle's topics bit for bit"
    return gpu, orc


def test_one_step_parity_tiny_50_iterations(ez, oracle_mod, tiny):
    w, d = tiny
    run_one_step_parity(ez, oracle_mod, w, d, TINY["n_docs"], TINY["V"], 16, 50, check_every=5)


def test_one_step_parity_small(ez, oracle_mod, small):
    w, d = small
    run_one_step_parity(ez, oracle_mod, w, d, SMALL["n_docs"], SMALL["V"], 64, 8, check_every=4)


@pytest.mark.parametrize("g", [1, 3])
def test_one_step_parity_g(ez, oracle_mod, tiny, g):
    w, d = tiny
    run_one_step_parity(ez, oracle_mod, w, d, TINY["n_docs"], TINY["V"], 16, 6, g=g, check_every=3)


def test_long_docs_block_tier_and_large_rows(ez, oracle_mod):
    """Docs longer than 512 tokens (block tier of the doc pass), D rows with > 128 nonzeros
    (register-spill path of the S' descent), K not a multiple of 32."""
    w, d = planted_corpus_np(n_docs=60, V=3000, mean_len=1200.0, sigma=0.6, K_true=100, seed=5)
    run_one_step_parity(ez, oracle_mod, w, d, 60, 3000, 1000, 4, check_every=2)


@pytest.mark.parametrize("K", [5000, 16384, 16385, 32768, 40000])
def test_large_K_paths(ez, oracle_mod, K):
    """K > 4096: bitonic doc-pass tier, 32 .. 256-entry S' segments, chunked warp-per-word
    word-prep, HBM slot histograms and Q' tables; K > 16384: 16-bit topic field in the packed D
    entries and the HBM-row LLPT kernel; K > 32768: no C1 marker (NEXT-2, P:168 / P:1282)."""
    w, d = planted_corpus_np(n_docs=100, V=2000, mean_len=300.0, sigma=0.8, K_true=50, seed=21)
    run_one_step_parity(ez, oracle_mod, w, d, 100, 2000, K, 3, check_every=3)


@pytest.mark.parametrize("K", [8000, 16384, 32768])
def test_wide_segment_fallback(ez, oracle_mod, K):
    """K > 4096 with documents holding more than 4096 distinct topics (256 segments of 16): those
    runs take the wide-segment fallback of the sampler (32 .. 256-entry segments)."""
    w, d = planted_corpus_np(n_docs=30, V=2000, mean_len=3000.0, sigma=0.8, K_true=50, seed=33)
    assert np.bincount(d).max() > 8000
    run_one_step_parity(ez, oracle_mod, w, d, 30, 2000, K, 2, check_every=2)


def test_exact_draws_knob_identical(ez, oracle_mod, small):
    """exact_draws=1 sends every sampled token through the fp64 path: topics identical to
    the default certified fixed-point path and to the oracle; the default path redraws few tokens."""
    w, d = small
    K = 64
    a = ez.EzLDA(w, d, SMALL["n_docs"], SMALL["V"], K, seed=SAMPLER_SEED)
    b = ez.EzLDA(w, d, SMALL["n_docs"], SMALL["V"], K, seed=SAMPLER_SEED, exact_draws=True)
    orc = oracle_mod.OracleLDA(w, d, SMALL["n_docs"], SMALL["V"], K, seed=SAMPLER_SEED)
    for i in range(1, 5):
        orc.set_topics(a.topics(), i - 1)
        b.set_topics(a.topics(), i - 1)
        a.iterate(1)
        b.iterate(1)
        orc.iterate(1)
        assert np.array_equal(a.topics(), b.topics()), i
        assert np.array_equal(a.topics(), orc.topics()), i
        sa, sb = a.stats(), b.stats()
        assert sb["exact_redraws"] == sb["sampled"]
        assert sa["exact_redraws"] <= 0.01 * sa["sampled"], sa


def test_chain_parity_llpt_100_iterations(ez, oracle_mod, tiny):
    """Independent 100-iteration chains: LLPT within 1e-3 relative (expected identical)."""
    w, d = tiny
    gpu = ez.EzLDA(w, d, TINY["n_docs"], TINY["V"], 16, seed=SAMPLER_SEED)
    orc = oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], 16, seed=SAMPLER_SEED)
    gpu.iterate(100)
    orc.iterate(100)
    lg, lo = gpu.loglik(), orc.loglik(1)
    print("LLPT gpu", lg, "oracle", lo, "topic agreement", np.mean(gpu.topics() == orc.topics()))
    assert abs(lg - lo) <= 1e-3 * abs(lo)


def test_llpt_parity_and_set_topics(ez, oracle_mod, small):
    w, d = small
    K = 64
    gpu = ez.EzLDA(w, d, SMALL["n_docs"], SMALL["V"], K, seed=SAMPLER_SEED)
    orc = oracle_mod.OracleLDA(w, d, SMALL["n_docs"], SMALL["V"], K, seed=SAMPLER_SEED)
    for it in (0, 3):
        if it:
            gpu.iterate(it)
        z = gpu.topics()
        orc.set_topics(z, gpu.stats()["iteration"] if it else 0)
        lg, lo = gpu.loglik(), orc.loglik(1)
        assert abs(lg - lo) <= 1e-10 * abs(lo), (lg, lo)
    # set_topics: arbitrary state, GPU rebuilds W / n_k; loglik matches
    rng = np.random.default_rng(3)
    z = rng.integers(0, K, size=len(w)).astype(np.uint16)
    gpu.set_topics(z, 7)
    assert np.array_equal(gpu.topics(), z)
    check_counts(ez, gpu, w, d, SMALL["n_docs"], SMALL["V"], K, z)
    orc.set_topics(z, 7)
    assert abs(gpu.loglik() - orc.loglik(1)) <= 1e-10 * abs(orc.loglik(1))
    gpu.iterate(1)
    orc.iterate(1)
    assert np.mean(gpu.topics() == orc.topics()) >= 0.9999


def test_appendix_a_state_loglik(ez):
    app = [(0, 0, 2), (0, 2, 1), (1, 1, 1), (1, 2, 0), (2, 0, 1), (2, 2, 3), (3, 1, 0)]
    w = np.array([t[0] for t in app], np.uint32)
    d = np.array([t[1] for t in app], np.uint32)
    g = ez.EzLDA(w, d, 3, 4, 4, alpha=16.7, beta=0.01)
    g.set_topics(np.array([t[2] for t in app], np.uint16), 0)
    assert abs(g.loglik() - (-1.963006)) < 1e-6


@pytest.mark.parametrize("knobs", [
    dict(w_mode=1), dict(w_mode=2), dict(dense_threshold=3), dict(split_threshold=64),
    dict(split_threshold=64, w_mode=1), dict(g=1), dict(g=3), dict(doc_block_kb=1),
    dict(doc_block_kb=1, split_threshold=100), dict(schedule=1), dict(schedule=2),
])
def test_knob_invariance(ez, oracle_mod, tiny, knobs):
    """Dense threshold, W mode, region split, doc windows and g change speed only: T
    bit-identical to the default GPU chain AND to the oracle's chain, every iteration."""
    w, d = tiny
    ref = ez.EzLDA(w, d, TINY["n_docs"], TINY["V"], 16, seed=SAMPLER_SEED)
    alt = ez.EzLDA(w, d, TINY["n_docs"], TINY["V"], 16, seed=SAMPLER_SEED, **knobs)
    orc = oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], 16, seed=SAMPLER_SEED, g=knobs.get("g", 2))
    for _ in range(6):
        ref.iterate(1)
        alt.iterate(1)
        orc.iterate(1)
        assert np.array_equal(alt.topics(), orc.topics()), knobs
        assert np.array_equal(ref.topics(), alt.topics()), knobs
    assert np.array_equal(ref.n_k(), alt.n_k())
    assert np.array_equal(alt.n_k(), orc.counts()[2])


def test_determinism(ez, small):
    w, d = small
    a = ez.EzLDA(w, d, SMALL["n_docs"], SMALL["V"], 64, seed=11)
    b = ez.EzLDA(w, d, SMALL["n_docs"], SMALL["V"], 64, seed=11)
    a.iterate(5)
    b.iterate(5)
    assert np.array_equal(a.topics(), b.topics())
    assert a.loglik() == b.loglik()


def test_input_order_and_empty_docs(ez, oracle_mod):
    """Tokens not grouped by doc, empty docs, absent words: same topics as the oracle."""
    rng = np.random.default_rng(8)
    w, d = planted_corpus_np(n_docs=80, V=400, mean_len=60.0, sigma=0.7, seed=9)
    d = d * 2  # odd doc ids are empty
    perm = rng.permutation(len(w))
    w, d = w[perm], d[perm]
    V = 450  # words 400..449 never occur
    gpu = ez.EzLDA(w, d, 161, V, 12, seed=4)
    orc = oracle_mod.OracleLDA(w, d, 161, V, 12, seed=4)
    for _ in range(5):
        gpu.iterate(1)
        orc.iterate(1)
        assert np.mean(gpu.topics() == orc.topics()) >= 0.9999
    check_counts(ez, gpu, w, d, 161, V, 12)


@pytest.mark.parametrize("K", [1, 2, 3])
def test_degenerate_K(ez, oracle_mod, tiny, K):
    w, d = tiny
    run_one_step_parity(ez, oracle_mod, w, d, TINY["n_docs"], TINY["V"], K, 3)


def test_single_token(ez):
    g = ez.EzLDA(np.array([0], np.uint32), np.array([0], np.uint32), 1, 1, 1, alpha=50.0)
    g.iterate(2)
    assert g.topics()[0] == 0
    assert g.loglik() == 0.0


def test_invalid_arguments(ez):
    w = np.array([0, 1], np.uint32)
    d = np.array([0, 0], np.uint32)
    with pytest.raises(ez.EzLDAError, match="E_INVALID"):
        ez.EzLDA(w, d, 1, 1, 4)  # word id 1 >= V
    with pytest.raises(ez.EzLDAError, match="E_INVALID"):
        ez.EzLDA(w, d, 1, 2, 4, alpha=0.0)
    with pytest.raises(ez.EzLDAError, match="E_RANGE"):
        ez.EzLDA(w, d, 1, 2, 70000)
    with pytest.raises(ez.EzLDAError, match="E_RANGE"):
        ez.EzLDA(w, d, 1, 2, 65535)  # valid for the packing, too wide for the sampler's slot
    long_doc = np.zeros(70000, np.uint32)
    with pytest.raises(ez.EzLDAError, match="E_RANGE"):
        ez.EzLDA(long_doc, long_doc, 1, 1, 4)


@pytest.mark.parametrize("sampler", [3, 2])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("delta", [True, False])
def test_multi_rank_library_path_one_gpu(ez, oracle_mod, world, sampler, delta, dperm=False):
    """The library's multi-rank path (doc shards with token bases, global word counts and
    relabelling, the hybrid W merged every iteration -- the dense block as packed 16-bit deltas
    against the previous W (default) or as int32 counts (EZLDA_DEBUG_NO_W_DELTA), the tail as
    all-gathered topics -- LLPT reduction) with the ranks as handles of this process on one
    GPU (options.local_group: the merge is an in-process device sum instead of NCCL).
    Concatenated topics, W, n_k and LLPT must equal the single-rank chain bit for bit
    (P-invariance of the counter-based draws), and the exchanged bytes the path's size."""
    import threading

    w, d = planted_corpus_np(n_docs=600, V=4000, mean_len=90.0, sigma=0.5, seed=17)
    n_docs, V, K, iters = 600, 4000, 64, 5
    ref = ez.EzLDA(w, d, n_docs, V, K, seed=SAMPLER_SEED, sampler=sampler)
    ref.iterate(iters)
    z_ref, nk_ref, ll_ref = ref.topics(), ref.n_k(), ref.loglik()
    W_ref = ez.EzLDA.csr_to_dense(*ref.W_csr(), K)
    L = np.bincount(d, minlength=n_docs)
    b = ez.partition_docs(L, world)
    cum = np.concatenate([[0], np.cumsum(L)])
    out, errs = {}, []

    def rank_main(r):
        try:
            t0, t1 = int(cum[b[r]]), int(cum[b[r + 1]])
            h = ez.EzLDA(w[t0:t1], d[t0:t1] - b[r], b[r + 1] - b[r], V, K, seed=SAMPLER_SEED, rank=r, world=world,
                         token_base=t0, local_group=1000 + 200 * int(dperm) + 100 * int(delta) + 10 * sampler + world,
                         sampler=sampler, debug_flags=(0 if delta else ez.EZLDA_DEBUG_NO_W_DELTA)
                         | (ez.EZLDA_DEBUG_DPERM_ON if dperm else 0))
            h.iterate(iters)
            xb = h.stats()["exchange_bytes"]
            out[r] = (h.topics(), ez.EzLDA.csr_to_dense(*h.W_csr(), K), h.n_k(), h.loglik(), xb)
        except Exception as e:  # surfaced below (the other ranks would wait forever otherwise)
            errs.append(repr(e))

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    z = np.concatenate([out[r][0] for r in range(world)])
    assert np.array_equal(z, z_ref)
    # ... and equal the oracle's chain (independent of the GPU)
    orc = oracle_chain(oracle_mod, w, d, n_docs, V, K, iters, sampler)
    assert np.array_equal(z, orc.topics())
    _, W_orc, nk_orc = orc.counts()
    assert np.array_equal(nk_ref, nk_orc) and np.array_equal(W_ref, W_orc)
    assert abs(ll_ref - orc.loglik(1)) <= 1e-10 * abs(ll_ref)
    for r in range(world):
        assert np.array_equal(out[r][1], W_ref), r
        assert np.array_equal(out[r][2], nk_ref), r
        assert abs(out[r][3] - ll_ref) <= 1e-12 * abs(ll_ref), (out[r][3], ll_ref)
    # bytes of the last exchange: dense block (Vd x K: packed u32 pairs, or int32) + the tail
    # all-gather (world slots of the largest local tail-token count, u16)
    cnt = np.bincount(w, minlength=V)
    dense_words = cnt > K
    Vd = int(dense_words.sum())
    tail_max = max(int((~dense_words[w[int(cum[b[r]]):int(cum[b[r + 1]])]]).sum()) for r in range(world))
    dense_bytes = 4 * ((Vd * K + 1) // 2) if delta else 4 * Vd * K
    for r in range(world):
        assert out[r][4] == dense_bytes + world * 2 * tail_max, (r, out[r][4], dense_bytes, tail_max)


@pytest.mark.parametrize("sampler", [3, 2])
def test_multi_rank_interleaved_rows(ez, oracle_mod, sampler):
    """The multi-rank path with every rank's D rows sector-interleaved (forced on short docs)."""
    test_multi_rank_library_path_one_gpu(ez, oracle_mod, 2, sampler, True, dperm=True)


TWO_BRANCH_CASES = {
    "tiny_K16": (dict(n_docs=100, V=500, mean_len=100.0, sigma=0.5), 16, 12),
    "small_K64": (dict(n_docs=2000, V=5000, mean_len=90.0, sigma=0.5), 64, 4),
    "long_docs_K1000": (dict(n_docs=60, V=3000, mean_len=1200.0, sigma=0.6, K_true=100, seed=5), 1000, 2),
    "K5000": (dict(n_docs=100, V=2000, mean_len=300.0, sigma=0.8, K_true=50, seed=21), 5000, 2),
    # K too large for the word's tables in shared memory: HBM tables + doc-major draw + W count
    "K16384_hbm_tables": (dict(n_docs=100, V=2000, mean_len=300.0, sigma=0.8, K_true=50, seed=21), 16384, 2),
    "K32768_hbm_tables": (dict(n_docs=100, V=2000, mean_len=300.0, sigma=0.8, K_true=50, seed=21), 32768, 2),
}


@pytest.mark.parametrize("case", list(TWO_BRANCH_CASES))
def test_two_branch_mode_parity(ez, oracle_mod, case):
    """sampler=2 (two-branch ESCA mode, NEXT-1, reading #11): one-step parity with
    the oracle's two-branch chain, bit-identical topics, exact D / W / n_k, no skipping."""
    spec, K, iters = TWO_BRANCH_CASES[case]
    w, d = planted_corpus_np(**spec)
    n_docs, V = spec["n_docs"], spec["V"]
    gpu = ez.EzLDA(w, d, n_docs, V, K, seed=SAMPLER_SEED, sampler=2)
    orc = oracle_mod.OracleLDA(w, d, n_docs, V, K, seed=SAMPLER_SEED, branches=2)
    chain = oracle_mod.OracleLDA(w, d, n_docs, V, K, seed=SAMPLER_SEED, branches=2)
    z = gpu.topics()
    assert np.array_equal(z, orc.topics())
    for i in range(1, iters + 1):
        orc.set_topics(z, i - 1)
        orc.iterate(1)
        chain.iterate(1)
        gpu.iterate(1)
        zg = gpu.topics()
        assert np.array_equal(zg, orc.topics()), (i, int((zg != orc.topics()).sum()))
        st = gpu.stats()
        assert st["skip_S"] == 0 and st["sampled"] == len(zg)
        check_counts(ez, gpu, w, d, n_docs, V, K, zg)
        z = zg
    # chain parity: the independent oracle chain reached the same state
    assert np.array_equal(gpu.topics(), chain.topics())
    assert abs(gpu.loglik() - chain.loglik(1)) <= 1e-10 * abs(chain.loglik(1))


@pytest.mark.parametrize("sampler", [3, 2])
def test_checkpoint_resume_is_exact(ez, oracle_mod, small, sampler):
    """Checkpoint = (topics, iterations done) from ezlda_counts; resume = a fresh handle +
    ezlda_set_topics: the resumed chain equals the uninterrupted one bit for bit (the draws
    are keyed by (token, iteration))."""
    w, d = small
    K = 64
    a = ez.EzLDA(w, d, SMALL["n_docs"], SMALL["V"], K, seed=SAMPLER_SEED, sampler=sampler)
    a.iterate(4)
    ckpt = a.topics().copy()
    a.iterate(4)
    b = ez.EzLDA(w, d, SMALL["n_docs"], SMALL["V"], K, seed=SAMPLER_SEED, sampler=sampler)
    b.set_topics(ckpt, 4)
    b.iterate(4)
    assert b.stats()["iteration"] == 8
    assert np.array_equal(a.topics(), b.topics())
    assert np.array_equal(a.n_k(), b.n_k())
    assert a.loglik() == b.loglik()
    orc = oracle_chain(oracle_mod, w, d, SMALL["n_docs"], SMALL["V"], K, 8, sampler)
    assert np.array_equal(b.topics(), orc.topics())
    assert abs(b.loglik() - orc.loglik(1)) <= 1e-10 * abs(orc.loglik(1))


@pytest.mark.parametrize("sampler", [3, 2])
def test_one_rank_nccl_group_matches_single_gpu(ez, oracle_mod, sampler):
    """world = 1 with an ncclUniqueId: the library's multi-rank path -- global word counts
    all-reduced at create, every W row dense, W and n_k merged by ncclAllReduce every
    iteration, LLPT reduced -- through a real one-rank NCCL communicator (the only NCCL
    group one GPU can hold).  Topics, W, n_k and LLPT equal the single-GPU chain bit for bit."""
    w, d = planted_corpus_np(n_docs=600, V=4000, mean_len=90.0, sigma=0.5, seed=17)
    n_docs, V, K, iters = 600, 4000, 64, 5
    ref = ez.EzLDA(w, d, n_docs, V, K, seed=SAMPLER_SEED, sampler=sampler)
    ref.iterate(iters)
    h = ez.EzLDA(w, d, n_docs, V, K, seed=SAMPLER_SEED, sampler=sampler, rank=0, world=1,
                 nccl_id=ez.nccl_unique_id())
    h.iterate(iters)
    assert np.array_equal(h.topics(), ref.topics())
    assert np.array_equal(ez.EzLDA.csr_to_dense(*h.W_csr(), K), ez.EzLDA.csr_to_dense(*ref.W_csr(), K))
    assert np.array_equal(h.n_k(), ref.n_k())
    assert h.loglik() == ref.loglik()
    orc = oracle_chain(oracle_mod, w, d, n_docs, V, K, iters, sampler)
    assert np.array_equal(h.topics(), orc.topics())
    assert np.array_equal(h.n_k(), orc.counts()[2])


DEBUG_CASES = {
    # every tail-word item staged by a sampler warp (stage_tail_row_warp + per-slot QP scratch)
    "no_tail_rows_K1000": (dict(n_docs=60, V=3000, mean_len=1200.0, sigma=0.6, K_true=100, seed=5), 1000, 3, 1),
    "no_tail_rows_K64": (SMALL, 64, 3, 1),
    "no_tail_rows_K16384": (dict(n_docs=100, V=2000, mean_len=300.0, sigma=0.8, K_true=50, seed=21), 16384, 2, 1),
    # C1 never carried in the z^i marker: every sampled token looks C1 up in its packed D row
    "c1_lookup_K64": (SMALL, 64, 3, 2),
    "c1_lookup_K1000": (dict(n_docs=60, V=3000, mean_len=1200.0, sigma=0.6, K_true=100, seed=5), 1000, 2, 2),
    "both_K5000": (dict(n_docs=100, V=2000, mean_len=300.0, sigma=0.8, K_true=50, seed=21), 5000, 2, 3),
    # sector-interleaved D rows (kernels.h d_phys) forced on short docs / off on long docs, and
    # with the C1 lookup (binary search through the mapped row)
    "dperm_on_K64": (SMALL, 64, 3, 4),
    "dperm_on_K1000": (dict(n_docs=60, V=3000, mean_len=1200.0, sigma=0.6, K_true=100, seed=5), 1000, 3, 4),
    "dperm_on_c1_K1000": (dict(n_docs=60, V=3000, mean_len=1200.0, sigma=0.6, K_true=100, seed=5), 1000, 2, 6),
    "dperm_on_K4096": (dict(n_docs=100, V=2000, mean_len=300.0, sigma=0.8, K_true=50, seed=21), 4096, 2, 4),
    "dperm_off_K1000": (dict(n_docs=60, V=3000, mean_len=1200.0, sigma=0.6, K_true=100, seed=5), 1000, 2, 8),
}


@pytest.mark.parametrize("case", list(DEBUG_CASES))
def test_rare_paths_parity(ez, oracle_mod, case):
    """Paths the default configs rarely or never take, forced by ezlda_options.debug_flags:
    one-step parity with the oracle, bit-identical topics and exact counts."""
    spec, K, iters, flags = DEBUG_CASES[case]
    w, d = planted_corpus_np(**spec)
    gpu, orc = run_one_step_parity(ez, oracle_mod, w, d, spec["n_docs"], spec["V"], K, iters, check_every=iters,
                                   debug_flags=flags)
    # LLPT reads every packed D row (through the interleaved layout when dperm is on)
    lg, lo = gpu.loglik(), orc.loglik(1)
    assert abs(lg - lo) <= 1e-10 * abs(lo), (lg, lo)


def test_live_handles_with_different_K(ez, oracle_mod, tiny):
    """Two live handles with different K (different sampler layouts / grids / shared-memory
    sizes) iterated alternately: each equals its oracle chain (per-handle grid,
    shared-memory limits only raised)."""
    w, d = tiny
    big = ez.EzLDA(w, d, TINY["n_docs"], TINY["V"], 16384, seed=SAMPLER_SEED)
    small_ = ez.EzLDA(w, d, TINY["n_docs"], TINY["V"], 64, seed=SAMPLER_SEED)
    ob = oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], 16384, seed=SAMPLER_SEED)
    os_ = oracle_mod.OracleLDA(w, d, TINY["n_docs"], TINY["V"], 64, seed=SAMPLER_SEED)
    for _ in range(3):
        small_.iterate(1)
        big.iterate(1)
        ob.iterate(1)
        os_.iterate(1)
        assert np.array_equal(big.topics(), ob.topics())
        assert np.array_equal(small_.topics(), os_.topics())


def test_set_topics_validates_device_input(ez, tiny):
    """A topic >= K passed in DEVICE memory is rejected (E_INVALID) before any state change."""
    import torch

    w, d = tiny
    g = ez.EzLDA(w, d, TINY["n_docs"], TINY["V"], 16, seed=SAMPLER_SEED)
    g.iterate(1)
    z0 = g.topics()
    bad = torch.from_numpy(z0.astype(np.int16)).cuda()
    bad[17] = 16
    with pytest.raises(ez.EzLDAError, match="E_INVALID"):
        g.set_topics(bad, 5)
    assert np.array_equal(g.topics(), z0)
    ok = torch.from_numpy(z0.astype(np.int16)).cuda()
    g.set_topics(ok, 1)
    assert np.array_equal(g.topics(), z0)


def test_local_group_world_mismatch_rejected(ez, tiny):
    """A local_group key in use with another world is rejected at once; the group then
    completes with the right world, and the key is reusable once its handles are destroyed
    (ADVICE r01)."""
    import threading

    w, d = tiny
    n = len(w) // 2
    out = {}

    def rank0():
        out[0] = ez.EzLDA(w[:n], d[:n], TINY["n_docs"], TINY["V"], 16, rank=0, world=2, local_group=777)

    t = threading.Thread(target=rank0)
    t.start()
    import time

    time.sleep(2.0)  # rank 0 registered the key (it now waits for rank 1 in create)
    with pytest.raises(ez.EzLDAError, match="E_INVALID"):
        ez.EzLDA(w[n:], d[n:], TINY["n_docs"], TINY["V"], 16, rank=1, world=3, local_group=777)
    b = ez.EzLDA(w[n:], d[n:], TINY["n_docs"], TINY["V"], 16, rank=1, world=2, local_group=777, token_base=n)
    t.join(timeout=120)
    assert 0 in out
    out[0].close()
    b.close()
    # the key is free again: a 3-rank group reuses it
    hs, errs = {}, []

    def rank_main(r, world=3):
        try:
            t0, t1 = r * len(w) // world, (r + 1) * len(w) // world
            hs[r] = ez.EzLDA(w[t0:t1], d[t0:t1], TINY["n_docs"], TINY["V"], 16, rank=r, world=world,
                             local_group=777, token_base=t0)
        except Exception as e:
            errs.append(repr(e))

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(3)]
    for x in ts:
        x.start()
    for x in ts:
        x.join(timeout=120)
    assert not errs and len(hs) == 3, errs
