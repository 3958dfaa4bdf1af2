"""Oracle pinned to the mathematics: the three-branch map samples the textbook
conditional p(k) ∝ (D[d][k]+alpha) What[v][k] (Eq 1-2) exactly, the
skip is exact because S_est >= S' (Eq 9-10), and the topic does not depend
on g or on the appendix bound.  Random states follow SURVEY A.2."""
import numpy as np
import pytest
from scipy import stats

from paper_2007_08725_b200.synth import random_state


def textbook_p(D, What, alpha):
    p = (D.astype(np.float64) + alpha) * What  # Eq (2): (D[d][k] + alpha) * What[v][k]
    return p / p.sum()


@pytest.mark.parametrize("seed", range(40))
def test_u_measure_equals_conditional(oracle_mod, seed):
    rng = np.random.default_rng(1000 + seed)
    K = int(rng.integers(3, 12))
    alpha = float(rng.uniform(0.05, 5.0))
    D, What = random_state(rng, K)
    G = 20000
    u = (np.arange(G) + 0.5) / G
    p = textbook_p(D, What, alpha)
    ref_topics = None
    for g in (0, 1, 2, 3):
        topics, branch = oracle_mod.draw_grid(D, What, alpha, g, u)
        freq = np.bincount(topics, minlength=K) / G
        # each topic is a union of at most 2 intervals (K1: [0, M/Z)), 2 grid cells of error each
        np.testing.assert_allclose(freq, p, atol=4.0 / G + 1e-12)
        # map is monotone piecewise constant in x: topic identical for every bound (exact skip)
        if ref_topics is None:
            ref_topics = topics
        else:
            assert np.array_equal(topics, ref_topics)
        assert set(np.unique(branch)) <= {0, 1, 2, 3}
        # zero-weight topics never drawn: every topic has p > 0 here since alpha > 0


@pytest.mark.parametrize("g", [0, 1, 2, 3])
def test_sest_upper_bounds_sprime(oracle_mod, g):
    rng = np.random.default_rng(7 + g)
    for _ in range(3000):
        K = int(rng.integers(2, 40))
        D, What = random_state(rng, K, density=float(rng.uniform(0.05, 1.0)), max_count=int(rng.integers(1, 30)))
        alpha = float(rng.uniform(0.01, 3.0))
        det = oracle_mod.draw_three_branch(D, What, alpha, g, 0.0)
        K1 = det["K_sel"][0]
        # S' = W.D - M + a1 alpha (Eq 9) = sum_{k != K1} D_k What_k, computed independently
        Sprime = float(np.dot(D.astype(np.float64), What) - D[K1] * What[K1])
        assert det["S_est"] >= Sprime * (1 - 1e-12) - 1e-300
        # top entries are the true descending order statistics (ties -> smaller k)
        order = sorted(range(K), key=lambda k: (-What[k], k))
        n = min(4, K)
        assert det["K_sel"][:n] == order[:n]


def test_chi_square_on_philox_draws(oracle_mod):
    rng = np.random.default_rng(99)
    K = 12
    D, What = random_state(rng, K, density=0.6)
    alpha = 0.8
    n = 200_000
    u = np.array([oracle_mod.uniform(1, 5, t) for t in range(n)])
    topics, _ = oracle_mod.draw_grid(D, What, alpha, 2, u)
    obs = np.bincount(topics, minlength=K)
    exp = textbook_p(D, What, alpha) * n
    chi2, pval = stats.chisquare(obs, exp)
    assert pval > 1e-4, (chi2, pval)


def test_uniform_and_init_distribution(oracle_mod):
    n = 100_000
    u = np.array([oracle_mod.uniform(123, 3, t) for t in range(n)])
    assert u.min() >= 0.0 and u.max() < 1.0
    assert stats.kstest(u, "uniform").pvalue > 1e-4
    # 53-bit dyadic values
    assert np.all(np.floor(u * 2.0**53) == u * 2.0**53)
    K = 37
    z = np.array([oracle_mod.init_topic(123, t, K) for t in range(n)])
    assert z.max() < K
    assert stats.chisquare(np.bincount(z, minlength=K)).pvalue > 1e-4
    # different iterations / seeds give different streams
    assert oracle_mod.uniform(123, 3, 0) != oracle_mod.uniform(123, 4, 0)
    assert oracle_mod.uniform(123, 3, 0) != oracle_mod.uniform(124, 3, 0)


def test_degenerate_K1_and_K2(oracle_mod):
    # K = 1: everything stays in topic 0 (S' = Q' = 0, thr = 1)
    det = oracle_mod.draw_three_branch([5], [0.7], 50.0, 2, 0.999999)
    assert det["topic"] == 0 and det["branch"] == 0 and det["thr"] == 1.0
    # K = 2: g forced to 1, S_est = a2 (L - C1)
    det = oracle_mod.draw_three_branch([3, 2], [0.2, 0.9], 1.0, 2, 0.0)
    assert det["K_sel"][:2] == [1, 0]
    assert det["S_est"] == pytest.approx(0.2 * (5 - 2))
    # doc with every token at K1: S_est = S' = 0
    det = oracle_mod.draw_three_branch([0, 4, 0], [0.1, 0.9, 0.3], 1.0, 2, 0.0)
    assert det["S_est"] == 0.0


@pytest.mark.parametrize("seed", range(20))
def test_two_branch_u_measure_equals_conditional(oracle_mod, seed):
    """The two-branch (ESCA) map of the Fig 2 text (reading #11) samples the
    same textbook conditional: S branch on [0, S/Z] with u' = uZ, Q branch with u' = (1-u)Z."""
    rng = np.random.default_rng(5000 + seed)
    K = int(rng.integers(2, 12))
    alpha = float(rng.uniform(0.05, 5.0))
    D, What = random_state(rng, K)
    G = 20000
    u = (np.arange(G) + 0.5) / G
    p = textbook_p(D, What, alpha)
    topics = np.array([oracle_mod.draw_two_branch(D, What, alpha, float(x))["topic"] for x in u])
    freq = np.bincount(topics, minlength=K) / G
    # each topic: one interval in the S branch, one (reversed) in the Q branch
    np.testing.assert_allclose(freq, p, atol=4.0 / G + 1e-12)
    # the S branch only ever returns topics present in the doc row
    r = oracle_mod.draw_two_branch(D, What, alpha, 0.0)
    assert D[r["topic"]] > 0 or D.sum() == 0
