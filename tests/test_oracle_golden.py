"""Oracle pinned to values the paper prints (tests/golden/*, each line cited there).

Fig 2, Fig 4 (Alg MPTC), Fig 5, and the
Random123 Philox4x32-10 known-answer vectors (the paper is silent on the RNG).
"""
import numpy as np
import pytest

from tests._golden import load, load_rows

# Corpus of Figs 1/2/5, reconstruction of SURVEY App. A.1: (word, doc, topic)
APP_A = [(0, 0, 2), (0, 2, 1), (1, 1, 1), (1, 2, 0), (2, 0, 1), (2, 2, 3), (3, 1, 0)]


def fig2_state(oracle_mod):
    g = load("fig2_worked_example.txt")
    w = np.array([t[0] for t in APP_A], dtype=np.uint32)
    d = np.array([t[1] for t in APP_A], dtype=np.uint32)
    z = np.array([t[2] for t in APP_A], dtype=np.uint16)
    h = oracle_mod.OracleLDA(w, d, n_docs=3, V=g["V"], K=g["K"], alpha=g["alpha"], beta=g["beta"], seed=1)
    h.set_topics(z, 0)
    return g, h


def test_philox_known_answers(oracle_mod):
    for row in load_rows("philox_kat.txt"):
        vals = [int(x, 16) for x in row]
        assert oracle_mod.philox4x32_10(vals[0:4], vals[4:6]) == vals[6:10]


def test_fig2_counts_match_printed_state(oracle_mod):
    g, h = fig2_state(oracle_mod)
    D, W, nk = h.counts()
    assert list(W[0]) == g["W0"]
    assert list(D[2]) == g["D2"]
    assert list(nk) == g["n_k"]


def test_fig2_what_and_prefix_sums(oracle_mod):
    g, h = fig2_state(oracle_mod)
    what0 = h.what(0)
    np.testing.assert_allclose(what0, g["what0"], atol=6e-5)           # 4 printed decimals
    np.testing.assert_allclose(g["alpha"] * what0, g["alpha_what0"], atol=1e-3)  # reading #2
    r = oracle_mod.draw_two_branch(g["D2"], what0, g["alpha"], g["u"])
    np.testing.assert_allclose(r["Q_prefix"], g["q_prefix"], atol=1e-3)
    np.testing.assert_allclose(r["S_prefix"], g["s_prefix_corrected"], atol=6e-5)
    # the printed S weights are What o D
    np.testing.assert_allclose(what0 * np.array(g["D2"]), g["s_weights"], atol=6e-5)


def test_fig2_two_branch_draw(oracle_mod):
    g, h = fig2_state(oracle_mod)
    r = oracle_mod.draw_two_branch(g["D2"], h.what(0), g["alpha"], g["u"])
    assert g["u"] > r["S"] / (r["S"] + r["Q"])  # 0.51 is not smaller than S/(S+Q) -> Q tree
    assert abs(r["uprime"] - g["uprime"]) < 1e-3
    assert r["topic"] == g["topic"]


def test_fig4_M_and_appendix_bound(oracle_mod):
    g, h = fig2_state(oracle_mod)
    f4 = load("fig4_three_branch.txt")
    det = oracle_mod.draw_three_branch(g["D2"], h.what(0), g["alpha"], 0, 0.51)  # g=0: appendix bound
    assert abs(det["M"] - f4["M"]) < f4["tolerance"]
    assert abs(det["S_est"] - f4["S_est_appendix"]) < f4["tolerance"]
    assert det["K_sel"][:3] == [2, 1, 3]


@pytest.mark.parametrize("u,branch,topic", [
    (0.51, 0, 2),     # below thr(g=2) = 0.725308: skipped in the MPT test
    (0.7254, 1, 2),   # thr < u < t_M = 0.725461 (= exact p(2)): second chance
    (0.73, 2, 1),     # t_M < u < t_S = 0.740971: S' tree, y = 0.1014 -> prefix {0.0049, 0.3371, ...} -> 1
    (0.9, 3, 1),      # Q' tree, y = 3.555 -> alpha P = {0.0819, 5.630, 5.630, 5.791} -> 1
    (0.999, 3, 3),    # Q' tree, y = 5.7685 -> 3
])
def test_fig2_token_three_branch_closed_form(oracle_mod, u, branch, topic):
    """Closed-form values of the three-branch map on the Fig 2 token:
    M = a1(C1+alpha), Q' = alpha(What_0+What_1+What_3), S' = sum_{k!=K1} D_k What_k,
    S_est(g=2) = a2 C2 + a3 (L - C1 - C2) with K = (2,1,3), C = (0,1,1), L = 3."""
    g, h = fig2_state(oracle_mod)
    what0 = h.what(0)
    det = oracle_mod.draw_three_branch(g["D2"], what0, g["alpha"], 2, u)
    exact_M = what0[2] * (0 + g["alpha"])
    exact_Q = g["alpha"] * (what0[0] + what0[1] + what0[3])
    exact_Sest = what0[1] * 1 + what0[3] * (3 - 0 - 1)
    assert abs(det["M"] - 16.218269) < 1e-5 and abs(det["M"] - exact_M) < 1e-12
    assert abs(det["Qp"] - 5.790795) < 1e-5 and abs(det["Qp"] - exact_Q) < 1e-12
    assert abs(det["S_est"] - 0.351468) < 1e-5 and abs(det["S_est"] - exact_Sest) < 1e-12
    assert abs(det["thr"] - 0.725308) < 1e-6
    if branch:
        assert abs(det["Sp"] - 0.346754) < 1e-6
        assert abs(det["Z"] - 22.355818) < 1e-5
    assert det["branch"] == branch
    assert det["topic"] == topic


def test_fig5_inverted_index(oracle_mod):
    f5 = load("fig5_inverted_index.txt")
    toks = [tuple(int(x) for x in s.split(",")) for s in f5["tokens"]]
    w = np.array([t[0] for t in toks], dtype=np.uint32)
    d = np.array([t[1] for t in toks], dtype=np.uint32)
    ofs, pos = oracle_mod.inverted_index(w, d, 3)
    got = [list(pos[ofs[i]:ofs[i + 1]]) for i in range(3)]
    assert got == [f5["doc0"], f5["doc1"], f5["doc2"]]


def test_fig2_what_row_primitive(oracle_mod):
    """ezlda_oracle_what_row (used to feed full-size parity checks) on the printed Fig 2 state:
    W[0] = {0,1,1,0}, n_k = {2,3,1,1}, V = 4, beta = 0.01 -> What[0] as printed, and
    identical to the chain's own What row."""
    g, h = fig2_state(oracle_mod)
    row = oracle_mod.what_row(g["W0"], g["n_k"], g["V"], g["beta"])
    np.testing.assert_allclose(row, g["what0"], atol=6e-5)
    assert np.array_equal(row, h.what(0))
