/*
 * ezlda_oracle.h -- CPU ORACLE for the ezLDA three-branch Gibbs hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * library.  The product path (paper_2007_08725_b200/, include/ezlda.h) never
 * links, imports or executes anything under oracle/, and this oracle shares no
 * code, header, table or helper with the CUDA path.
 *
 * What it computes: plain, slow, fp64 (-ffp-contract=off) collapsed-Gibbs
 * sweeps with the paper's three-branch sampler, following SURVEY.md 8(c)
 * step by step.  Citations are PAPER.md line numbers ("P:n") of
 * arXiv 2007.08725 ("ezLDA: Efficient and Scalable LDA on GPUs").
 *
 * Pins (tests/test_oracle_*.py): Fig 2 worked example, Fig 4
 * M / appendix bound, Fig 5 inverted index,
 * Random123 Philox4x32-10 known-answer vectors, brute-force u-measure of each
 * topic vs the textbook conditional Eq (1)/(2), S_est >= S',
 * topic invariance across g, count invariants, K=1 unigram LLPT
 * closed form (Eq 5), dense-vs-identity LLPT cross-check; the two-branch
 * (ESCA) draw and chain (ezlda_oracle_set_sampler): u-measure of every topic equals the
 * textbook conditional, count invariants, LLPT rise, doc-shard emulation.
 * Parity pinned for every exported function except as stated in DESIGN.md.
 */
#ifndef EZLDA_ORACLE_H
#define EZLDA_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct ezlda_oracle ezlda_oracle;

/* Per-token record of one three-branch draw. */
typedef struct {
  uint32_t K_sel[4];   /* K1..K4: topics of the largest What entries, ties -> smaller k (P:546 step 1) */
  double a[4];         /* a1..a4 = What at K1..K4 (Eq 7) */
  uint32_t C[4];       /* C_j = D[d][K_j] (P:546 step 2) */
  uint32_t L;          /* document length L_d */
  double M;            /* Eq 8: a1 (C1 + alpha) */
  double S_est;        /* Eq 10 (g >= 1) or appendix bound (g == 0) */
  double Qp;           /* Q' = alpha * sum_{k != K1} What_k              (Eq 6) */
  double thr;          /* M / (M + S_est + Q')                           (P:546 step 3) */
  double Sp;           /* S' = sum_{k in nz(D), k != K1} D_k What_k  (only when not skipped) */
  double Z;            /* M + S' + Q' */
  double x;            /* u * Z */
  int branch;          /* 0 = skip (MPT test), 1 = M second chance, 2 = S', 3 = Q' */
  uint32_t topic;      /* the new topic */
} ezlda_oracle_draw_detail;

/* ---- primitives (used by golden tests) ---- */

/* Philox4x32-10 (Salmon et al., SC'11 / Random123), reading #14 of SURVEY 8(c). */
void ezlda_oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* u = ((r0 >> 5) 2^26 + (r1 >> 6)) 2^-53 with ctr = (t_g lo, t_g hi, iter, 0), key = seed. */
double ezlda_oracle_uniform(uint64_t seed, uint32_t iteration, uint64_t t_g);
/* Iteration-0 topic: floor(r0 K / 2^32) with iter = 0. */
uint32_t ezlda_oracle_init_topic(uint64_t seed, uint64_t t_g, uint32_t K);

/* Three-branch draw of ONE token given the dense rows D[d] (K ints) and What[v] (K doubles).
 * g in {1,2,3} selects Eq (10); g == 0 selects the appendix bound (L - C1) a1.
 * Returns 0 on success, nonzero on invalid arguments. */
int ezlda_oracle_draw_three_branch(const int32_t* Drow, const double* What, uint32_t K, double alpha,
                                   uint32_t g, double u, ezlda_oracle_draw_detail* out);
/* Batched variant: topics[i] = three-branch topic for u[i] (same row pair), branch[i] optional. */
int ezlda_oracle_draw_grid(const int32_t* Drow, const double* What, uint32_t K, double alpha, uint32_t g,
                           const double* u, uint64_t n, uint32_t* topics, int32_t* branch);
/* Two-branch (ESCA) draw per the Fig 2 text: S if u <= S/(S+Q) with
 * u' = u (S+Q), else Q with u' = (1-u)(S+Q); descend prefix sums of D o What resp. alpha o What.
 * Writes S, Q, u' and the prefix arrays (K doubles each, may be NULL). Returns the topic. */
uint32_t ezlda_oracle_draw_two_branch(const int32_t* Drow, const double* What, uint32_t K, double alpha,
                                      double u, double* S, double* Q, double* uprime,
                                      double* S_prefix, double* Q_prefix);
/* Inverted index of a token list (Fig 5): positions of each doc's tokens in the
 * list sorted by (word, doc, input position).  doc_ofs[n_docs+1], pos[n] (caller-allocated). */
void ezlda_oracle_inverted_index(const uint32_t* word_ids, const uint32_t* doc_ids, uint64_t n,
                                 uint32_t n_docs, uint64_t* doc_ofs, uint64_t* pos);

/* ---- whole-corpus chain ---- */
int ezlda_oracle_create(const uint32_t* word_ids, const uint32_t* doc_ids, uint64_t n_tokens,
                        uint32_t n_docs, uint32_t V, uint32_t K, double alpha, double beta,
                        uint64_t seed, uint32_t g, uint64_t token_base, ezlda_oracle** out);
void ezlda_oracle_destroy(ezlda_oracle* h);
/* Global doc-major RNG index t_g of every input token (input order). */
void ezlda_oracle_token_index(const ezlda_oracle* h, uint64_t* t_g);
/* Replace the state: topics in input order, and the number of completed iterations. */
int ezlda_oracle_set_topics(ezlda_oracle* h, const uint16_t* topics, uint32_t iterations_done);
int ezlda_oracle_topics(const ezlda_oracle* h, uint16_t* topics);
uint32_t ezlda_oracle_iterations(const ezlda_oracle* h);
/* What[v][k] = (W[v][k] + beta) / (n_k + V beta) of the current state (Eq 1-2), row[K].
 * W_global/nk_global override the snapshot as in iterate (may be NULL). */
int ezlda_oracle_what(const ezlda_oracle* h, uint32_t v, const int32_t* W_global, const int32_t* nk_global,
                      double* row);
/* What row of one word from its count row: row[k] = (W_row[k] + beta) / (n_k[k] + V beta)
 * (Eq 1-2; the same expression what_row applies inside the chain). */
void ezlda_oracle_what_row(const int32_t* W_row, const int32_t* n_k, uint32_t K, uint32_t V, double beta,
                           double* row);
/* Sampler of the chain: 3 = three-branch (default), 2 = two-branch ESCA
 * (ezlda_oracle_draw_two_branch per token, no skip test, Alg P:1481-1507).
 * last_stats then reports skip_S = skip_final = 0 and branch_hist[2] / [3] = S / Q draws. */
int ezlda_oracle_set_sampler(ezlda_oracle* h, uint32_t branches);
/* Run n snapshot iterations.  W_global/nk_global (V*K and K ints) override the W snapshot
 * of the FIRST of them when non-NULL (multi-shard emulation: W is the sum over shards). */
int ezlda_oracle_iterate(ezlda_oracle* h, uint32_t n, const int32_t* W_global, const int32_t* nk_global);
/* Dense counts of the current state (any pointer may be NULL): D [n_docs*K], W [V*K], n_k [K]. */
int ezlda_oracle_counts(const ezlda_oracle* h, int32_t* D, int32_t* W, int32_t* n_k);
/* LLPT, Eq (5), log2; method 0 = dense O(K) sum, 1 = S_full + Q_full identity.
 * W_global/nk_global as in iterate.  sum_out (may be NULL) receives the un-normalised sum. */
int ezlda_oracle_loglik(const ezlda_oracle* h, int method, const int32_t* W_global,
                        const int32_t* nk_global, double* llpt, double* sum_out);
/* Per-iteration counters of the last iterate() step: tokens skipped by the MPT test (skip_S),
 * tokens assigned K1 without descent (skip_final, includes skip_S), branch histogram[4]. */
void ezlda_oracle_last_stats(const ezlda_oracle* h, uint64_t* skip_S, uint64_t* skip_final,
                             uint64_t branch_hist[4]);

#ifdef __cplusplus
}
#endif
#endif
