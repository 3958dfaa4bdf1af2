/*
 * ezlda_oracle.c -- plain, slow CPU oracle for the ezLDA three-branch hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see ezlda_oracle.h): loaded only by tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline legs.  Shares no code with
 * the CUDA path.  Built with -O2 -ffp-contract=off so every fp64 operation below
 * is rounded exactly as written (no fused multiply-add).
 *
 * Notation follows the paper (arXiv 2007.08725, PAPER.md = "P:n"):
 *   D[d][k]  doc-topic counts,  W[v][k]  word-topic counts,  n_k column sums,
 *   What[v][k] = (W[v][k] + beta) / (n_k + V beta)             Eq (1)-(2)
 *   p = D o What' + alpha o What' + (D + alpha) o What^m        Eq (6),
 *   M = a1 (b1 + alpha)                                         Eq (8),
 *   S_est = sum_{2<=i<=g} a_i b_i + a_{g+1} sum_{i>g} b_i       Eq (10),
 * and the normative readings of SURVEY.md 8(c) (listed again in DESIGN.md).
 */
#include "ezlda_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11; Random123 reference).     */
/* ------------------------------------------------------------------------- */
void ezlda_oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { /* key bump between rounds */
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void philox_token(uint64_t seed, uint32_t iteration, uint64_t t_g, uint32_t r[4]) {
  uint32_t ctr[4] = {(uint32_t)t_g, (uint32_t)(t_g >> 32), iteration, 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  ezlda_oracle_philox4x32_10(ctr, key, r);
}

/* u ~ U[0,1) with 53 random bits (reading #14/#16). */
double ezlda_oracle_uniform(uint64_t seed, uint32_t iteration, uint64_t t_g) {
  uint32_t r[4];
  philox_token(seed, iteration, t_g, r);
  uint64_t bits = ((uint64_t)(r[0] >> 5) << 26) | (uint64_t)(r[1] >> 6);
  return (double)bits * 0x1p-53;
}

/* z^0 = floor(r0 K / 2^32), iteration 0 ("Iteration 0"). */
uint32_t ezlda_oracle_init_topic(uint64_t seed, uint64_t t_g, uint32_t K) {
  uint32_t r[4];
  philox_token(seed, 0u, t_g, r);
  return (uint32_t)(((uint64_t)r[0] * (uint64_t)K) >> 32);
}

/* ------------------------------------------------------------------------- */
/* Per-word preparation: "MPT generate" (P:546 step 1; Alg MPTG)  */
/* ------------------------------------------------------------------------- */
typedef struct {
  uint32_t n_sel;      /* number of top entries selected: min(4, K) */
  uint32_t K_sel[4];
  double a[4];
  double Qp;           /* Q' = alpha * P[K-1] */
} word_rec;

/* What: K doubles. P (K doubles, out): P[k] = sum_{j<=k, j != K1} What[j], ascending. */
static void word_prep(const double* What, uint32_t K, double alpha, word_rec* rec, double* P) {
  rec->n_sel = K < 4 ? K : 4;
  for (uint32_t s = 0; s < 4; ++s) { rec->K_sel[s] = 0; rec->a[s] = 0.0; }
  /* top-n by repeated argmax; strict '>' keeps the smaller k on ties (reading #15) */
  for (uint32_t s = 0; s < rec->n_sel; ++s) {
    int64_t best = -1;
    for (uint32_t k = 0; k < K; ++k) {
      int taken = 0;
      for (uint32_t t = 0; t < s; ++t) taken |= (rec->K_sel[t] == k);
      if (taken) continue;
      if (best < 0 || What[k] > What[best]) best = (int64_t)k;
    }
    rec->K_sel[s] = (uint32_t)best;
    rec->a[s] = What[best];
  }
  /* What' = What with its maximum entry set to 0 (Eq 6); prefix for the Q' tree */
  double acc = 0.0;
  for (uint32_t k = 0; k < K; ++k) {
    if (k != rec->K_sel[0]) acc = acc + What[k];
    P[k] = acc;
  }
  rec->Qp = alpha * P[K - 1];
}

/* ------------------------------------------------------------------------- */
/* Per-token three-branch draw (P:546 steps 2-6; Alg P:1513-1537; Alg MPTC    */
/* P:1625-1646), normative [M | S' | Q'] layout (SURVEY 8(c) reading #10).   */
/* ------------------------------------------------------------------------- */
static void token_draw(const word_rec* rec, const double* P, const double* What, const int32_t* Drow,
                       uint32_t K, double alpha, uint32_t g, double u, ezlda_oracle_draw_detail* o) {
  memset(o, 0, sizeof(*o));
  uint32_t L = 0;
  for (uint32_t k = 0; k < K; ++k) L += (uint32_t)Drow[k];
  for (uint32_t s = 0; s < 4; ++s) {
    o->K_sel[s] = rec->K_sel[s];
    o->a[s] = rec->a[s];
    o->C[s] = (s < rec->n_sel) ? (uint32_t)Drow[rec->K_sel[s]] : 0u;
  }
  o->L = L;
  const uint32_t K1 = rec->K_sel[0];
  const double a1 = rec->a[0], a2 = rec->a[1], a3 = rec->a[2], a4 = rec->a[3];
  const uint32_t C1 = o->C[0], C2 = o->C[1], C3 = o->C[2];

  /* step 2-3: M (Eq 8) and S_est (Eq 10, g = min(g, K-1); g == 0: appendix bound) */
  o->M = a1 * ((double)C1 + alpha);
  uint32_t ge = g;
  if (g != 0 && ge > K - 1) ge = K - 1;
  if (g == 0) {
    o->S_est = (double)(L - C1) * a1;
  } else if (ge == 0) {
    o->S_est = 0.0; /* K == 1: no residual topics */
  } else if (ge == 1) {
    o->S_est = a2 * (double)(L - C1);
  } else if (ge == 2) {
    o->S_est = a2 * (double)C2 + a3 * (double)(L - C1 - C2);
  } else {
    o->S_est = (a2 * (double)C2 + a3 * (double)C3) + a4 * (double)(L - C1 - C2 - C3);
  }
  o->Qp = rec->Qp;
  o->thr = o->M / ((o->M + o->S_est) + o->Qp);
  if (u < o->thr) { /* step 3: skipped, stays in the most popular topic */
    o->branch = 0;
    o->topic = K1;
    return;
  }
  /* step 4-5: S' tree over D[d] o What'[v], ascending topic order */
  double Sp = 0.0;
  for (uint32_t k = 0; k < K; ++k)
    if (Drow[k] > 0 && k != K1) Sp = Sp + (double)Drow[k] * What[k];
  o->Sp = Sp;
  o->Z = (o->M + Sp) + o->Qp;
  o->x = u * o->Z;
  const double x = o->x;
  if (x < o->M) { /* step 6: second chance, u < M / (M + S' + Q') */
    o->branch = 1;
    o->topic = K1;
    return;
  }
  if (x < o->M + Sp) { /* S' branch: first k in the prefix list with prefix > y */
    const double y = x - o->M;
    double acc = 0.0;
    uint32_t last = K1;
    for (uint32_t k = 0; k < K; ++k) {
      if (!(Drow[k] > 0 && k != K1)) continue;
      acc = acc + (double)Drow[k] * What[k];
      last = k;
      if (acc > y) {
        o->branch = 2;
        o->topic = k;
        return;
      }
    }
    o->branch = 2;
    o->topic = last; /* past the end (rounding): last k in the list */
    return;
  }
  /* Q' branch: first k != K1 (ascending) with alpha * P[k] > y */
  {
    const double y = (x - o->M) - Sp;
    uint32_t last = K1;
    for (uint32_t k = 0; k < K; ++k) {
      if (k == K1) continue;
      last = k;
      if (alpha * P[k] > y) {
        o->branch = 3;
        o->topic = k;
        return;
      }
    }
    o->branch = 3;
    o->topic = last;
  }
}

int ezlda_oracle_draw_three_branch(const int32_t* Drow, const double* What, uint32_t K, double alpha,
                                   uint32_t g, double u, ezlda_oracle_draw_detail* out) {
  if (!Drow || !What || !out || K == 0 || g > 3) return 1;
  double* P = (double*)malloc(sizeof(double) * K);
  if (!P) return 3;
  word_rec rec;
  word_prep(What, K, alpha, &rec, P);
  token_draw(&rec, P, What, Drow, K, alpha, g, u, out);
  free(P);
  return 0;
}

int ezlda_oracle_draw_grid(const int32_t* Drow, const double* What, uint32_t K, double alpha, uint32_t g,
                           const double* u, uint64_t n, uint32_t* topics, int32_t* branch) {
  if (!Drow || !What || !u || !topics || K == 0 || g > 3) return 1;
  double* P = (double*)malloc(sizeof(double) * K);
  if (!P) return 3;
  word_rec rec;
  word_prep(What, K, alpha, &rec, P);
  for (uint64_t i = 0; i < n; ++i) {
    ezlda_oracle_draw_detail det;
    token_draw(&rec, P, What, Drow, K, alpha, g, u[i], &det);
    topics[i] = det.topic;
    if (branch) branch[i] = det.branch;
  }
  free(P);
  return 0;
}

/* Two-branch ESCA draw as in the Fig 2 walk-through. */
uint32_t ezlda_oracle_draw_two_branch(const int32_t* Drow, const double* What, uint32_t K, double alpha,
                                      double u, double* S_out, double* Q_out, double* uprime,
                                      double* S_prefix, double* Q_prefix) {
  double S = 0.0, Q = 0.0;
  for (uint32_t k = 0; k < K; ++k) {
    S = S + (double)Drow[k] * What[k]; /* prefix-sum of What o D[d] (S tree) */
    Q = Q + alpha * What[k];           /* prefix-sum of What o alpha (Q tree) */
    if (S_prefix) S_prefix[k] = S;
    if (Q_prefix) Q_prefix[k] = Q;
  }
  if (S_out) *S_out = S;
  if (Q_out) *Q_out = Q;
  uint32_t topic = K - 1;
  if (u <= S / (S + Q)) { /* S tree with u' = u (S+Q) (reading #11) */
    double up = u * (S + Q);
    if (uprime) *uprime = up;
    double acc = 0.0;
    for (uint32_t k = 0; k < K; ++k) {
      acc = acc + (double)Drow[k] * What[k];
      if (Drow[k] > 0) topic = k;
      if (acc > up) { topic = k; break; }
    }
  } else { /* Q tree with u' = (1-u)(S+Q) */
    double up = (1.0 - u) * (S + Q);
    if (uprime) *uprime = up;
    double acc = 0.0;
    for (uint32_t k = 0; k < K; ++k) {
      acc = acc + alpha * What[k];
      if (acc > up) { topic = k; break; }
    }
  }
  return topic;
}

/* ------------------------------------------------------------------------- */
/* Inverted index (Fig 5) -- CSR of each doc's positions in the token   */
/* list sorted by (word, doc, input position) (reading #21).                  */
/* ------------------------------------------------------------------------- */
static const uint32_t* g_sort_word;
static const uint32_t* g_sort_doc;
static int cmp_word_doc_pos(const void* pa, const void* pb) {
  uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
  if (g_sort_word[a] != g_sort_word[b]) return g_sort_word[a] < g_sort_word[b] ? -1 : 1;
  if (g_sort_doc[a] != g_sort_doc[b]) return g_sort_doc[a] < g_sort_doc[b] ? -1 : 1;
  return a < b ? -1 : (a > b ? 1 : 0);
}
static int cmp_doc_word_pos(const void* pa, const void* pb) {
  uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
  if (g_sort_doc[a] != g_sort_doc[b]) return g_sort_doc[a] < g_sort_doc[b] ? -1 : 1;
  if (g_sort_word[a] != g_sort_word[b]) return g_sort_word[a] < g_sort_word[b] ? -1 : 1;
  return a < b ? -1 : (a > b ? 1 : 0);
}

void ezlda_oracle_inverted_index(const uint32_t* word_ids, const uint32_t* doc_ids, uint64_t n,
                                 uint32_t n_docs, uint64_t* doc_ofs, uint64_t* pos) {
  uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  for (uint64_t t = 0; t < n; ++t) order[t] = t;
  g_sort_word = word_ids;
  g_sort_doc = doc_ids;
  qsort(order, n, sizeof(uint64_t), cmp_word_doc_pos);
  for (uint32_t d = 0; d <= n_docs; ++d) doc_ofs[d] = 0;
  for (uint64_t t = 0; t < n; ++t) doc_ofs[doc_ids[t] + 1] += 1;
  for (uint32_t d = 0; d < n_docs; ++d) doc_ofs[d + 1] += doc_ofs[d];
  uint64_t* fill = (uint64_t*)calloc(n_docs ? n_docs : 1, sizeof(uint64_t));
  for (uint64_t p = 0; p < n; ++p) { /* scan T in word-sorted order, append p to its doc */
    uint32_t d = doc_ids[order[p]];
    pos[doc_ofs[d] + fill[d]++] = p;
  }
  free(fill);
  free(order);
}

/* ------------------------------------------------------------------------- */
/* Whole-corpus chain                                                          */
/* ------------------------------------------------------------------------- */
struct ezlda_oracle {
  uint64_t N;
  uint32_t n_docs, V, K, g;
  double alpha, beta;
  uint64_t seed, token_base;
  uint32_t* word;       /* [N] input order */
  uint32_t* doc;        /* [N] */
  uint64_t* tg;         /* [N] global doc-major RNG index */
  uint16_t* z;          /* [N] current topics */
  uint64_t* wofs;       /* [V+1] CSR of tokens by word */
  uint64_t* wtok;       /* [N] */
  uint32_t iterations;
  uint32_t branches;    /* 3 = three-branch sampler (default), 2 = two-branch ESCA */
  uint64_t skip_S, skip_final, branch_hist[4];
};

static void recount(const ezlda_oracle* h, int32_t* D, uint32_t* L, int32_t* W, int32_t* nk) {
  const uint32_t K = h->K;
  if (D) memset(D, 0, sizeof(int32_t) * (size_t)h->n_docs * K);
  if (L) memset(L, 0, sizeof(uint32_t) * h->n_docs);
  if (W) memset(W, 0, sizeof(int32_t) * (size_t)h->V * K);
  if (nk) memset(nk, 0, sizeof(int32_t) * K);
  for (uint64_t t = 0; t < h->N; ++t) {
    uint32_t k = h->z[t];
    if (D) D[(size_t)h->doc[t] * K + k] += 1;
    if (L) L[h->doc[t]] += 1;
    if (W) W[(size_t)h->word[t] * K + k] += 1;
    if (nk) nk[k] += 1;
  }
}

int ezlda_oracle_create(const uint32_t* word_ids, const uint32_t* doc_ids, uint64_t n_tokens,
                        uint32_t n_docs, uint32_t V, uint32_t K, double alpha, double beta,
                        uint64_t seed, uint32_t g, uint64_t token_base, ezlda_oracle** out) {
  if (!out) return 1;
  *out = NULL;
  if (!word_ids || !doc_ids || n_tokens == 0 || K == 0 || V == 0 || n_docs == 0) return 1;
  if (!(alpha > 0.0) || !(beta > 0.0) || g > 3) return 1;
  if (K > 65535) return 2;
  for (uint64_t t = 0; t < n_tokens; ++t)
    if (word_ids[t] >= V || doc_ids[t] >= n_docs) return 1;
  ezlda_oracle* h = (ezlda_oracle*)calloc(1, sizeof(ezlda_oracle));
  h->N = n_tokens; h->n_docs = n_docs; h->V = V; h->K = K; h->g = g;
  h->alpha = alpha; h->beta = beta; h->seed = seed; h->token_base = token_base;
  h->word = (uint32_t*)malloc(sizeof(uint32_t) * n_tokens);
  h->doc = (uint32_t*)malloc(sizeof(uint32_t) * n_tokens);
  h->tg = (uint64_t*)malloc(sizeof(uint64_t) * n_tokens);
  h->z = (uint16_t*)malloc(sizeof(uint16_t) * n_tokens);
  h->wofs = (uint64_t*)calloc((size_t)V + 1, sizeof(uint64_t));
  h->wtok = (uint64_t*)malloc(sizeof(uint64_t) * n_tokens);
  memcpy(h->word, word_ids, sizeof(uint32_t) * n_tokens);
  memcpy(h->doc, doc_ids, sizeof(uint32_t) * n_tokens);
  /* doc lengths must fit the 16-bit packing */
  uint32_t* L = (uint32_t*)calloc(n_docs, sizeof(uint32_t));
  for (uint64_t t = 0; t < n_tokens; ++t) L[doc_ids[t]] += 1;
  for (uint32_t d = 0; d < n_docs; ++d)
    if (L[d] > 65535) { free(L); ezlda_oracle_destroy(h); return 2; }
  free(L);
  /* t_g: rank in (doc, word, input position) order, plus the shard's global base (reading #14) */
  uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * n_tokens);
  for (uint64_t t = 0; t < n_tokens; ++t) order[t] = t;
  g_sort_word = h->word;
  g_sort_doc = h->doc;
  qsort(order, n_tokens, sizeof(uint64_t), cmp_doc_word_pos);
  for (uint64_t r = 0; r < n_tokens; ++r) h->tg[order[r]] = token_base + r;
  free(order);
  /* tokens grouped by word (the per-word loop of P:402 / P:546 step 1) */
  for (uint64_t t = 0; t < n_tokens; ++t) h->wofs[h->word[t] + 1] += 1;
  for (uint32_t v = 0; v < V; ++v) h->wofs[v + 1] += h->wofs[v];
  uint64_t* fill = (uint64_t*)calloc(V, sizeof(uint64_t));
  for (uint64_t t = 0; t < n_tokens; ++t) h->wtok[h->wofs[h->word[t]] + fill[h->word[t]]++] = t;
  free(fill);
  /* iteration 0: random initial topics */
  for (uint64_t t = 0; t < n_tokens; ++t) h->z[t] = (uint16_t)ezlda_oracle_init_topic(seed, h->tg[t], K);
  h->iterations = 0;
  h->branches = 3;
  *out = h;
  return 0;
}

int ezlda_oracle_set_sampler(ezlda_oracle* h, uint32_t branches) {
  if (!h || (branches != 2 && branches != 3)) return 1;
  h->branches = branches;
  return 0;
}

void ezlda_oracle_destroy(ezlda_oracle* h) {
  if (!h) return;
  free(h->word); free(h->doc); free(h->tg); free(h->z); free(h->wofs); free(h->wtok);
  free(h);
}

void ezlda_oracle_token_index(const ezlda_oracle* h, uint64_t* t_g) {
  memcpy(t_g, h->tg, sizeof(uint64_t) * h->N);
}

int ezlda_oracle_set_topics(ezlda_oracle* h, const uint16_t* topics, uint32_t iterations_done) {
  for (uint64_t t = 0; t < h->N; ++t)
    if (topics[t] >= h->K) return 1;
  memcpy(h->z, topics, sizeof(uint16_t) * h->N);
  h->iterations = iterations_done;
  return 0;
}

int ezlda_oracle_topics(const ezlda_oracle* h, uint16_t* topics) {
  memcpy(topics, h->z, sizeof(uint16_t) * h->N);
  return 0;
}

uint32_t ezlda_oracle_iterations(const ezlda_oracle* h) { return h->iterations; }

/* What[v][k] for every k (Eq 1-2) into row[K]. */
static void what_row(const ezlda_oracle* h, const int32_t* W, const double* den, uint32_t v, double* row) {
  for (uint32_t k = 0; k < h->K; ++k) row[k] = ((double)W[(size_t)v * h->K + k] + h->beta) / den[k];
}

void ezlda_oracle_what_row(const int32_t* W_row, const int32_t* n_k, uint32_t K, uint32_t V, double beta,
                           double* row) {
  for (uint32_t k = 0; k < K; ++k) {
    const double den = (double)n_k[k] + (double)V * beta;
    row[k] = ((double)W_row[k] + beta) / den;
  }
}

int ezlda_oracle_what(const ezlda_oracle* h, uint32_t v, const int32_t* W_global, const int32_t* nk_global,
                      double* row) {
  if (v >= h->V) return 1;
  int32_t* W = (int32_t*)malloc(sizeof(int32_t) * (size_t)h->V * h->K);
  int32_t* nk = (int32_t*)malloc(sizeof(int32_t) * h->K);
  double* den = (double*)malloc(sizeof(double) * h->K);
  recount(h, NULL, NULL, W, nk);
  if (W_global) memcpy(W, W_global, sizeof(int32_t) * (size_t)h->V * h->K);
  if (nk_global) memcpy(nk, nk_global, sizeof(int32_t) * h->K);
  for (uint32_t k = 0; k < h->K; ++k) den[k] = (double)nk[k] + (double)h->V * h->beta;
  what_row(h, W, den, v, row);
  free(W); free(nk); free(den);
  return 0;
}

int ezlda_oracle_iterate(ezlda_oracle* h, uint32_t n, const int32_t* W_global, const int32_t* nk_global) {
  const uint32_t K = h->K;
  int32_t* D = (int32_t*)malloc(sizeof(int32_t) * (size_t)h->n_docs * K);
  int32_t* W = (int32_t*)malloc(sizeof(int32_t) * (size_t)h->V * K);
  int32_t* nk = (int32_t*)malloc(sizeof(int32_t) * K);
  double* den = (double*)malloc(sizeof(double) * K);
  double* What = (double*)malloc(sizeof(double) * K);
  double* P = (double*)malloc(sizeof(double) * K);
  uint16_t* znew = (uint16_t*)malloc(sizeof(uint16_t) * h->N);
  if (!D || !W || !nk || !den || !What || !P || !znew) {
    free(D); free(W); free(nk); free(den); free(What); free(P); free(znew);
    return 3;
  }
  for (uint32_t it = 0; it < n; ++it) {
    const uint32_t i = h->iterations + 1;
    /* step 1: recount the snapshot from z^{i-1} (Alg codeframe) */
    recount(h, D, NULL, W, nk);
    if (it == 0 && W_global) memcpy(W, W_global, sizeof(int32_t) * (size_t)h->V * K);
    if (it == 0 && nk_global) memcpy(nk, nk_global, sizeof(int32_t) * K);
    for (uint32_t k = 0; k < K; ++k) den[k] = (double)nk[k] + (double)h->V * h->beta;
    /* step 2-3: per word, then per token of that word.  Every draw reads only the snapshot
     * and writes its own znew entry, so the words are independent: the OpenMP build
     * (libezlda_oracle_omp.so, bench.py's all-core CPU leg) splits them over threads with
     * identical results; the default build compiles the pragmas away. */
    uint64_t skS = 0, skF = 0, bh0 = 0, bh1 = 0, bh2 = 0, bh3 = 0;
#ifdef _OPENMP
#pragma omp parallel reduction(+ : skS, skF, bh0, bh1, bh2, bh3)
#endif
    {
      double* What_t = What;
      double* P_t = P;
#ifdef _OPENMP
      What_t = (double*)malloc(sizeof(double) * K);
      P_t = (double*)malloc(sizeof(double) * K);
#pragma omp for schedule(dynamic, 16)
#endif
      for (uint32_t v = 0; v < h->V; ++v) {
        if (h->wofs[v] == h->wofs[v + 1]) continue;
        what_row(h, W, den, v, What_t);
        word_rec rec;
        word_prep(What_t, K, h->alpha, &rec, P_t);
        for (uint64_t q = h->wofs[v]; q < h->wofs[v + 1]; ++q) {
          const uint64_t t = h->wtok[q];
          const double u = ezlda_oracle_uniform(h->seed, i, h->tg[t]);
          if (h->branches == 2) { /* two-branch ESCA draw (Fig 2 text, reading #11); no skip test */
            double S, Q;
            znew[t] = (uint16_t)ezlda_oracle_draw_two_branch(D + (size_t)h->doc[t] * K, What_t, K, h->alpha, u,
                                                             &S, &Q, NULL, NULL, NULL);
            if (u <= S / (S + Q)) bh2 += 1; else bh3 += 1;
            continue;
          }
          ezlda_oracle_draw_detail det;
          token_draw(&rec, P_t, What_t, D + (size_t)h->doc[t] * K, K, h->alpha, h->g, u, &det);
          znew[t] = (uint16_t)det.topic;
          if (det.branch == 0) bh0 += 1;
          else if (det.branch == 1) bh1 += 1;
          else if (det.branch == 2) bh2 += 1;
          else bh3 += 1;
          if (det.branch == 0) skS += 1;
          if (det.branch <= 1) skF += 1;
        }
      }
#ifdef _OPENMP
      free(What_t);
      free(P_t);
#endif
    }
    h->skip_S = skS;
    h->skip_final = skF;
    h->branch_hist[0] = bh0;
    h->branch_hist[1] = bh1;
    h->branch_hist[2] = bh2;
    h->branch_hist[3] = bh3;
    /* step 4: commit all topics simultaneously (snapshot, reading #13) */
    memcpy(h->z, znew, sizeof(uint16_t) * h->N);
    h->iterations = i;
  }
  free(D); free(W); free(nk); free(den); free(What); free(P); free(znew);
  return 0;
}

int ezlda_oracle_counts(const ezlda_oracle* h, int32_t* D, int32_t* W, int32_t* n_k) {
  recount(h, D, NULL, W, n_k);
  return 0;
}

int ezlda_oracle_loglik(const ezlda_oracle* h, int method, const int32_t* W_global,
                        const int32_t* nk_global, double* llpt, double* sum_out) {
  const uint32_t K = h->K;
  int32_t* D = (int32_t*)malloc(sizeof(int32_t) * (size_t)h->n_docs * K);
  uint32_t* L = (uint32_t*)malloc(sizeof(uint32_t) * h->n_docs);
  int32_t* W = (int32_t*)malloc(sizeof(int32_t) * (size_t)h->V * K);
  int32_t* nk = (int32_t*)malloc(sizeof(int32_t) * K);
  double* den = (double*)malloc(sizeof(double) * K);
  double* What = (double*)malloc(sizeof(double) * K);
  if (!D || !L || !W || !nk || !den || !What) {
    free(D); free(L); free(W); free(nk); free(den); free(What);
    return 3;
  }
  recount(h, D, L, W, nk);
  if (W_global) memcpy(W, W_global, sizeof(int32_t) * (size_t)h->V * K);
  if (nk_global) memcpy(nk, nk_global, sizeof(int32_t) * K);
  for (uint32_t k = 0; k < K; ++k) den[k] = (double)nk[k] + (double)h->V * h->beta;
  double total = 0.0;
  for (uint32_t v = 0; v < h->V; ++v) {
    if (h->wofs[v] == h->wofs[v + 1]) continue;
    what_row(h, W, den, v, What);
    double Qfull = 0.0;
    for (uint32_t k = 0; k < K; ++k) Qfull = Qfull + What[k];
    Qfull = h->alpha * Qfull;
    for (uint64_t q = h->wofs[v]; q < h->wofs[v + 1]; ++q) {
      const uint64_t t = h->wtok[q];
      const int32_t* Drow = D + (size_t)h->doc[t] * K;
      const double Ld = (double)L[h->doc[t]] + (double)K * h->alpha;
      double p;
      if (method == 0) { /* Eq (5) as printed: sum_k (D+alpha)/(L+K alpha) * What */
        p = 0.0;
        for (uint32_t k = 0; k < K; ++k) p = p + (((double)Drow[k] + h->alpha) / Ld) * What[k];
      } else { /* identity sum_k (D+alpha) What = S_full + Q_full */
        double Sfull = 0.0;
        for (uint32_t k = 0; k < K; ++k)
          if (Drow[k] > 0) Sfull = Sfull + (double)Drow[k] * What[k];
        p = (Sfull + Qfull) / Ld;
      }
      total = total + log2(p);
    }
  }
  if (sum_out) *sum_out = total;
  if (llpt) *llpt = total / (double)h->N;
  free(D); free(L); free(W); free(nk); free(den); free(What);
  return 0;
}

void ezlda_oracle_last_stats(const ezlda_oracle* h, uint64_t* skip_S, uint64_t* skip_final,
                             uint64_t branch_hist[4]) {
  if (skip_S) *skip_S = h->skip_S;
  if (skip_final) *skip_final = h->skip_final;
  if (branch_hist) memcpy(branch_hist, h->branch_hist, sizeof(h->branch_hist));
}
