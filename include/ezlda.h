/*
 * ezlda.h -- C ABI of the B200-native (sm_100a) ezLDA three-branch Gibbs hot path.
 *
 * Paper: "ezLDA: Efficient and Scalable LDA on GPUs", arXiv 2007.08725
 * (PAPER.md line numbers are cited as P:n).  The library implements, on one
 * GPU per process, the per-iteration collapsed-Gibbs sweep over the token list
 * T of <wordId, docId, topicId> triplets with the paper's three-branch sampler
 * (Eq 6-10, Fig 4 steps 1-6 P:546), followed by the rebuild of the
 * doc-topic matrix D and word-topic matrix W, for a corpus held
 * resident in HBM.  Multi-GPU: documents are partitioned across ranks and W is
 * summed across ranks every iteration with NCCL.
 *
 * Normative semantics:
 *   - snapshot iterations: iteration i reads D, W, n_k of z^{i-1} only and commits
 *     every z^i at once; the current token is not excluded from its own counts;
 *   - What[v][k] = (W[v][k] + beta) / (n_k + V beta) in fp64 (Eq 1-2);
 *   - u = U53(Philox4x32-10(ctr = (t_g lo, t_g hi, i, 0), key = seed)), where t_g
 *     is the token's global doc-major index in (doc, word, input position) order;
 *     iteration 0 draws z^0 = floor(r0 K / 2^32);
 *   - interval layout [M | S' | Q'] with ascending-topic prefixes, ties to the
 *     smaller topic, and S_est of Eq (10) with depth g.
 * The topics are bit-identical to the CPU oracle's (oracle/, test infrastructure)
 * and do not depend on the performance knobs (dense threshold, split threshold, g,
 * W storage mode, number of GPUs, exact_draws).  options.sampler = 2 selects the
 * paper's two-branch (ESCA) map instead (Eq 3-4): the same conditional,
 * a different chain, equal to the oracle's two-branch chain bit for bit.
 *
 * Conventions
 *   - Ownership: input arrays are read during the call only and copied; output
 *     arrays are caller-allocated.  The library owns all its device memory.
 *   - Errors: every call returns an ezlda_status; no exception or abort crosses
 *     the ABI.  A CUDA or NCCL failure is sticky: later calls on the handle
 *     return EZLDA_E_STATE.  ezlda_last_error() gives a message.
 *   - Device/stream: the library uses the calling thread's current CUDA device
 *     and the stream given in the options (or one it creates).
 *   - Threading: one handle per host thread; calls on a handle are serialised.
 *   - Limits (16+16-bit packing): K <= 65535, doc length <= 65535,
 *     tokens per shard < 2^31 (the setup sorts index tokens with int).  K is further
 *     limited by the sampler's shared-memory slot, which holds the word's fixed-point What'
 *     row (4 K bytes): K <= ~47,000 on B200 (K = 32768, the paper's headline, works);
 *     a larger K returns EZLDA_E_RANGE.
 */
#ifndef EZLDA_H
#define EZLDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ezlda ezlda; /* opaque; owned by the library */

typedef enum {
  EZLDA_OK = 0,
  EZLDA_E_INVALID = 1, /* bad argument: n_tokens = 0, K = 0, alpha <= 0, beta <= 0, id out of range, NULL */
  EZLDA_E_RANGE = 2,   /* packing limit exceeded: K, doc length, tokens per shard (>= 2^31) */
  EZLDA_E_NOMEM = 3,   /* device or host allocation failed */
  EZLDA_E_CUDA = 4,    /* CUDA runtime error (sticky) */
  EZLDA_E_NCCL = 5,    /* NCCL error or NCCL unavailable when world > 1 (sticky) */
  EZLDA_E_STATE = 6    /* handle unusable after an earlier sticky error */
} ezlda_status;

/* W storage mode.  HYBRID: dense int32 rows for words with more
 * tokens than dense_threshold (default K, "larger than the topic number",
 * P:761/765), packed (topic<<16|count) sparse rows for the Zipf tail. */
enum { EZLDA_W_HYBRID = 0, EZLDA_W_ALL_DENSE = 1, EZLDA_W_ALL_SPARSE = 2 };

typedef struct {
  uint32_t struct_size;      /* sizeof(ezlda_options); 0 is accepted                       */
  uint32_t g;                /* S_est depth g in {1,2,3}; 0 -> 2                   */
  uint32_t w_mode;           /* EZLDA_W_*                                                 */
  uint32_t dense_threshold;  /* HYBRID: dense iff c_v > this; 0 -> K              */
  uint32_t split_threshold;  /* large-word region size in tokens; 0 -> 10000     */
  int32_t rank;              /* this process's rank (doc shard index)                     */
  int32_t world;             /* number of ranks; 0 or 1 = single GPU.  world == 1 WITH      */
                             /* nccl_unique_id set: a one-rank NCCL group running the       */
                             /* multi-rank path (all-dense W, per-iteration ncclAllReduce)  */
                             /* on one GPU -- exercises the NCCL calls (tests)              */
  const void* nccl_unique_id;/* 128-byte ncclUniqueId from rank 0 (caller broadcasts it)   */
  uint64_t token_base;       /* global doc-major index of this shard's first token (RNG)  */
  void* stream;              /* cudaStream_t to run on, or NULL (library creates one)      */
  uint32_t input_on_device;  /* 1: word_ids/doc_ids passed to ezlda_create are device ptrs */
  uint32_t no_phase_timing;  /* 1: do not record per-phase CUDA events                     */
  uint32_t doc_block_kb;     /* L2 tiling: cut hot-word sampler items at doc windows of     */
                             /* this many KiB of D rows, run them window-major;            */
                             /* 0 -> 32768 (32 MiB); 0xFFFFFFFF -> one window (off)        */
  uint32_t exact_draws;      /* 1: skip the fixed-point fast path, draw every sampled token */
                             /* in fp64 (identical topics by construction; test knob)      */
  uint32_t sampler;          /* 0 or 3: the three-branch sampler; 2: the two-branch */
                             /* ESCA sampler (Eq 3-4, Alg P:1481-1507) on the same   */
                             /* D/W rebuild -- the paper's baseline (reading #11 of SURVEY 8c). */
                             /* Any other value -> EZLDA_E_INVALID.                             */
  uint64_t local_group;      /* test hook, world > 1: nonzero key = the ranks are handles of */
                             /* THIS process on one device (one host thread per rank); the  */
                             /* W / n_k merge is an in-process device sum instead of NCCL.  */
                             /* Every rank of a key must pass the same world (else E_INVALID)*/
  uint32_t debug_flags;      /* test hooks forcing rarely taken paths (EZLDA_DEBUG_*); the   */
                             /* topics do not depend on them                                */
  uint32_t schedule;         /* sampler work schedule (hierarchical balancing): */
                             /* 0: items split every split_threshold tokens and at L2 doc   */
                             /*    windows, heavy first, rebuilt every iteration from the   */
                             /*    flagged runs (items without one never reach the sampler) */
                             /* 1: the same static list, every item staged every iteration  */
                             /* 2: no balancing: one item per word, in word order (ablation)*/
                             /* Performance only: the topics do not depend on it.           */
} ezlda_options;

/* debug_flags bits.  NO_TAIL_ROWS: word-prep precomputes the fixed-point rows of the dense
 * words only, so every tail-word item is staged by a sampler warp (the path large V x K
 * shards take when the rows do not fit).  C1_LOOKUP: the doc pass never carries C1 in the
 * z^i marker, so every sampled token looks C1 up in the packed D row (the path of
 * C1 >= 0x7FFF).  DPERM_ON / DPERM_OFF: force the sector-interleaved D-row layout on / off
 * (by default it is used when K <= 4096 and the shard averages >= 192 tokens per doc).
 * NO_W_DELTA (world > 1): the dense W block is always exchanged as int32 local counts (by
 * default it goes as packed 16-bit deltas against the previous W whenever they fit). */
enum {
  EZLDA_DEBUG_NO_TAIL_ROWS = 1u,
  EZLDA_DEBUG_C1_LOOKUP = 2u,
  EZLDA_DEBUG_DPERM_ON = 4u,
  EZLDA_DEBUG_DPERM_OFF = 8u,
  EZLDA_DEBUG_NO_W_DELTA = 16u
};

/* Compressed sparse rows of a count matrix, caller-allocated.  Pass col = val = NULL
 * to query nnz (row_ptr may also be NULL then).  row_ptr has rows+1 entries. */
typedef struct {
  uint64_t* row_ptr;
  uint16_t* col;
  int32_t* val;
  uint64_t nnz;  /* in: capacity of col/val; out: number of nonzeros */
  uint32_t rows; /* out */
} ezlda_csr;

/* Counters and timings of the last completed iteration (all fields valid after
 * ezlda_iterate; times are CUDA-event milliseconds on the library stream). */
typedef struct {
  uint32_t iteration;        /* index i of the last completed iteration (1-based)          */
  double ms_total;           /* whole iteration                                            */
  double ms_wordprep;        /* H1: den_k, What, top-(g+1), Q' (P:546 step 1)             */
  double ms_docpass;         /* H2+H3: D rebuild, C_j, MPT skip test (steps 2-3)          */
  double ms_sample;          /* H5+H6: residual sampling + W/n_k rebuild (steps 4-6)      */
  double ms_allreduce;       /* H7: cross-GPU W merge (0 when world == 1)                 */
  uint64_t n_tokens;         /* tokens of this shard                                       */
  uint64_t skip_S;           /* tokens assigned K1 by the MPT test ("skip S")       */
  uint64_t skip_final;       /* tokens assigned K1 without a tree descent (>= skip_S)      */
  uint64_t sampled;          /* tokens that went through S' construction                   */
  uint64_t active_runs;      /* (doc, word) runs holding at least one sampled token        */
  uint64_t drow_words;       /* 32-bit D-row words read by the sampler (headers included)  */
  uint64_t d_nnz;            /* nonzeros of D written by the doc pass                      */
  double model_bytes;        /* DESIGN.md byte model of the whole iteration (algorithmic)  */
  double model_bytes_sample; /* ... of the sampler kernel alone                            */
  double model_bytes_docpass;/* ... of the doc-pass kernels                                */
  uint64_t kernel_launches;  /* library kernels launched by the iteration                  */
  uint64_t exact_redraws;    /* sampled tokens redrawn on the exact fp64 path (fixed-point decision
                                not certified by its error margin)      */
  double exchange_bytes;     /* H7 collective payload of the iteration (world > 1): all-reduce  */
                             /* of the dense W block (packed 16-bit deltas: 2 B per entry, or  */
                             /* int32 counts: 4 B) + u16 all-gather of the tail topics (output */
                             /* size); 0 when world == 1                                       */
  double ms_sampler_kernel;  /* the k_sampler launch alone (inside ms_sample, which also holds  */
                             /* the H4 item schedule and the n_k column sums)                   */
} ezlda_iter_stats;

/* Build the resident corpus and draw z^0 (iteration 0).
 *   word_ids, doc_ids: n_tokens entries each (host memory unless opts->input_on_device),
 *     word_ids[t] < V, doc_ids[t] < n_docs (doc ids local to this shard).
 *   V: vocabulary size (global; enters What through V beta).  K: topics.
 *   alpha, beta > 0 (paper: 50/K and 0.01).  seed: Philox key.
 *   opts: may be NULL (paper defaults, single GPU).  out: receives the handle.
 * Returns EZLDA_OK or an error; on error *out is NULL and ezlda_last_error(NULL) explains. */
ezlda_status ezlda_create(const uint32_t* word_ids, const uint32_t* doc_ids, uint64_t n_tokens,
                          uint32_t n_docs, uint32_t V, uint32_t K, double alpha, double beta,
                          uint64_t seed, const ezlda_options* opts, ezlda** out);

/* Run n_iters snapshot iterations (Fig 4 steps 1-6 + D/W rebuild). */
ezlda_status ezlda_iterate(ezlda* h, uint32_t n_iters);

/* State after the last completed iteration, in the caller's ids:
 *   topics[n_tokens] in input order (or NULL); n_k[K] (or NULL);
 *   W: V rows in original word ids (or NULL); D: n_docs rows (or NULL). */
ezlda_status ezlda_counts(ezlda* h, uint16_t* topics, int32_t* n_k, ezlda_csr* W, ezlda_csr* D);

/* Replace the state with caller topics (input order, each < K; host or device memory) as if
 * `iterations_done` iterations had completed (resume / test hook).  Rebuilds W and n_k.
 * A topic >= K returns EZLDA_E_INVALID and leaves the state unchanged. */
ezlda_status ezlda_set_topics(ezlda* h, const uint16_t* topics, uint32_t iterations_done);

/* Log-likelihood per token, Eq (5), log2, of the current state; for
 * world > 1 the sum and token count are reduced over all ranks. */
ezlda_status ezlda_loglik(ezlda* h, double* llpt);

/* Counters/timings of the last iteration (synchronises the library stream). */
ezlda_status ezlda_stats(const ezlda* h, ezlda_iter_stats* last);

/* Field-wise sums of the per-iteration stats over every iteration since the previous
 * reset (or create); sum->iteration receives the number of iterations summed.
 * reset != 0 starts a new window.  Synchronises the library stream. */
ezlda_status ezlda_stats_sum(ezlda* h, ezlda_iter_stats* sum, int reset);

/* Message of the last error on h, or of the last failed ezlda_create on this thread (h NULL). */
const char* ezlda_last_error(const ezlda* h);

/* Free everything (safe on NULL). */
void ezlda_destroy(ezlda* h);

/* Size in bytes of the ncclUniqueId expected by ezlda_options.nccl_unique_id (128), and a
 * helper that creates one (rank 0 only; returns EZLDA_E_NCCL if NCCL cannot be loaded). */
size_t ezlda_nccl_id_size(void);
ezlda_status ezlda_nccl_get_unique_id(void* id_out);

#ifdef __cplusplus
}
#endif
#endif /* EZLDA_H */
