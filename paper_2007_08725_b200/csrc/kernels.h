// kernels.h -- device state layout and kernel launchers of the ezLDA hot path.
//
// HBM layout (one shard; N tokens, Dn docs, R (doc, word) runs, V words, K topics):
//   doc-major token arrays (j in [0, N), docs contiguous, tokens of a doc sorted by word):
//     tw[j]   u32  relabelled word id (words ordered by count desc)
//     trid[j] u32  index of the token's run in word-major run order
//     z[2][j] u16  topics, double-buffered (snapshot semantics)
//     perm[j] u32  input index of token j (output order only)
//   dofs[Dn+1] u32 token offsets of docs; D rows at ddb[d] (32-byte aligned = one sector,
//     capacity 8 + roundup8(min(L_d, K)) words; entries start 32-byte aligned after an
//     8-word header and are zero padded to a multiple of 8 entries, so the sampler reads
//     whole sectors without masking):
//     D[ddb] = (L_d << 16) | nnz_d, D[ddb+1] = dofs[d], D[ddb+8+i] = (topic << 18) | count
//     sorted by topic (packed CSR; rebuilt every iteration); long-doc
//     shards with K <= 4096 (Dev::dperm): entries 128-byte aligned (ddb = 24 mod 32 words),
//     capacity 32 + roundup64(min(L_d, K)), logical entry i at D[ddb+8+d_phys(i)] (below)
//   word-major runs r in [0, R) (runs of word v contiguous, docs ascending):
//     run_j0[r] u32 first doc-major token, run_dbase[r] u32 D-row base, run_len[r] u16
//   flags[R/32] u32: run r holds a token that failed the MPT skip test (L2 resident)
//   W: dense rows int32 [Vd x K] for words v < Vd, packed sparse tail rows (capacity
//     min(c_v, K) at tofs[v-Vd]) with tnnz[v-Vd]; double-buffered with n_k[K].
//   rec[V] WordRec (48 B): top-4 topics/values and Q' of every word.
//   wrow[Vw][rs_bytes]: sampler heads of the words with a live item: u32 m[Kpad] (fixed-point
//     What', K1 entry 0) | f64 {2^-s, 2^s, 2^-t, 2^t} | u32 qfx[Kpad] (fixed-point Q' prefix,
//     XOR-swizzled within 32-topic chunks: q_swz) | u32 ce[] (its chunk ends); bulk-copied (TMA)
//     into a sampler slot.  Words v >= Vw (when
//     V heads do not fit in HBM) are staged by a sampler warp (stage_row_warp).
//   items: (word, run range, tokens): the sampler's work list, heavy first.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

namespace ezl {

constexpr uint16_t kUnsampled = 0xFFFFu;  // z^i of a token the sampler must draw (K <= 65535)
// packed D entry: (topic << dt) | count, count < 2^16.  dt = 18 when K <= 16384 (topic < 2^14):
// the byte offset of topic in a u32 table is then simply entry >> 16 (one LEA.HI per gather);
// dt = 16 for larger K (topic < 2^16)
constexpr uint32_t kDTSmall = 18, kDTLarge = 16;
constexpr uint32_t kDTSmallMaxK = 16384;
__host__ __device__ __forceinline__ uint32_t d_shift(uint32_t K) { return K <= kDTSmallMaxK ? kDTSmall : kDTLarge; }
__host__ __device__ __forceinline__ uint32_t d_entry(uint32_t k, uint32_t c, uint32_t dt) { return (k << dt) | c; }
__host__ __device__ __forceinline__ uint32_t d_topic(uint32_t w, uint32_t dt) { return w >> dt; }
constexpr uint32_t kDHdr = 8;  // header words in front of every packed D row (one 32 B sector)
// Sector-interleaved D rows (K <= 4096, Dev::dperm).  The sampler reads a row as 16-entry
// segments, one per lane, two 32-byte sectors each; stored in topic order, the first load of a
// warp (sector 0 of 32 consecutive segments) would touch 16 lines and use half of each.  So the
// entries are kept in 64-entry blocks (two 128-byte lines, the row's entries starting on a line)
// whose logical (topic-sorted) sector s = 2 g + h of the block's segment g is stored at physical
// sector 4 h + g: the first sectors of a block's four segments fill one line, the second
// sectors the other.  Logical order (and every prefix, checkpoint and search) is unchanged;
// only addresses are mapped.
__host__ __device__ __forceinline__ uint32_t d_psec(uint32_t s) { return ((s & 1u) << 2) | ((s >> 1) & 3u); }
__host__ __device__ __forceinline__ uint32_t d_phys(uint32_t e) {  // logical entry -> physical word
  return (e & ~63u) | (d_psec((e >> 3) & 7u) << 3) | (e & 7u);
}
__host__ __device__ __forceinline__ uint32_t d_at(uint32_t perm, uint32_t e) { return perm ? d_phys(e) : e; }
#ifndef EZLDA_DPERM
#define EZLDA_DPERM 1
#endif
constexpr bool kDPermOn = EZLDA_DPERM != 0;  // build switch (A/B): 0 keeps every row in topic order
constexpr uint32_t kDPermMaxK = 4096;  // the interleaved layout is used iff K <= this (sampler <16, 8> path)
#ifndef EZLDA_SEGCAP
#define EZLDA_SEGCAP 256
#endif
constexpr uint32_t kSegCap = EZLDA_SEGCAP;  // sampler: S' segments per warp batch

struct Counters {  // device-side per-iteration counters
  unsigned long long skip_S, skip_M, sampled, active_runs, drow_words, d_nnz;
  unsigned long long item_ctr;  // sampler work-list cursor (claimed items)
  unsigned long long exact;     // tokens redrawn on the exact fp64 path
  unsigned long long items;     // items the sampler armed (this iteration's live items)
};

struct Dev {
  // sizes and parameters
  uint32_t N, Dn, V, K, Kpad, nch, Vd, geff;
  uint32_t nslots;   // sampler item slots per block (sampler_layout(K))
  uint32_t hist_global;  // 1: slot histograms in hist_scratch (large K), 0: in shared memory
  uint32_t hist_bitmap;
  uint32_t qfx_global;   // 1 (large K): the fixed-point Q' table is searched in HBM, not staged  // 1 (K >= 2048): item epilogues visit only the topics marked in a bitmap
  uint32_t slot_bytes, ws_bytes;  // sampler shared-memory layout
  uint32_t* hist_scratch;  // [grid * nslots * Kpad] (zero between items)
  uint32_t* qfx_scratch;   // [grid * nslots * Kpad] fixed-point Q' tables in HBM (qfx_global)
  uint32_t exact_all;  // 1: every sampled token takes the exact fp64 path (test/ablation knob)
  uint32_t branches;   // 3: three-branch sampler (default); 2: two-branch ESCA mode (NEXT-1)
  double* tbw;         // two-branch mode: [V * Kpad] What rows (Eq 1-2)
  double* tbq;         // two-branch mode: [V * Kpad] Q tree prefix sum_{j<=k} alpha What_j
  uint32_t zmark;  // K <= 32768: the doc pass marks z^i of a failing token as 0x8000 | min(C1, c1_cap)
  uint32_t c1_cap; // 0x7FFF; a marker equal to it sends the sampler to the packed-row lookup of C1 (debug
                   // flag EZLDA_DEBUG_C1_LOOKUP sets it to 0: every failing token takes the lookup)
  uint32_t sampler_grid;  // persistent sampler grid of this handle (SMs x resident blocks, configure_kernels)
  uint32_t segw;  // entries per S' segment (power of two >= 16; ceil(K / segw) <= kSegCap)
  uint32_t segsub;  // entries per S' checkpoint chunk (8: one per sector; or segw)
  uint32_t segfb;   // fallback segment width for runs longer than kSegCap x segw (0: none)
  uint32_t dt;      // topic shift of the packed D entries (d_shift(K))
  uint32_t dperm;   // 1: sector-interleaved D rows (d_phys; K <= kDPermMaxK), entries 128-byte aligned
  uint32_t grp;     // runs per sampler work claim (32; smaller at large K, sampler_group_runs)
  double alpha, beta, Vbeta;
  uint64_t seed, token_base;
  PhiloxKeys pk;   // Philox round keys of seed (philox_keys)
  // static structure
  const uint32_t* dofs;
  const uint32_t* ddb;     // [Dn] D-row base of each doc (multiple of 8 words; dperm: 24 mod 32)
  const uint32_t* tw;
  const uint2* twr;       // [N] (tw, run id) per doc-major token (doc pass: one 8-byte load)
  const uint32_t* run_j0;
  const uint32_t* run_dbase;
  const uint16_t* run_len;
  const uint32_t* tofs;    // [V - Vd + 1] tail row offsets
  const uint32_t* wtok;    // [V + 1] token offsets per word (relabelled ids)
  const uint32_t* item_word;
  const uint32_t* item_r0;
  const uint32_t* item_r1;
  const uint32_t* item_ntok;
  // per-iteration schedule (H4): the items holding a flagged run, in the static heavy-first
  // order (item_act[0 .. *n_act)); nullptr = every item
  const uint32_t* item_act;
  const uint32_t* n_act;
  uint8_t* item_live;  // [items] 1 iff the item has a flagged run (k_item_schedule)
  // dynamic state
  uint32_t* D;
  uint32_t* flags;
  WordRec* rec;
  WordRecM* recm;   // [V] a0, a1, a2, Q' of rec (doc pass, g <= 2)
  uint32_t* reck;   // [V] K1 | K2 << 16 of rec (doc pass, g <= 2)
  double* den;    // [K] n_k + V beta
  double* what0;  // [K] beta / den_k (What of an absent (v, k) pair)
  uint32_t* w0ord;  // [K] topics by what0 desc, ties by topic asc (K > 4096 with tail words; per iteration)
  double* twv;      // [tail capacity] What = (W + beta) / den_k of each tail nonzero (k_word_rec_tail scratch)
  double* inv_den;  // [K] 1 / den_k (the sampler's fixed-point heads, stage_row_warp)
  double* qexact;   // [V * nch] exact running sums P_v(32 c + 31) of the word-prep (exact redraws)
  unsigned char* wrow;  // [Vw * rs_bytes] sampler heads m | scales | qfx | ce (k_word_heads)
  uint32_t Vw;          // words v < Vw have a precomputed head (V, or Vd when V heads do not fit)
  uint32_t rs_bytes;    // head_bytes(K)
  uint8_t* word_live;   // [V] 1 iff the word has a live item this iteration (nullptr: every word)
  Counters* ctr;
};

// Double-buffered pieces of the state.
struct Buf {
  uint16_t* z;
  int32_t* Wd;      // dense rows [Vd * K]
  uint32_t* Wt;     // tail packed rows
  uint32_t* tnnz;   // [V - Vd]
  int32_t* nk;      // [K]
};

// ----- per-iteration kernels -----
void launch_den(const Dev& d, const Buf& cur, cudaStream_t s);
void launch_word_prep(const Dev& d, const Buf& cur, cudaStream_t s);  // word records (top-4, Q')
void launch_word_heads(const Dev& d, const Buf& cur, cudaStream_t s);  // sampler heads of live words
uint32_t head_bytes(uint32_t K);
// doc pass over the two length tiers; skip_test=false only rebuilds D (for counts/loglik)
void launch_doc_pass(const Dev& d, const Buf& cur, const Buf& nxt, const uint32_t* docs_w, uint32_t n_w,
                     const uint32_t* docs_b, uint32_t n_b, uint32_t iteration, bool skip_test, cudaStream_t s);
// sampler over items; count_only=true rebuilds W/n_k of `cur.z` into `nxt` (init, set_topics)
void launch_sampler(const Dev& d, const Buf& cur, const Buf& nxt, uint32_t n_items, uint32_t iteration,
                    bool count_only, cudaStream_t s);
// H4: mark the items with a flagged run (item_live) and write the W / n_k contribution of the
// others (every token skipped, so all of them stay at K1) into nxt
void launch_item_schedule(const Dev& d, const Buf& nxt, uint32_t n_items, cudaStream_t s);
// two-branch (ESCA) mode: What rows + Q prefixes of every word, then one draw per token
// (D rows already rebuilt from cur.z) into nxt.z
// (and W / n_k of the new topics into nxt).  K small enough for the word's tables in shared
// memory: one word-major kernel; else What / Q tables in HBM, a doc-major draw, k_wcount.
void launch_two_branch(const Dev& d, const Buf& cur, const Buf& nxt, uint32_t n_items, uint32_t iteration,
                       cudaStream_t s);
bool two_branch_word_major(uint32_t K);
// H6: n_k = sum_v W[v][k] of the completed W (column sums of the dense block + the tail rows'
// entries): a two-level reduction, per block in shared memory then one atomic per (block, topic)
void launch_nk(const Dev& d, const Buf& b, cudaStream_t s);
// H7 (world > 1): global tail rows from every rank's all-gathered word-major tail topics
void launch_tail_rebuild(const Dev& d, const Buf& nxt, const uint16_t* tz_all, const uint32_t* off, uint32_t world,
                         uint64_t tail_max, cudaStream_t s);
// scratch: llpt_scratch_doubles(K) doubles, used when the fp64 row does not fit shared memory
void launch_llpt(const Dev& d, const Buf& cur, uint32_t n_items, double* partial, double* out, double* scratch,
                 cudaStream_t s);
size_t llpt_scratch_doubles(uint32_t K);
size_t llpt_smem_bytes(uint32_t K);

// ----- setup / IO kernels -----
void launch_init_topics(const Dev& d, uint16_t* z, cudaStream_t s);
void launch_topics_to_input(const uint16_t* z, const uint32_t* perm, uint32_t N, uint16_t* out, cudaStream_t s);
void launch_topics_from_input(const uint16_t* in, const uint32_t* perm, uint32_t N, uint16_t* z, cudaStream_t s);

size_t sampler_smem_bytes(uint32_t K);
uint32_t sampler_slots(uint32_t K);  // pipelined item slots per sampler block (0: K too large)
struct SamplerLayout {
  uint32_t nslots, hist_global, qfx_global, slot_bytes, ws_bytes;
  size_t smem_bytes;
};
SamplerLayout sampler_layout(uint32_t K);
void seg_config(uint32_t K, uint32_t* segw, uint32_t* sub, uint32_t* fb);
uint32_t sampler_group_runs(uint32_t K);
size_t doc_block_smem_bytes(uint32_t K);
// Raise the dynamic shared-memory limits of the kernels K needs (never lowered: handles with
// different K may be alive at once) and return this K's persistent sampler grid in *grid.
cudaError_t configure_kernels(uint32_t K, uint32_t* grid);

}  // namespace ezl
