// kernels.cu -- sm_100a kernels of the ezLDA three-branch Gibbs hot path.
//
// Per iteration i (snapshot semantics):
//   k_den        den_k = n_k + V beta, What of absent pairs beta / den_k        (Eq 1-2)
//   k_word_prep  per word: What row, top-4 (K1..K4, a1..a4), Q'                  (P:546 step 1)
//   k_doc_warp / k_doc_block
//                per doc: D row rebuilt from z^{i-1} (sort + run-length encode),
//                C_j lookups, MPT skip test; skipped tokens get K1, runs with a
//                failing token are flagged                                       (P:546 steps 2-3)
//   k_sampler    per work item (word, run range): stage What'[v] in shared memory,
//                for each flagged (doc, word) run read the D row once, build S'
//                with a warp scan, draw every failing token of the run with the
//                [M | S' | Q'] layout, then rebuild W and n_k from the item's
//                histogram (skipped tokens count at K1)                         (P:546 steps 4-6,
//                                                                                  P:822-846)
#include <algorithm>
#include <cstdio>

#include "kernels.h"

namespace ezl {

namespace {

constexpr int kDocWarpCap = 512; // doc-pass warp tier: documents up to 512 tokens
constexpr int kDocWarps = 8;
constexpr int kSampWarps = 8;
constexpr int kLlptWarps = 8;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------------------------
// What row staging (Eq 1-2): row[k] = (W[v][k] + beta) / (n_k + V beta), zero padded
// to Kpad.  Dense rows read the int32 row; tail rows start from beta / den_k and
// overwrite the word's nonzeros.
// ---------------------------------------------------------------------------------
__device__ void stage_row(const Dev& d, const Buf& b, uint32_t v, double* row) {
  const uint32_t tid = threadIdx.x, nt = blockDim.x;
  if (v < d.Vd) {
    const int32_t* w = b.Wd + (size_t)v * d.K;
    for (uint32_t k = tid; k < d.Kpad; k += nt) row[k] = (k < d.K) ? ((double)w[k] + d.beta) / d.den[k] : 0.0;
  } else {
    for (uint32_t k = tid; k < d.Kpad; k += nt) row[k] = (k < d.K) ? d.what0[k] : 0.0;
    __syncthreads();
    const uint32_t t = v - d.Vd;
    const uint32_t* tr = b.Wt + d.tofs[t];
    const uint32_t n = b.tnnz[t];
    for (uint32_t e = tid; e < n; e += nt) {
      const uint32_t p = tr[e];
      const uint32_t k = p >> 16;
      row[k] = ((double)(p & 0xFFFFu) + d.beta) / d.den[k];
    }
  }
  __syncthreads();
}

// Chunked prefix of a staged row (the Q' tree of P:384/P:400 in the order this
// implementation fixes): T[c] = sequential sum of the 32 entries of chunk c,
// CP[0] = 0, CP[c+1] = CP[c] + T[c] sequentially, and
//   P(k) := CP[k/32] + (sequential sum of row[32 (k/32) .. k]),
// which a single thread can evaluate (binary search over CP, then a walk of <= 32
// entries).  Used identically by word-prep (Q' = alpha CP[nch]), the sampler (Q'
// descent) and LLPT.
__device__ void chunk_prefix(const double* row, uint32_t nch, double* T, double* CP) {
  for (uint32_t c = threadIdx.x; c < nch; c += blockDim.x) {
    double acc = 0.0;
#pragma unroll 8
    for (uint32_t t = 0; t < 32; ++t) acc = acc + row[c * 32 + t];
    T[c] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    CP[0] = 0.0;
    for (uint32_t c = 0; c < nch; ++c) {
      acc = acc + T[c];
      CP[c + 1] = acc;
    }
  }
  __syncthreads();
}

// Q' prefix table of a staged What' row: QP[k] = alpha * P(k) with P(k) as above (the
// chunk prefix CP[k/32] plus the sequential sum inside the chunk).  QP is non-decreasing
// and QP[Kpad-1] = alpha CP[nch] = Q'; the Q' descent becomes one binary search.
__device__ void q_prefix(const double* row, uint32_t nch, const double* CP, double alpha, double* QP) {
  for (uint32_t c = threadIdx.x; c < nch; c += blockDim.x) {
    double acc = 0.0;
    for (uint32_t t = 0; t < 32; ++t) {
      acc = acc + row[c * 32 + t];
      QP[c * 32 + t] = alpha * (CP[c] + acc);
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------------
// top-4 (value desc, topic asc) -- P:546 step 1, ties to the smaller topic.
// ---------------------------------------------------------------------------------
struct Top4 {
  double v[4];
  uint32_t k[4];
};

__device__ __forceinline__ bool better(double va, uint32_t ka, double vb, uint32_t kb) {
  return va > vb || (va == vb && ka < kb);
}

__device__ __forceinline__ void top4_init(Top4& t) {
#pragma unroll
  for (int i = 0; i < 4; ++i) { t.v[i] = -1.0; t.k[i] = 0xFFFFFFFFu; }
}

__device__ __forceinline__ void top4_insert(Top4& t, double v, uint32_t k) {
  if (!better(v, k, t.v[3], t.k[3])) return;
  t.v[3] = v; t.k[3] = k;
#pragma unroll
  for (int p = 3; p > 0; --p) {
    if (better(t.v[p], t.k[p], t.v[p - 1], t.k[p - 1])) {
      const double tv = t.v[p]; t.v[p] = t.v[p - 1]; t.v[p - 1] = tv;
      const uint32_t tk = t.k[p]; t.k[p] = t.k[p - 1]; t.k[p - 1] = tk;
    }
  }
}

__device__ __forceinline__ void top4_warp_merge(Top4& t) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov[4];
    uint32_t ok[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      ov[i] = __shfl_xor_sync(kFull, t.v[i], o);
      ok[i] = __shfl_xor_sync(kFull, t.k[i], o);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) top4_insert(t, ov[i], ok[i]);
  }
}

// Block-wide ordered compaction: out[pos] = (k << 16) | hist[k] for every k < K with
// hist[k] > 0, ascending k.  Returns nnz in all threads.
__device__ uint32_t block_compact(const uint32_t* hist, uint32_t K, uint32_t* out, uint32_t* s_wsum,
                                  uint32_t* s_run) {
  const uint32_t tid = threadIdx.x, nt = blockDim.x, lane = tid & 31u, warp = tid >> 5, nw = nt >> 5;
  if (tid == 0) *s_run = 0;
  __syncthreads();
  for (uint32_t base = 0; base < K; base += nt) {
    const uint32_t k = base + tid;
    const uint32_t c = (k < K) ? hist[k] : 0u;
    const bool f = c > 0;
    const uint32_t m = __ballot_sync(kFull, f);
    if (lane == 0) s_wsum[warp] = __popc(m);
    __syncthreads();
    uint32_t before = 0;
    for (uint32_t w = 0; w < warp; ++w) before += s_wsum[w];
    const uint32_t pos = *s_run + before + __popc(m & lanemask_lt());
    if (f) out[pos] = (k << 16) | c;
    __syncthreads();
    if (tid == 0) {
      uint32_t tot = 0;
      for (uint32_t w = 0; w < nw; ++w) tot += s_wsum[w];
      *s_run += tot;
    }
    __syncthreads();
  }
  return *s_run;
}

// ---------------------------------------------------------------------------------
// H1: den_k and What of absent pairs.
// ---------------------------------------------------------------------------------
__global__ void k_den(Dev d, Buf cur) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < d.K) {
    const double den = (double)cur.nk[k] + d.Vbeta;
    d.den[k] = den;
    d.what0[k] = d.beta / den;
  }
}

// H1: word-prep ("MPT generate").  One block per word.
__global__ void __launch_bounds__(128) k_word_prep(Dev d, Buf cur) {
  const uint32_t v = blockIdx.x;
  if (d.wtok[v + 1] == d.wtok[v]) return;  // no token of v in this shard
  extern __shared__ __align__(16) unsigned char smem[];
  double* row = reinterpret_cast<double*>(smem);
  double* T = row + d.Kpad;
  double* CP = T + d.nch;
  __shared__ double s_v[4][4];
  __shared__ uint32_t s_k[4][4];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  stage_row(d, cur, v, row);
  Top4 t;
  top4_init(t);
  for (uint32_t k = tid; k < d.K; k += blockDim.x) top4_insert(t, row[k], k);
  top4_warp_merge(t);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) { s_v[warp][i] = t.v[i]; s_k[warp][i] = t.k[i]; }
  }
  __syncthreads();
  if (tid == 0) {
    Top4 f;
    top4_init(f);
    for (uint32_t w = 0; w < (blockDim.x >> 5); ++w)
      for (int i = 0; i < 4; ++i) top4_insert(f, s_v[w][i], s_k[w][i]);
    WordRec r;
    for (int i = 0; i < 4; ++i) {
      const bool ok = f.v[i] >= 0.0;
      r.a[i] = ok ? f.v[i] : 0.0;
      r.K[i] = ok ? (uint16_t)f.k[i] : (uint16_t)0;
    }
    r.Qp = 0.0;
    d.rec[v] = r;
    row[r.K[0]] = 0.0;  // What' (Eq 6): the maximum entry set to 0
  }
  __syncthreads();
  chunk_prefix(row, d.nch, T, CP);
  if (tid == 0) d.rec[v].Qp = d.alpha * CP[d.nch];
  if (v < d.Vd) {  // What'[v] | QP for the sampler's bulk copy (dense words)
    double* out = d.wrow + (size_t)v * d.rs;
    for (uint32_t k = tid; k < d.Kpad; k += blockDim.x) out[k] = row[k];
    q_prefix(row, d.nch, CP, d.alpha, out + d.Kpad);
  }
}

// ---------------------------------------------------------------------------------
// H2+H3: doc pass.  Warp tier: one warp per doc (L <= 512), topics sorted in shared
// memory by a bitonic network, run-length encoded into the packed D row.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t row_lookup(const uint16_t* keys, const uint16_t* cnts, uint32_t n, uint32_t k) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  return (lo < n && keys[lo] == k) ? cnts[lo] : 0u;
}

// Per-token MPT test of one doc's tokens (shared by both doc tiers).  C(k) = D[d][k].
template <typename LookupF>
__device__ __forceinline__ void doc_tokens_skip_test(const Dev& d, const Buf& nxt, uint32_t j0, uint32_t L,
                                                     uint32_t iter, uint32_t start, uint32_t stride,
                                                     LookupF C, unsigned long long& n_skip) {
  for (uint32_t i = start; i < L; i += stride) {
    const uint32_t j = j0 + i;
    const uint32_t v = d.tw[j];
    const WordRec r = d.rec[v];
    const uint32_t C1 = C(r.K[0]);
    const uint32_t C2 = d.geff >= 2 ? C(r.K[1]) : 0u;
    const uint32_t C3 = d.geff >= 3 ? C(r.K[2]) : 0u;
    const double M = mpt_M(r, C1, d.alpha);
    const double thr = mpt_threshold(r, M, C1, C2, C3, L, d.geff);
    const double u = philox_u(d.seed, iter, d.token_base + j);
    if (u < thr) {
      nxt.z[j] = r.K[0];
      ++n_skip;
    } else {
      // the sampler draws it; the marker carries C1 when K <= 32768 (see sample_batch)
      nxt.z[j] = d.zmark ? (uint16_t)(0x8000u | min(C1, 0x7FFFu)) : kUnsampled;
      const uint32_t rid = d.trid[j];
      atomicOr(&d.flags[rid >> 5], 1u << (rid & 31u));
    }
  }
}

// Warp tier, K <= 4096: one warp per doc with a private dense shared-memory histogram
// (two 16-bit counters per word), C_j read straight from it, then an ordered
// compaction over K that writes the packed D row and re-zeroes the counters.
template <bool kSkipTest>
__global__ void __launch_bounds__(kDocWarps * 32) k_doc_hist(Dev d, Buf cur, Buf nxt, const uint32_t* docs,
                                                              uint32_t n_docs, uint32_t iter) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t hw = d.Kpad >> 1;  // counter words per warp
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem) + warp * hw;
  for (uint32_t i = lane; i < hw; i += 32) hist[i] = 0;
  __syncwarp();
  unsigned long long n_skip = 0, n_nnz = 0;
  for (uint32_t idx = blockIdx.x * kDocWarps + warp; idx < n_docs; idx += gridDim.x * kDocWarps) {
    const uint32_t doc = docs[idx];
    const uint32_t j0 = d.dofs[doc];
    const uint32_t L = d.dofs[doc + 1] - j0;
    for (uint32_t i = lane; i < L; i += 32) {
      const uint32_t k = cur.z[j0 + i];
      atomicAdd(&hist[k >> 1], 1u << ((k & 1u) << 4));
    }
    __syncwarp();
    if (kSkipTest) {
      doc_tokens_skip_test(d, nxt, j0, L, iter, lane, 32,
                           [&](uint32_t k) { return (hist[k >> 1] >> ((k & 1u) << 4)) & 0xFFFFu; }, n_skip);
      __syncwarp();
    }
    uint32_t* Drow = d.D + d.ddb[doc];
    uint32_t nnz = 0;
    for (uint32_t base = 0; base < hw; base += 32) {
      const uint32_t w = base + lane;
      const uint32_t x = (w < hw) ? hist[w] : 0u;
      const uint32_t lo = x & 0xFFFFu, hi = x >> 16;
      const uint32_t mlo = __ballot_sync(kFull, lo != 0), mhi = __ballot_sync(kFull, hi != 0);
      const uint32_t lt = lanemask_lt();
      const uint32_t pos = nnz + __popc(mlo & lt) + __popc(mhi & lt);
      if (lo) Drow[kDHdr + pos] = ((2u * w) << 16) | lo;
      if (hi) Drow[kDHdr + pos + (lo != 0)] = ((2u * w + 1u) << 16) | hi;
      if (x) hist[w] = 0;
      nnz += __popc(mlo) + __popc(mhi);
    }
    for (uint32_t p = nnz + lane; p < ((nnz + 7u) & ~7u); p += 32) Drow[kDHdr + p] = 0u;  // pad to 8
    if (lane == 0) {
      Drow[0] = (L << 16) | nnz;
      Drow[1] = j0;
    }
    n_nnz += nnz;
    __syncwarp();
  }
  n_skip = warp_sum(n_skip);
  if (lane == 0) {
    atomicAdd(&d.ctr->d_nnz, n_nnz);
    if (kSkipTest) atomicAdd(&d.ctr->skip_S, n_skip);
  }
}

// Warp tier, K > 4096: topics sorted by a bitonic network in shared memory, then
// run-length encoded.
template <bool kSkipTest>
__global__ void __launch_bounds__(kDocWarps * 32) k_doc_warp(Dev d, Buf cur, Buf nxt, const uint32_t* docs,
                                                              uint32_t n_docs, uint32_t iter) {
  __shared__ uint16_t s_key[kDocWarps][kDocWarpCap];
  __shared__ uint16_t s_ukey[kDocWarps][kDocWarpCap];
  __shared__ uint16_t s_ust[kDocWarps][kDocWarpCap];
  __shared__ uint16_t s_ucnt[kDocWarps][kDocWarpCap];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t idx = blockIdx.x * kDocWarps + warp;
  if (idx >= n_docs) return;
  const uint32_t doc = docs[idx];
  const uint32_t j0 = d.dofs[doc];
  const uint32_t L = d.dofs[doc + 1] - j0;
  const uint32_t dbase = d.ddb[doc];
  uint16_t* buf = s_key[warp];
  uint32_t P2 = 32;
  while (P2 < L) P2 <<= 1;
  for (uint32_t i = lane; i < P2; i += 32) buf[i] = (i < L) ? cur.z[j0 + i] : (uint16_t)0xFFFF;
  __syncwarp();
  for (uint32_t k = 2; k <= P2; k <<= 1) {
    for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
      for (uint32_t i = lane; i < P2; i += 32) {
        const uint32_t ixj = i ^ jj;
        if (ixj > i) {
          const uint16_t a = buf[i], b = buf[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) { buf[i] = b; buf[ixj] = a; }
        }
      }
      __syncwarp();
    }
  }
  // run-length encode the sorted topics
  uint16_t* ukey = s_ukey[warp];
  uint16_t* ust = s_ust[warp];
  uint16_t* ucnt = s_ucnt[warp];
  uint32_t nnz = 0;
  for (uint32_t base = 0; base < L; base += 32) {
    const uint32_t i = base + lane;
    const bool valid = i < L;
    const uint16_t key = valid ? buf[i] : (uint16_t)0;
    const bool head = valid && (i == 0 || key != buf[i - 1]);
    const uint32_t m = __ballot_sync(kFull, head);
    const uint32_t pos = nnz + __popc(m & lanemask_lt());
    if (head) { ukey[pos] = key; ust[pos] = (uint16_t)i; }
    nnz += __popc(m);
  }
  __syncwarp();
  uint32_t* Drow = d.D + dbase;
  for (uint32_t p = lane; p < nnz; p += 32) {
    const uint32_t s0 = ust[p];
    const uint32_t s1 = (p + 1 < nnz) ? (uint32_t)ust[p + 1] : L;
    const uint32_t cnt = s1 - s0;
    ucnt[p] = (uint16_t)cnt;
    Drow[kDHdr + p] = ((uint32_t)ukey[p] << 16) | cnt;
  }
  for (uint32_t p = nnz + lane; p < ((nnz + 7u) & ~7u); p += 32) Drow[kDHdr + p] = 0u;  // pad to 8
  if (lane == 0) {
    Drow[0] = (L << 16) | nnz;
    Drow[1] = j0;
  }
  __syncwarp();
  unsigned long long n_skip = 0;
  if (kSkipTest) {
    doc_tokens_skip_test(d, nxt, j0, L, iter, lane, 32, [&](uint32_t k) { return row_lookup(ukey, ucnt, nnz, k); },
                         n_skip);
  }
  n_skip = warp_sum(n_skip);
  if (lane == 0) {
    atomicAdd(&d.ctr->d_nnz, (unsigned long long)nnz);
    if (kSkipTest) atomicAdd(&d.ctr->skip_S, n_skip);
  }
}

// Block tier: one block per long doc (L > 512): dense shared-memory histogram over K,
// ordered compaction into the packed row; C_j read straight from the histogram.
template <bool kSkipTest>
__global__ void __launch_bounds__(256) k_doc_block(Dev d, Buf cur, Buf nxt, const uint32_t* docs, uint32_t iter) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
  __shared__ uint32_t s_wsum[32], s_run;
  __shared__ unsigned long long s_skip;
  const uint32_t tid = threadIdx.x, nt = blockDim.x;
  const uint32_t doc = docs[blockIdx.x];
  const uint32_t j0 = d.dofs[doc];
  const uint32_t L = d.dofs[doc + 1] - j0;
  const uint32_t dbase = d.ddb[doc];
  for (uint32_t k = tid; k < d.Kpad; k += nt) hist[k] = 0;
  if (tid == 0) s_skip = 0;
  __syncthreads();
  for (uint32_t i = tid; i < L; i += nt) atomicAdd(&hist[cur.z[j0 + i]], 1u);
  __syncthreads();
  uint32_t* Drow = d.D + dbase;
  const uint32_t nnz = block_compact(hist, d.K, Drow + kDHdr, s_wsum, &s_run);
  for (uint32_t p = nnz + tid; p < ((nnz + 7u) & ~7u); p += nt) Drow[kDHdr + p] = 0u;  // pad to 8
  if (tid == 0) {
    Drow[0] = (L << 16) | nnz;
    Drow[1] = j0;
    atomicAdd(&d.ctr->d_nnz, (unsigned long long)nnz);
  }
  if (kSkipTest) {
    unsigned long long n_skip = 0;
    doc_tokens_skip_test(d, nxt, j0, L, iter, tid, nt, [&](uint32_t k) { return hist[k]; }, n_skip);
    n_skip = warp_sum(n_skip);
    if ((tid & 31u) == 0) atomicAdd(&s_skip, n_skip);
    __syncthreads();
    if (tid == 0) atomicAdd(&d.ctr->skip_S, s_skip);
  }
}

// ---------------------------------------------------------------------------------
// H5+H6: the residual three-branch sampler + W/n_k rebuild (one block per item).
// ---------------------------------------------------------------------------------
//
// A block owns one work item (word v, a range of its (doc, word) runs).  What'[v] (Eq 6,
// the K1 entry zeroed) and its chunk prefix CP are staged in shared memory: dense words
// with ONE TMA bulk copy (cp.async.bulk + mbarrier) of the row word-prep wrote, tail words
// from beta / den_k plus the word's packed nonzeros.  Warps take groups of 32 runs from an
// in-block cursor, queue the flagged ones (a token of the run failed the doc pass's MPT
// test) and process them in batches (P:546 steps 4-6):
//
//  A (lane per run)      run table + D-row header; the row is cut into segments of segw
//                        entries (8 = one 32-byte sector); a batch admits runs while the
//                        segment total fits kSegCap;
//  B (lane per segment)  all 32 lanes busy; consecutive lanes read consecutive sectors of
//                        a row (coalesced): partial[s] = sequential sum over the segment
//                        of D[d][k] What'[v][k] in ascending topic order; C1..C3 =
//                        D[d][K1..K3] are picked up by the lane whose segment holds K_j;
//  C (lane per run)      P[s] = P[s-1] + partial[s] sequentially over the run's segments,
//                        S' = P[last]; M (Eq 8), the MPT threshold (Eq 10), Z = M + S' + Q';
//  D (lane per token)    u (Philox), MPT retest (the doc pass already wrote K1 for skipped
//                        tokens), x = u Z lands in [M | S' | Q']; S' descent: the first
//                        segment with P[s] > y (binary search), then the walk
//                        P[s-1] + (sequential sum inside the segment) -- the same prefix
//                        definition, so the walk ends exactly at P[s]; Q' descent: binary
//                        search over CP, then one 32-topic chunk.
// The S' prefix is a two-level (segment, entry) sum, like the Q' prefix: it differs from
// the oracle's single sequential sum by rounding only.
struct RunCounters {
  uint32_t sampled, hitM, runs, words;
};

constexpr int kQueue = 64;  // one batch + one refill group

struct __align__(16) WarpScratch {
  double P[2 * kSegCap];  // prefix checkpoints of the batch's runs, flattened (see sample_batch)
  uint32_t q[kQueue];  // queue of flagged runs
};

// 32-byte (one sector) read-only load
__device__ __forceinline__ void ldg256(const uint32_t* p, uint4& a, uint4& b) {
  asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// D[d][k] What'[v][k] of one packed entry (topic << 16 | count); padding (0) adds +0.0.
// The count is converted exactly with the 2^52 trick (one DADD instead of an I2F.F64).
__device__ __forceinline__ double entry_term(uint32_t w, uint32_t row_s) {
  const double c = __hiloint2double(0x43300000, (int)(w & 0xFFFFu)) - 0x1p52;
  return c * lds_f64(row_s + ((w >> 16) << 3));
}

// sequential sum of the 8 entries of one sector, continuing acc
__device__ __forceinline__ double sector_sum(double acc, const uint4& a, const uint4& b, uint32_t row_s) {
  acc = acc + entry_term(a.x, row_s);
  acc = acc + entry_term(a.y, row_s);
  acc = acc + entry_term(a.z, row_s);
  acc = acc + entry_term(a.w, row_s);
  acc = acc + entry_term(b.x, row_s);
  acc = acc + entry_term(b.y, row_s);
  acc = acc + entry_term(b.z, row_s);
  acc = acc + entry_term(b.w, row_s);
  return acc;
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst_s, const void* src, uint32_t bytes, uint32_t mbar_s) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar_s), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_s),
               "l"(src), "r"(bytes), "r"(mbar_s)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar_s, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(mbar_s), "r"(parity)
        : "memory");
  } while (!done);
}

// C1 = D[d][K1] by binary search in the sorted packed row (fallback path: K > 32768 or
// C1 >= 0x7FFF, where the doc pass cannot carry C1 in the z^i marker).
__device__ __forceinline__ uint32_t row_count(const uint32_t* E, uint32_t nnz, uint32_t k) {
  uint32_t lo = 0, hi = nnz;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((__ldg(E + mid) >> 16) < k) lo = mid + 1u; else hi = mid;
  }
  if (lo < nnz) {
    const uint32_t w = __ldg(E + lo);
    if ((w >> 16) == k) return w & 0xFFFFu;
  }
  return 0u;
}

// One batch of flagged runs (warp-uniform control flow).  Returns the number of queue
// entries consumed.  kSegW: entries per segment (multiple of 16); the per-run state lives
// in the registers of the run's lane and is fetched by shuffles.
template <uint32_t kSegW>
__device__ __forceinline__ uint32_t sample_batch(const Dev& d, const Buf& nxt, const WordRec& rec, uint32_t row_s,
                                                 const double* QP, uint32_t* hist, WarpScratch& ws, uint32_t qn,
                                                 uint32_t iter, RunCounters& rc) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t K1 = rec.K[0];
  // ---- A: lane per run: run table + header, segment admission
  const uint32_t nc = min(qn, 32u);
  uint32_t j0 = 0, ebase = 0, len = 0, nnz = 0, nseg = 0;
  if (lane < nc) {
    const uint32_t r = ws.q[lane];
    j0 = d.run_j0[r];
    const uint32_t dbase = d.run_dbase[r];
    len = d.run_len[r];
    nnz = d.D[dbase] & 0xFFFFu;
    ebase = dbase + kDHdr;
    nseg = (nnz + kSegW - 1u) / kSegW;
  }
  uint32_t sincl = nseg, tincl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, sincl, o);
    if (lane >= (uint32_t)o) sincl += y;
  }
  const uint32_t nb = __popc(__ballot_sync(kFull, lane < nc && sincl <= kSegCap));  // >= 1
  const uint32_t T = __shfl_sync(kFull, sincl, nb - 1u);
  const uint32_t soff = sincl - nseg;
  tincl = (lane < nb) ? len : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, tincl, o);
    if (lane >= (uint32_t)o) tincl += y;
  }
  const uint32_t ntb = __shfl_sync(kFull, tincl, 31);
  const uint32_t tofs = tincl - ((lane < nb) ? len : 0u);
  if (lane < nb) {
    rc.runs += 1;
    rc.words += 1u + nnz;
  }
  // slot (run lane) of the item with index B0 + lane; first = per-run start offsets held by
  // the run lanes (soff / tofs), ascending
  auto slot_of = [&](uint32_t B0, uint32_t first) -> uint32_t {
    const bool inw = lane < nb && first >= B0 && first < B0 + 32u;
    const uint32_t bits = __reduce_or_sync(kFull, inw ? (1u << (first - B0)) : 0u);
    const uint32_t nbefore = __popc(__ballot_sync(kFull, lane < nb && first < B0));
    return nbefore + __popc(bits & (0xFFFFFFFFu >> (31u - lane))) - 1u;
  };
  // ---- B: lane per segment (kSegW entries, 16 = two 32-byte sectors); consecutive lanes
  //      read consecutive sectors of a row.  The segment sums are combined into the run
  //      prefixes by a segmented warp scan (carry across rounds).  Checkpoints: kSec
  //      (kSegW = 16) keeps two per segment, P[2g] = P(before g) + (first sector) and
  //      P[2g+1] = P(end of g), so a descent walks at most one sector; otherwise P[g] = P(end
  //      of g).  S' = the run's last checkpoint.
  constexpr bool kSec = kSegW == 16u;
  double carry = 0.0;
  for (uint32_t B0 = 0; B0 < T; B0 += 32u) {
    const uint32_t g = B0 + lane;
    const uint32_t slot = slot_of(B0, soff);
    const uint32_t s_soff = __shfl_sync(kFull, soff, slot);
    const uint32_t s_ebase = __shfl_sync(kFull, ebase, slot);
    const uint32_t s_nnz = __shfl_sync(kFull, nnz, slot);
    const uint32_t e0 = (g - s_soff) * kSegW;
    const uint32_t* p = d.D + s_ebase + e0;
    double acc = 0.0, acc8 = 0.0;
    if (g < T) {
#pragma unroll
      for (uint32_t b = 0; b < kSegW; b += 16u) {
        uint4 qa = make_uint4(0u, 0u, 0u, 0u), qb = qa, qc = qa, qd = qa;
        if (e0 + b < s_nnz) ldg256(p + b, qa, qb);
        if (e0 + b + 8u < s_nnz) ldg256(p + b + 8u, qc, qd);
        acc = sector_sum(acc, qa, qb, row_s);
        if (kSec) acc8 = acc;
        acc = sector_sum(acc, qc, qd, row_s);
      }
    }
    // segmented inclusive scan over the lanes of one run (lanes >= rs belong to it)
    const uint32_t rs = (s_soff > B0) ? s_soff - B0 : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(kFull, acc, o);
      if (lane >= rs + (uint32_t)o) acc = y + acc;
    }
    const bool cont = s_soff < B0;  // the run started in an earlier round
    if (cont) acc = carry + acc;
    if (kSec) {
      double excl = __shfl_up_sync(kFull, acc, 1);
      if (lane == rs) excl = cont ? carry : 0.0;
      if (g < T) {
        ws.P[2u * g] = excl + acc8;
        ws.P[2u * g + 1u] = acc;
      }
    } else if (g < T) {
      ws.P[g] = acc;
    }
    carry = __shfl_sync(kFull, acc, 31);
  }
  __syncwarp();
  // ---- D: lane per token.  The doc pass left a marker in z^i for the tokens that failed
  //      the MPT test (the others already hold K1): 0x8000 | min(C1, 0x7FFF) when K <=
  //      32768 (d.zmark), else 0xFFFF.
  const double Qp = rec.Qp;
  for (uint32_t B0 = 0; B0 < ntb; B0 += 32u) {
    const uint32_t slot = slot_of(B0, tofs);
    const uint32_t s_j0 = __shfl_sync(kFull, j0, slot);
    const uint32_t s_tofs = __shfl_sync(kFull, tofs, slot);
    const uint32_t s_soff = __shfl_sync(kFull, soff, slot);
    const uint32_t s_nseg = __shfl_sync(kFull, nseg, slot);
    const uint32_t s_ebase = __shfl_sync(kFull, ebase, slot);
    const uint32_t s_nnz = __shfl_sync(kFull, nnz, slot);
    const uint32_t i = B0 + lane;
    if (i >= ntb) continue;
    const uint32_t j = s_j0 + (i - s_tofs);
    const uint32_t zm = nxt.z[j];
    uint32_t C1;
    if (d.zmark) {
      if (!(zm & 0x8000u)) continue;  // skipped by the MPT test (z^i = K1 < 0x8000)
      C1 = zm & 0x7FFFu;
      if (C1 == 0x7FFFu) C1 = row_count(d.D + s_ebase, s_nnz, K1);
    } else {
      if (zm != kUnsampled) continue;
      C1 = row_count(d.D + s_ebase, s_nnz, K1);
    }
    constexpr uint32_t kCk = kSec ? 2u : 1u;  // checkpoints per segment
    const uint32_t c0 = kCk * s_soff, nck = kCk * s_nseg;
    const double Sp = nck ? ws.P[c0 + nck - 1u] : 0.0;
    const double M = mpt_M(rec, C1, d.alpha);
    const double Z = (M + Sp) + Qp;
    const double u = philox_u(d.seed, iter, d.token_base + j);
    const double x = u * Z;
    uint32_t topic;
    if (x < M) {
      topic = K1;  // second chance: u < M / (M + S' + Q')
      rc.hitM += 1;
    } else if (x < M + Sp) {
      // S' branch: first checkpoint with P > y, then the walk from the previous one
      const double y = x - M;
      uint32_t a = c0, b = c0 + nck - 1u;
      while (a < b) {
        const uint32_t mid = (a + b) >> 1;
        if (ws.P[mid] > y) b = mid; else a = mid + 1u;
      }
      const double base = (a > c0) ? ws.P[a - 1u] : 0.0;
      const uint32_t* E = d.D + s_ebase;
      uint32_t last = 0xFFFFFFFFu;
      topic = 0xFFFFFFFFu;
      if (kSec) {  // one sector (8 entries; zero padding past nnz) from registers
        uint4 qa, qb;
        ldg256(E + (a - c0) * 8u, qa, qb);
        const uint32_t wv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
        double acc = 0.0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t w = wv[e];
          if (topic == 0xFFFFFFFFu && w != 0u) {
            const uint32_t k = w >> 16;
            acc = acc + entry_term(w, row_s);
            if (k != K1) {
              last = k;
              if (base + acc > y) topic = k;
            }
          }
        }
      } else {
        const uint32_t e0 = (a - c0) * kSegW;
        const uint32_t e1 = min(e0 + kSegW, s_nnz);
        double acc = 0.0;
        for (uint32_t e = e0; e < e1; ++e) {
          const uint32_t w = __ldg(E + e);
          const uint32_t k = w >> 16;
          acc = acc + entry_term(w, row_s);
          if (k != K1) {
            last = k;
            if (base + acc > y) {
              topic = k;
              break;
            }
          }
        }
      }
      if (topic == 0xFFFFFFFFu) {  // rounding at the end of the walk / of S'
        if (last == 0xFFFFFFFFu) {  // the walked entries hold K1 only: last topic != K1 of the row
          for (uint32_t e = s_nnz; e-- > 0;) {
            const uint32_t k = __ldg(E + e) >> 16;
            if (k != K1) { last = k; break; }
          }
          if (last == 0xFFFFFFFFu) last = K1;
        }
        topic = last;
      }
    } else {
      // Q' branch: first topic k != K1 with alpha P(k) > y (binary search over QP, which
      // is flat across K1); none -> last topic != K1
      const double y = (x - M) - Sp;
      uint32_t a = 0, b = d.Kpad - 1u;
      while (a < b) {
        const uint32_t mid = (a + b) >> 1;
        if (QP[mid] > y) b = mid; else a = mid + 1u;
      }
      if (a == K1 && QP[a] > y) ++a;  // only when K1 = 0 and y < 0
      if (a >= d.K || !(QP[a] > y)) a = (d.K - 1 != K1) ? d.K - 1 : d.K - 2;
      topic = a;
    }
    nxt.z[j] = (uint16_t)topic;
    atomicAdd(&hist[topic], 1u);
    rc.sampled += 1;
  }
  __syncwarp();
  return nb;
}

// W / n_k of one item from its topic histogram (dense rows: atomics, the item may be one
// of several regions of the word; tail rows: ordered compaction into the packed row).
__device__ void item_epilogue(const Dev& d, const Buf& nxt, uint32_t v, const uint32_t* hist, uint32_t* s_wsum,
                              uint32_t* s_run) {
  const uint32_t tid = threadIdx.x;
  if (v < d.Vd) {
    int32_t* Wrow = nxt.Wd + (size_t)v * d.K;
    for (uint32_t k = tid; k < d.K; k += blockDim.x) {
      const uint32_t c = hist[k];
      if (c) {
        atomicAdd(&Wrow[k], (int32_t)c);
        atomicAdd(&nxt.nk[k], (int32_t)c);
      }
    }
  } else {
    const uint32_t t = v - d.Vd;
    const uint32_t nz = block_compact(hist, d.K, nxt.Wt + d.tofs[t], s_wsum, s_run);
    if (tid == 0) nxt.tnnz[t] = nz;
    for (uint32_t k = tid; k < d.K; k += blockDim.x) {
      const uint32_t c = hist[k];
      if (c) atomicAdd(&nxt.nk[k], (int32_t)c);
    }
  }
}

// byte offset of the per-warp scratch in the sampler's dynamic shared memory:
// What' [Kpad] | QP [Kpad] | T [nch] | CP [nch + 1] | hist [Kpad] u32 | (16-aligned) scratch
__host__ __device__ __forceinline__ uint32_t sampler_ws_offset(uint32_t K) {
  const uint32_t nch = (K + 31) / 32;
  const uint32_t b = 2u * nch * 32u * 8u + (2u * nch + 1u) * 8u + nch * 32u * 4u;
  return (b + 15u) & ~15u;
}

#ifndef EZLDA_SAMP_MINB
#define EZLDA_SAMP_MINB 3  // sampler blocks per SM the register allocation must allow
#endif

// shared memory of the sampler: What' row [Kpad] | CP [nch + 1] (one bulk copy, rs doubles)
// | T [nch] | hist [Kpad] u32 | kSampWarps x WarpScratch
__global__ void __launch_bounds__(kSampWarps * 32, EZLDA_SAMP_MINB) k_sampler(Dev d, Buf cur, Buf nxt, uint32_t iter) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* row = reinterpret_cast<double*>(smem);
  double* QP = row + d.Kpad;
  double* T = row + d.rs;
  double* CP = T + d.nch;
  uint32_t* hist = reinterpret_cast<uint32_t*>(CP + d.nch + 1);
  WarpScratch* s_ws = reinterpret_cast<WarpScratch*>(smem + sampler_ws_offset(d.K));
  __shared__ uint32_t s_cursor, s_wsum[32], s_run;
  __shared__ uint32_t s_sampled, s_hitM, s_runs, s_words;
  __shared__ __align__(8) uint64_t s_mbar;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t item = blockIdx.x;
  const uint32_t v = d.item_word[item], r0 = d.item_r0[item], r1 = d.item_r1[item];
  const uint32_t ntok = d.item_ntok[item];
  const uint32_t mbar_s = (uint32_t)__cvta_generic_to_shared(&s_mbar);
  const bool dense = v < d.Vd;
  if (dense && tid == 0) {  // TMA bulk copy of the precomputed What' row + QP
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar_s), "r"(1u) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    bulk_g2s((uint32_t)__cvta_generic_to_shared(row), d.wrow + (size_t)v * d.rs, d.rs * 8u, mbar_s);
  }
  for (uint32_t k = tid; k < d.Kpad; k += blockDim.x) hist[k] = 0;
  if (tid == 0) { s_cursor = 0; s_sampled = 0; s_hitM = 0; s_runs = 0; s_words = 0; }
  const WordRec rec = d.rec[v];
  if (dense) {
    __syncthreads();
    mbar_wait(mbar_s, 0);
  } else {
    stage_row(d, cur, v, row);
    if (tid == 0) row[rec.K[0]] = 0.0;  // What'
    __syncthreads();
    chunk_prefix(row, d.nch, T, CP);
    q_prefix(row, d.nch, CP, d.alpha, QP);
  }
  RunCounters rc{0, 0, 0, 0};
  {
    WarpScratch& ws = s_ws[warp];
    const uint32_t row_s = (uint32_t)__cvta_generic_to_shared(row);
    uint32_t qn = 0;
    bool exhausted = false;
    while (true) {
      // refill the queue with flagged runs (warp-uniform control flow throughout)
      while (qn < 32 && !exhausted) {
        uint32_t grp = 0;
        if (lane == 0) grp = atomicAdd(&s_cursor, 1u);
        grp = __shfl_sync(kFull, grp, 0);
        const uint32_t rb = r0 + grp * 32u;
        if (rb >= r1) {
          exhausted = true;
          break;
        }
        const uint32_t r = rb + lane;
        const bool act = (r < r1) && ((d.flags[r >> 5] >> (r & 31u)) & 1u);
        const uint32_t m = __ballot_sync(kFull, act);
        if (act) ws.q[qn + __popc(m & lanemask_lt())] = r;
        qn += __popc(m);
        __syncwarp();
      }
      if (qn == 0) break;
      uint32_t nb;
      switch (d.segw) {
        case 16u: nb = sample_batch<16u>(d, nxt, rec, row_s, QP, hist, ws, qn, iter, rc); break;
        case 32u: nb = sample_batch<32u>(d, nxt, rec, row_s, QP, hist, ws, qn, iter, rc); break;
        case 64u: nb = sample_batch<64u>(d, nxt, rec, row_s, QP, hist, ws, qn, iter, rc); break;
        case 128u: nb = sample_batch<128u>(d, nxt, rec, row_s, QP, hist, ws, qn, iter, rc); break;
        default: nb = sample_batch<256u>(d, nxt, rec, row_s, QP, hist, ws, qn, iter, rc); break;
      }
      // drop the processed runs from the queue
      const uint32_t keep0 = (lane + nb < qn) ? ws.q[lane + nb] : 0u;
      const uint32_t keep1 = (lane + 32u + nb < qn) ? ws.q[lane + 32u + nb] : 0u;
      __syncwarp();
      if (lane + nb < qn) ws.q[lane] = keep0;
      if (lane + 32u + nb < qn) ws.q[lane + 32u] = keep1;
      qn -= nb;
      __syncwarp();
    }
  }
  {
    const uint32_t smp = warp_sum(rc.sampled), hm = warp_sum(rc.hitM);
    const uint32_t nr = warp_sum(rc.runs), nw = warp_sum(rc.words);
    if (lane == 0) {
      atomicAdd(&s_sampled, smp);
      atomicAdd(&s_hitM, hm);
      atomicAdd(&s_runs, nr);
      atomicAdd(&s_words, nw);
    }
  }
  __syncthreads();
  if (tid == 0) hist[rec.K[0]] += ntok - s_sampled;  // skipped tokens stay at K1
  __syncthreads();
  item_epilogue(d, nxt, v, hist, s_wsum, &s_run);
  if (tid == 0) {
    atomicAdd(&d.ctr->sampled, (unsigned long long)s_sampled);
    atomicAdd(&d.ctr->skip_M, (unsigned long long)s_hitM);
    atomicAdd(&d.ctr->active_runs, (unsigned long long)s_runs);
    atomicAdd(&d.ctr->drow_words, (unsigned long long)s_words);
  }
}

// W / n_k of z (init, set_topics): the item histogram of the current topics.
__global__ void __launch_bounds__(256) k_wcount(Dev d, Buf cur, Buf nxt) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
  __shared__ uint32_t s_wsum[32], s_run;
  const uint32_t tid = threadIdx.x;
  const uint32_t item = blockIdx.x;
  const uint32_t v = d.item_word[item], r0 = d.item_r0[item], r1 = d.item_r1[item];
  for (uint32_t k = tid; k < d.Kpad; k += blockDim.x) hist[k] = 0;
  __syncthreads();
  for (uint32_t r = r0 + tid; r < r1; r += blockDim.x) {
    const uint32_t j0 = d.run_j0[r], len = d.run_len[r];
    for (uint32_t t = 0; t < len; ++t) atomicAdd(&hist[cur.z[j0 + t]], 1u);
  }
  __syncthreads();
  item_epilogue(d, nxt, v, hist, s_wsum, &s_run);
}

// ---------------------------------------------------------------------------------
// H8: LLPT, Eq (5) via sum_k (D+alpha) What = S_full + Q_full, one value per (d, v) run.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(kLlptWarps * 32) k_llpt(Dev d, Buf cur, double* partial) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* row = reinterpret_cast<double*>(smem);
  double* T = row + d.Kpad;
  double* CP = T + d.nch;
  __shared__ double s_acc[kLlptWarps];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t item = blockIdx.x;
  const uint32_t v = d.item_word[item], r0 = d.item_r0[item], r1 = d.item_r1[item];
  stage_row(d, cur, v, row);
  chunk_prefix(row, d.nch, T, CP);
  const double Qfull = d.alpha * CP[d.nch];
  const double Kalpha = (double)d.K * d.alpha;
  double acc = 0.0;
  for (uint32_t r = r0 + warp; r < r1; r += kLlptWarps) {
    const uint32_t dbase = d.run_dbase[r], len = d.run_len[r];
    const uint32_t hdr = d.D[dbase];
    const uint32_t L = hdr >> 16, nnz = hdr & 0xFFFFu;
    const uint32_t* Drow = d.D + dbase + kDHdr;
    double carry = 0.0;
    for (uint32_t c = 0; c * 32u < nnz; ++c) {
      const uint32_t i = c * 32u + lane;
      const uint32_t e = (i < nnz) ? Drow[i] : 0u;
      const double w = (i < nnz) ? (double)(e & 0xFFFFu) * row[e >> 16] : 0.0;
      carry = carry + __shfl_sync(kFull, warp_incl_scan(w), 31);
    }
    const double p = (carry + Qfull) / ((double)L + Kalpha);
    acc = acc + (double)len * log2(p);
  }
  if (lane == 0) s_acc[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kLlptWarps; ++w) s = s + s_acc[w];
    partial[item] = s;
  }
}

__global__ void k_sum(const double* partial, uint32_t n, double* out) {
  __shared__ double s[256];
  double acc = 0.0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) acc = acc + partial[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (uint32_t o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] = s[threadIdx.x] + s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// ---------------------------------------------------------------------------------
// setup / IO
// ---------------------------------------------------------------------------------
__global__ void k_init_topics(Dev d, uint16_t* z) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < d.N) z[j] = (uint16_t)philox_init_topic(d.seed, d.token_base + j, d.K);
}

__global__ void k_topics_to_input(const uint16_t* z, const uint32_t* perm, uint32_t N, uint16_t* out) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < N) out[perm[j]] = z[j];
}

__global__ void k_topics_from_input(const uint16_t* in, const uint32_t* perm, uint32_t N, uint16_t* z) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < N) z[j] = in[perm[j]];
}

}  // namespace

size_t word_prep_smem_bytes(uint32_t K) {
  const uint32_t nch = (K + 31) / 32;
  return (size_t)nch * 32 * 8 + (size_t)nch * 8 + (size_t)(nch + 1) * 8;
}
uint32_t wrow_stride(uint32_t K) { return 2u * ((K + 31) / 32) * 32; }  // What' | QP
uint32_t seg_width(uint32_t K) {  // entries per S' segment: a power of two >= 16 with K <= kSegCap segw
  uint32_t w = 16u;
  while (w * kSegCap < K) w <<= 1;
  return w;
}
size_t sampler_smem_bytes(uint32_t K) { return sampler_ws_offset(K) + sizeof(WarpScratch) * kSampWarps; }
size_t wcount_smem_bytes(uint32_t K) { return (size_t)((K + 31) / 32) * 32 * 4; }
size_t doc_block_smem_bytes(uint32_t K) { return (size_t)((K + 31) / 32) * 32 * 4; }

cudaError_t configure_kernels(uint32_t K) {
  cudaError_t e;
  const int wp = (int)word_prep_smem_bytes(K), sp = (int)sampler_smem_bytes(K), db = (int)doc_block_smem_bytes(K);
  if ((e = cudaFuncSetAttribute(k_word_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, wp))) return e;
  if ((e = cudaFuncSetAttribute(k_llpt, cudaFuncAttributeMaxDynamicSharedMemorySize, wp))) return e;
  if ((e = cudaFuncSetAttribute(k_sampler, cudaFuncAttributeMaxDynamicSharedMemorySize, sp))) return e;
  if ((e = cudaFuncSetAttribute(k_wcount, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wcount_smem_bytes(K))))
    return e;
  if ((e = cudaFuncSetAttribute(k_doc_block<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, db))) return e;
  if ((e = cudaFuncSetAttribute(k_doc_block<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, db))) return e;
  if (K <= 4096) {
    const int dh = kDocWarps * (int)(((K + 31) / 32) * 16) * 4;
    if ((e = cudaFuncSetAttribute(k_doc_hist<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dh))) return e;
    if ((e = cudaFuncSetAttribute(k_doc_hist<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dh))) return e;
  }
  return cudaSuccess;
}

void launch_den(const Dev& d, const Buf& cur, cudaStream_t s) {
  k_den<<<(d.K + 255) / 256, 256, 0, s>>>(d, cur);
}

void launch_word_prep(const Dev& d, const Buf& cur, cudaStream_t s) {
  k_word_prep<<<d.V, 128, word_prep_smem_bytes(d.K), s>>>(d, cur);
}

void launch_doc_pass(const Dev& d, const Buf& cur, const Buf& nxt, const uint32_t* docs_w, uint32_t n_w,
                     const uint32_t* docs_b, uint32_t n_b, uint32_t iteration, bool skip_test, cudaStream_t s) {
  if (n_b) {
    if (skip_test)
      k_doc_block<true><<<n_b, 256, doc_block_smem_bytes(d.K), s>>>(d, cur, nxt, docs_b, iteration);
    else
      k_doc_block<false><<<n_b, 256, doc_block_smem_bytes(d.K), s>>>(d, cur, nxt, docs_b, iteration);
  }
  if (n_w && d.K <= 4096) {
    const uint32_t grid = std::min<uint32_t>((n_w + kDocWarps - 1) / kDocWarps, 148u * 16u);
    const size_t smem = (size_t)kDocWarps * (d.Kpad / 2) * 4;
    if (skip_test)
      k_doc_hist<true><<<grid, kDocWarps * 32, smem, s>>>(d, cur, nxt, docs_w, n_w, iteration);
    else
      k_doc_hist<false><<<grid, kDocWarps * 32, smem, s>>>(d, cur, nxt, docs_w, n_w, iteration);
  } else if (n_w) {
    const uint32_t grid = (n_w + kDocWarps - 1) / kDocWarps;
    if (skip_test)
      k_doc_warp<true><<<grid, kDocWarps * 32, 0, s>>>(d, cur, nxt, docs_w, n_w, iteration);
    else
      k_doc_warp<false><<<grid, kDocWarps * 32, 0, s>>>(d, cur, nxt, docs_w, n_w, iteration);
  }
}

void launch_sampler(const Dev& d, const Buf& cur, const Buf& nxt, uint32_t n_items, uint32_t iteration,
                    bool count_only, cudaStream_t s) {
  if (!n_items) return;
  if (count_only)
    k_wcount<<<n_items, 256, wcount_smem_bytes(d.K), s>>>(d, cur, nxt);
  else
    k_sampler<<<n_items, kSampWarps * 32, sampler_smem_bytes(d.K), s>>>(d, cur, nxt, iteration);
}

void launch_llpt(const Dev& d, const Buf& cur, uint32_t n_items, double* partial, double* out, cudaStream_t s) {
  if (n_items) k_llpt<<<n_items, kLlptWarps * 32, word_prep_smem_bytes(d.K), s>>>(d, cur, partial);
  k_sum<<<1, 256, 0, s>>>(partial, n_items, out);
}

void launch_init_topics(const Dev& d, uint16_t* z, cudaStream_t s) {
  k_init_topics<<<(d.N + 255) / 256, 256, 0, s>>>(d, z);
}

void launch_topics_to_input(const uint16_t* z, const uint32_t* perm, uint32_t N, uint16_t* out, cudaStream_t s) {
  k_topics_to_input<<<(N + 255) / 256, 256, 0, s>>>(z, perm, N, out);
}

void launch_topics_from_input(const uint16_t* in, const uint32_t* perm, uint32_t N, uint16_t* z, cudaStream_t s) {
  k_topics_from_input<<<(N + 255) / 256, 256, 0, s>>>(in, perm, N, z);
}

}  // namespace ezl
