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
#include <cstdio>

#include "kernels.h"

namespace ezl {

namespace {

constexpr int kDrowCap = 1024;   // D-row entries staged per sampler warp (4 KB)
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

// Chunked prefix of a staged row: T[c] = warp-scan total of chunk c (32 entries),
// CP[0] = 0, CP[c+1] = CP[c] + T[c] sequentially.  P(k) := CP[k/32] + scan_c(k%32).
// Used identically by word-prep (Q'), the sampler (Q' descent) and LLPT.
__device__ void chunk_prefix(const double* row, uint32_t nch, double* T, double* CP) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (uint32_t c = warp; c < nch; c += nw) {
    const double s = warp_incl_scan(row[c * 32 + lane]);
    if (lane == 31) T[c] = s;
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
  __shared__ uint32_t s_K1;
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
    s_K1 = r.K[0];
    row[r.K[0]] = 0.0;  // What' (Eq 6): the maximum entry set to 0
  }
  __syncthreads();
  chunk_prefix(row, d.nch, T, CP);
  if (tid == 0) d.rec[v].Qp = d.alpha * CP[d.nch];
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
      const uint32_t rid = d.trid[j];
      atomicOr(&d.flags[rid >> 5], 1u << (rid & 31u));
    }
  }
}

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
  const uint32_t dbase = j0 + 2u * doc;
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
    Drow[2 + p] = ((uint32_t)ukey[p] << 16) | cnt;
  }
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
  const uint32_t dbase = j0 + 2u * doc;
  for (uint32_t k = tid; k < d.Kpad; k += nt) hist[k] = 0;
  if (tid == 0) s_skip = 0;
  __syncthreads();
  for (uint32_t i = tid; i < L; i += nt) atomicAdd(&hist[cur.z[j0 + i]], 1u);
  __syncthreads();
  uint32_t* Drow = d.D + dbase;
  const uint32_t nnz = block_compact(hist, d.K, Drow + 2, s_wsum, &s_run);
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
struct RunCounters {
  uint32_t sampled, hitM, runs, words;
};

// Warp-cooperative processing of one flagged run (doc d, word v), P:546 steps 4-6:
// the D row is read once (staged in this warp's shared buffer), each lane takes a
// contiguous block of B entries (ascending topic order) and sums D[d][k] What'[v][k]
// sequentially, one warp scan turns the 32 block sums into block offsets O_l, and
//   prefix(entry) = O_l + (sequential partial within the block),  T_l = O_l + P_l,
//   S' = T of the lane holding the last entry.
// A descent picks the first lane with T_l > y and walks that lane's block alone.  Each
// token of the run then redraws its u, repeats the MPT test and, if it fails, lands
// in [M | S' | Q'].
__device__ __forceinline__ void warp_max_u32(uint32_t& x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(kFull, x, o));
}

__device__ __forceinline__ void sample_run(const Dev& d, const Buf& nxt, const WordRec& rec, const double* row,
                                           const double* CP, uint32_t* hist, uint32_t* sbuf, uint32_t r,
                                           uint32_t iter, RunCounters& rc) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t j0 = d.run_j0[r];
  const uint32_t dbase = d.run_dbase[r];
  const uint32_t len = d.run_len[r];
  const uint32_t* Dp = d.D + dbase;
  const uint32_t hdr = Dp[0];
  const uint32_t L = hdr >> 16, nnz = hdr & 0xFFFFu;
  const uint32_t* Drow = Dp + 2;
  const uint32_t K1 = rec.K[0], K2 = rec.K[1], K3 = rec.K[2];
  // stage (coalesced) when it fits; otherwise read the blocks straight from global memory
  const bool staged = nnz <= (uint32_t)kDrowCap;
  if (staged) {
    for (uint32_t i = lane; i < nnz; i += 32) sbuf[i] = Drow[i];
    __syncwarp();
  }
  const uint32_t* src = staged ? sbuf : Drow;
  uint32_t B = (nnz + 31u) >> 5;
  if (staged && B > 1 && !(B & 1u)) B += 1;  // odd stride: conflict-free shared-memory reads
  const uint32_t b0 = min(lane * B, nnz), b1 = min(b0 + B, nnz);
  double P = 0.0;
  uint32_t c1 = 0, c2 = 0, c3 = 0, li = 0;  // li = 1 + index of the lane's last entry != K1
  for (uint32_t i = b0; i < b1; ++i) {
    const uint32_t e = src[i];
    const uint32_t k = e >> 16, cnt = e & 0xFFFFu;
    P = P + (double)cnt * row[k];  // row[K1] = 0: What'
    c1 = (k == K1) ? cnt : c1;
    c2 = (k == K2) ? cnt : c2;
    c3 = (k == K3) ? cnt : c3;
    li = (k != K1) ? i + 1 : li;
  }
  const double incl = warp_incl_scan(P);
  double O = __shfl_up_sync(kFull, incl, 1);
  if (lane == 0) O = 0.0;
  const double T = O + P;
  warp_max_u32(c1);
  warp_max_u32(c2);
  warp_max_u32(c3);
  warp_max_u32(li);
  const uint32_t C1 = c1, C2 = c2, C3 = c3;
  const uint32_t lastk = li ? (src[li - 1] >> 16) : K1;
  const uint32_t l_last = nnz ? (nnz - 1) / B : 0;
  const double Sp = __shfl_sync(kFull, T, l_last);
  rc.runs += 1;
  rc.words += 2 + nnz;

  const double M = mpt_M(rec, C1, d.alpha);
  const double thr = mpt_threshold(rec, M, C1, C2, C3, L, d.geff);
  const double MS = M + Sp;
  const double Z = MS + rec.Qp;

  // first entry (k != K1) of the S' prefix list with prefix > y; none -> last such entry
  auto s_descent = [&](double y) -> uint32_t {
    uint32_t m = __ballot_sync(kFull, b0 < b1 && T > y);
    while (m) {
      const int l = __ffs(m) - 1;
      m &= m - 1;
      uint32_t res = 0xFFFFFFFFu;
      if ((int)lane == l) {
        double s = 0.0;
        for (uint32_t i = b0; i < b1; ++i) {
          const uint32_t e = src[i];
          const uint32_t k = e >> 16;
          s = s + (double)(e & 0xFFFFu) * row[k];
          if (k != K1 && O + s > y) {
            res = k;
            break;
          }
        }
      }
      res = __shfl_sync(kFull, res, l);
      if (res != 0xFFFFFFFFu) return res;
    }
    return lastk;
  };
  // first topic k != K1 (ascending) with alpha * P(k) > y; none -> last topic != K1
  auto q_descent = [&](double y) -> uint32_t {
    uint32_t lo = 0, hi = d.nch;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (d.alpha * CP[mid + 1] > y) hi = mid; else lo = mid + 1;
    }
    for (uint32_t c = lo; c < d.nch; ++c) {
      const uint32_t k = c * 32u + lane;
      const double val = CP[c] + warp_incl_scan(row[k]);
      const uint32_t m = __ballot_sync(kFull, k < d.K && k != K1 && d.alpha * val > y);
      if (m) return c * 32u + (uint32_t)(__ffs(m) - 1);
    }
    return (d.K - 1 != K1) ? d.K - 1 : d.K - 2;
  };

  for (uint32_t tb = 0; tb < len; tb += 32) {
    const uint32_t t = tb + lane;
    const uint32_t j = j0 + t;
    int br = 0;  // 0: skipped by the MPT test (or no token), 1: M, 2: S', 3: Q'
    double y = 0.0;
    if (t < len) {
      const double u = philox_u(d.seed, iter, d.token_base + j);
      if (!(u < thr)) {
        const double x = u * Z;
        if (x < M) {
          br = 1;
        } else if (x < MS) {
          br = 2;
          y = x - M;
        } else {
          br = 3;
          y = (x - M) - Sp;
        }
      }
    }
    uint32_t topic = K1;
    uint32_t ms = __ballot_sync(kFull, br == 2);
    while (ms) {
      const int l = __ffs(ms) - 1;
      ms &= ms - 1;
      const uint32_t tk = s_descent(__shfl_sync(kFull, y, l));
      if ((int)lane == l) topic = tk;
    }
    uint32_t mq = __ballot_sync(kFull, br == 3);
    while (mq) {
      const int l = __ffs(mq) - 1;
      mq &= mq - 1;
      const uint32_t tk = q_descent(__shfl_sync(kFull, y, l));
      if ((int)lane == l) topic = tk;
    }
    if (br != 0) {
      nxt.z[j] = (uint16_t)topic;
      atomicAdd(&hist[topic], 1u);
      rc.sampled += 1;
      rc.hitM += (br == 1);
    }
  }
  __syncwarp();  // sbuf is reused by the warp's next run
}

template <bool kCount>
__global__ void __launch_bounds__(kSampWarps * 32) k_sampler(Dev d, Buf cur, Buf nxt, uint32_t iter) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* row = reinterpret_cast<double*>(smem);
  double* T = row + d.Kpad;
  double* CP = T + d.nch;
  uint32_t* hist = reinterpret_cast<uint32_t*>(CP + d.nch + 1);
  __shared__ uint32_t s_cursor, s_wsum[32], s_run;
  __shared__ uint32_t s_sampled, s_hitM, s_runs, s_words;
  __shared__ uint32_t s_drow[kSampWarps][kDrowCap];
  const uint32_t tid = threadIdx.x, lane = tid & 31u;
  const uint32_t item = blockIdx.x;
  const uint32_t v = d.item_word[item], r0 = d.item_r0[item], r1 = d.item_r1[item];
  const uint32_t ntok = d.item_ntok[item];
  for (uint32_t k = tid; k < d.Kpad; k += blockDim.x) hist[k] = 0;
  if (tid == 0) { s_cursor = 0; s_sampled = 0; s_hitM = 0; s_runs = 0; s_words = 0; }
  WordRec rec;
  if (!kCount) {
    rec = d.rec[v];
    stage_row(d, cur, v, row);
    if (tid == 0) row[rec.K[0]] = 0.0;  // What'
    __syncthreads();
    chunk_prefix(row, d.nch, T, CP);
  } else {
    __syncthreads();
  }
  RunCounters rc{0, 0, 0, 0};
  while (true) {
    uint32_t grp = 0;
    if (lane == 0) grp = atomicAdd(&s_cursor, 1u);
    grp = __shfl_sync(kFull, grp, 0);
    const uint32_t rb = r0 + grp * 32u;
    if (rb >= r1) break;
    const uint32_t r = rb + lane;
    if (kCount) {
      if (r < r1) {
        const uint32_t j0 = d.run_j0[r], len = d.run_len[r];
        for (uint32_t t = 0; t < len; ++t) atomicAdd(&hist[cur.z[j0 + t]], 1u);
      }
      continue;
    }
    const bool active = (r < r1) && ((d.flags[r >> 5] >> (r & 31u)) & 1u);
    uint32_t am = __ballot_sync(kFull, active);
    while (am) {
      const int l = __ffs(am) - 1;
      am &= am - 1;
      sample_run(d, nxt, rec, row, CP, hist, s_drow[tid >> 5], rb + (uint32_t)l, iter, rc);
    }
  }
  // per-block counters
  {
    const uint32_t smp = warp_sum(rc.sampled), hm = warp_sum(rc.hitM);
    if (lane == 0 && !kCount) {
      atomicAdd(&s_sampled, smp);
      atomicAdd(&s_hitM, hm);
      atomicAdd(&s_runs, rc.runs);
      atomicAdd(&s_words, rc.words);
    }
  }
  __syncthreads();
  if (!kCount && tid == 0) hist[rec.K[0]] += ntok - s_sampled;  // skipped tokens stay at K1
  __syncthreads();
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
    const uint32_t nz = block_compact(hist, d.K, nxt.Wt + d.tofs[t], s_wsum, &s_run);
    if (tid == 0) nxt.tnnz[t] = nz;
    for (uint32_t k = tid; k < d.K; k += blockDim.x) {
      const uint32_t c = hist[k];
      if (c) atomicAdd(&nxt.nk[k], (int32_t)c);
    }
  }
  if (!kCount && tid == 0) {
    atomicAdd(&d.ctr->sampled, (unsigned long long)s_sampled);
    atomicAdd(&d.ctr->skip_M, (unsigned long long)s_hitM);
    atomicAdd(&d.ctr->active_runs, (unsigned long long)s_runs);
    atomicAdd(&d.ctr->drow_words, (unsigned long long)s_words);
  }
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
    const uint32_t* Drow = d.D + dbase + 2;
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
size_t sampler_smem_bytes(uint32_t K) {
  const uint32_t nch = (K + 31) / 32;
  return word_prep_smem_bytes(K) + (size_t)nch * 32 * 4;
}
size_t doc_block_smem_bytes(uint32_t K) { return (size_t)((K + 31) / 32) * 32 * 4; }

cudaError_t configure_kernels(uint32_t K) {
  cudaError_t e;
  const int wp = (int)word_prep_smem_bytes(K), sp = (int)sampler_smem_bytes(K), db = (int)doc_block_smem_bytes(K);
  if ((e = cudaFuncSetAttribute(k_word_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, wp))) return e;
  if ((e = cudaFuncSetAttribute(k_llpt, cudaFuncAttributeMaxDynamicSharedMemorySize, wp))) return e;
  if ((e = cudaFuncSetAttribute(k_sampler<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp))) return e;
  if ((e = cudaFuncSetAttribute(k_sampler<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp))) return e;
  if ((e = cudaFuncSetAttribute(k_doc_block<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, db))) return e;
  if ((e = cudaFuncSetAttribute(k_doc_block<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, db))) return e;
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
  if (n_w) {
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
    k_sampler<true><<<n_items, kSampWarps * 32, sampler_smem_bytes(d.K), s>>>(d, cur, nxt, iteration);
  else
    k_sampler<false><<<n_items, kSampWarps * 32, sampler_smem_bytes(d.K), s>>>(d, cur, nxt, iteration);
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
