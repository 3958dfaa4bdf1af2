// kernels.cu -- sm_100a kernels of the ezLDA three-branch Gibbs hot path.
//
// Per iteration i (snapshot semantics):
//   k_den        den_k = n_k + V beta, What of absent pairs beta / den_k        (Eq 1-2)
//   k_word_prep  per word: What row, top-4 (K1..K4, a1..a4), Q'                  (P:546 step 1)
//   k_doc_hist / k_doc_warp / k_doc_block
//                per doc: D row rebuilt from z^{i-1} (histogram + bitmap, or sort +
//                run-length encode), C_j lookups, MPT skip test; skipped tokens get
//                K1, failing tokens a marker carrying C1, their runs are flagged  (P:546 steps 2-3)
//   k_sampler    persistent, per work item (word, run range): stage the word's
//                fixed-point What' row in shared memory, for each flagged (doc, word)
//                run read the D row once, build S' (exact integers, warp scan), draw
//                every failing token of the run with the [M | S' | Q'] layout
//                (certified or redrawn exactly), then rebuild W and n_k from the
//                item's histogram (skipped tokens count at K1)                  (P:546 steps 4-6,
//                                                                                  P:822-846)
#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <vector>

#include "kernels.h"

namespace ezl {

namespace {

constexpr int kDocWarpCap = 512; // doc-pass warp tier: documents up to 512 tokens
#ifndef EZLDA_DOC_WARPS
#define EZLDA_DOC_WARPS 8
#endif
constexpr int kDocWarps = EZLDA_DOC_WARPS;
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

// Block-wide ordered compaction: out[pos] = (k << shift) | hist[k] for every k < K with
// hist[k] > 0, ascending k.  Returns nnz in all threads.
__device__ uint32_t block_compact(const uint32_t* hist, uint32_t K, uint32_t* out, uint32_t* s_wsum,
                                  uint32_t* s_run, uint32_t shift, uint32_t perm = 0u) {
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
    if (f) out[d_at(perm, pos)] = (k << shift) | c;
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
    d.inv_den[k] = 1.0 / den;  // sampler heads (stage_row_warp); the exact paths divide
  }
}

// chunk ends of the fixed-point Q' table: ce[c] = qfx[32 c + 31] (contiguous, so the first
// half of a Q' search probes one 128-byte line instead of one bank), padded to 16 bytes
__host__ __device__ __forceinline__ uint32_t ce_words(uint32_t Kpad) { return ((Kpad / 32u) + 3u) & ~3u; }
// H1: word-prep, small K (K <= 4096).  One warp per word: stage the What row
// in shared memory, top-4 (value desc, topic asc) by per-lane insertion + a 4-round warp
// tournament, What' (K1 entry zeroed), then lane 0 runs the Q' prefix P_v(k) strictly
// sequentially (the oracle's order: QP[k] = alpha P_v(k), Q' = alpha P_v(K-1) bit for bit)
// while the other warps of the SM proceed with their words.
constexpr uint32_t kWpWarps = 4;
constexpr uint32_t kWpSmallK = 4096;  // warp-per-word word-prep up to this K, thread-per-word above

__global__ void __launch_bounds__(kWpWarps * 32) k_word_prep_w(Dev d, Buf cur) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t v = blockIdx.x * (blockDim.x >> 5) + warp;
  if (v >= d.V || d.wtok[v + 1] == d.wtok[v]) return;  // no token of v in this shard (warp-uniform)
  double* row = reinterpret_cast<double*>(smem) + (size_t)warp * d.Kpad;
  if (v < d.Vd) {
    const int32_t* w = cur.Wd + (size_t)v * d.K;
    for (uint32_t k = lane; k < d.Kpad; k += 32u) row[k] = (k < d.K) ? ((double)w[k] + d.beta) / d.den[k] : 0.0;
  } else {
    for (uint32_t k = lane; k < d.Kpad; k += 32u) row[k] = (k < d.K) ? d.what0[k] : 0.0;
    __syncwarp();
    const uint32_t t = v - d.Vd;
    const uint32_t* tr = cur.Wt + d.tofs[t];
    const uint32_t n = cur.tnnz[t];
    for (uint32_t e = lane; e < n; e += 32u) {
      const uint32_t p = tr[e];
      const uint32_t k = p >> 16;
      row[k] = ((double)(p & 0xFFFFu) + d.beta) / d.den[k];
    }
  }
  __syncwarp();
  // top-4: per-lane sorted lists over k = lane (mod 32), then 4 rounds of warp argmax
  Top4 t;
  top4_init(t);
  for (uint32_t k = lane; k < d.K; k += 32u) top4_insert(t, row[k], k);
  WordRec r;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double bv = t.v[0];
    uint32_t bk = t.k[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(kFull, bv, o);
      const uint32_t ok = __shfl_xor_sync(kFull, bk, o);
      if (better(ov, ok, bv, bk)) { bv = ov; bk = ok; }
    }
    if (t.k[0] == bk) {  // the owner pops its head
      t.v[0] = t.v[1]; t.k[0] = t.k[1];
      t.v[1] = t.v[2]; t.k[1] = t.k[2];
      t.v[2] = t.v[3]; t.k[2] = t.k[3];
      t.v[3] = -1.0; t.k[3] = 0xFFFFFFFFu;
    }
    const bool ok = bv >= 0.0;
    r.a[i] = ok ? bv : 0.0;
    r.K[i] = ok ? (uint16_t)bk : (uint16_t)0;
  }
  __syncwarp();  // every lane's reads of the row (top-4 scan) precede lane 0's write below
  if (lane == 0) row[r.K[0]] = 0.0;  // What' (Eq 6): the maximum entry set to 0
  __syncwarp();
  if (lane == 0) {
    // Q' = alpha sum_{k != K1} What[v][k], strictly sequential (the oracle's order, bit for
    // bit); the next 8 entries are loaded before the dependent adds.  Every 32 topics the
    // running sum is kept (qe: exact checkpoints of P_v for the sampler's exact redraws)
    double* qe = d.qexact + (size_t)v * d.nch;
    double acc = 0.0, x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = row[i];
    for (uint32_t k0 = 0; k0 < d.Kpad; k0 += 8u) {  // Kpad is a multiple of 32 (zero past K)
      double xn[8];
      const uint32_t kn = (k0 + 8u < d.Kpad) ? k0 + 8u : k0;
#pragma unroll
      for (int i = 0; i < 8; ++i) xn[i] = row[kn + i];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc = acc + x[i];
      if ((k0 & 31u) == 24u) qe[k0 >> 5] = acc;  // exact P_v(32 c + 31), c = k0 / 32
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = xn[i];
    }
    r.Qp = d.alpha * acc;
    d.rec[v] = r;
    d.recm[v] = WordRecM{r.a[0], r.a[1], r.a[2], r.Qp};
    d.reck[v] = (uint32_t)r.K[0] | ((uint32_t)r.K[1] << 16);
  }
}

// ---------------------------------------------------------------------------------
// H1: word-prep, large K (K > 4096).  One warp per word, the What row in 256-topic chunks
// staged in shared memory (2 KB per warp, so occupancy does not fall with K).  Pass 1: every
// chunk filled with What[v][k] = (W[v][k] + beta) / den_k (dense rows; tail rows: the
// absent-pair value beta / den_k with the sorted nonzeros merged in), per-lane top-4 lists
// + a 4-round warp tournament (value desc, topic asc).  Pass 2: the chunks refilled, the K1
// entry zeroed (What', Eq 6), m written by all lanes, and lane 0 runs the Q' prefix P_v(k)
// strictly sequentially across the chunks -- the oracle's order, so QP[k] = alpha P_v(k) and
// Q' = alpha P_v(K-1) are its values bit for bit; qfx / ce are written from each finished
// chunk with the scale 2^t fixed in pass 1 from a (parallel) estimate of Q'.
constexpr uint32_t kWbWarps = 8;
constexpr uint32_t kWbChunk = 256;

// What[v][c0 .. c0 + kWbChunk) into ch (zero past K); tcur: warp-uniform cursor into the
// word's tail row (entries below c0 were consumed by earlier chunks)
__device__ __forceinline__ void fill_what_chunk(const Dev& d, const Buf& cur, uint32_t v, uint32_t c0, double* ch,
                                                uint32_t& tcur) {
  const uint32_t lane = threadIdx.x & 31u;
  if (v < d.Vd) {
    const int32_t* w = cur.Wd + (size_t)v * d.K;
    for (uint32_t i = lane; i < kWbChunk; i += 32u) {
      const uint32_t k = c0 + i;
      ch[i] = (k < d.K) ? ((double)w[k] + d.beta) / d.den[k] : 0.0;
    }
  } else {
    for (uint32_t i = lane; i < kWbChunk; i += 32u) {
      const uint32_t k = c0 + i;
      ch[i] = (k < d.K) ? __ldg(d.what0 + k) : 0.0;
    }
    __syncwarp();
    const uint32_t t = v - d.Vd;
    const uint32_t* tr = cur.Wt + d.tofs[t];
    const uint32_t n = cur.tnnz[t];
    while (tcur < n) {  // the row's entries with topic in [c0, c0 + kWbChunk) (sorted by topic)
      const uint32_t e = tcur + lane;
      const uint32_t p = (e < n) ? tr[e] : 0u;
      const uint32_t k = p >> 16;
      const bool in = e < n && k < c0 + kWbChunk;
      if (in) ch[k - c0] = ((double)(p & 0xFFFFu) + d.beta) / d.den[k];
      const uint32_t cnt = __popc(__ballot_sync(kFull, in));
      tcur += cnt;
      if (cnt < 32u) break;
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kWbWarps * 32) k_word_prep_big(Dev d, Buf cur) {
  __shared__ double s_ch[kWbWarps][kWbChunk];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t v = blockIdx.x * kWbWarps + warp;
  if (v >= d.Vd || d.wtok[v + 1] == d.wtok[v]) return;  // dense words only (tail: k_word_rec_tail)
  double* ch = s_ch[warp];
  // ---- pass 1: top-4 (value desc, topic asc) and an estimate of sum_k What
  Top4 t;
  top4_init(t);
  uint32_t tcur = 0;
  for (uint32_t c0 = 0; c0 < d.K; c0 += kWbChunk) {
    fill_what_chunk(d, cur, v, c0, ch, tcur);
    for (uint32_t i = lane; i < kWbChunk && c0 + i < d.K; i += 32u) top4_insert(t, ch[i], c0 + i);
    __syncwarp();
  }
  WordRec r;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double bv = t.v[0];
    uint32_t bk = t.k[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(kFull, bv, o);
      const uint32_t ok = __shfl_xor_sync(kFull, bk, o);
      if (better(ov, ok, bv, bk)) { bv = ov; bk = ok; }
    }
    if (t.k[0] == bk) {  // the owner pops its head
      t.v[0] = t.v[1]; t.k[0] = t.k[1];
      t.v[1] = t.v[2]; t.k[1] = t.k[2];
      t.v[2] = t.v[3]; t.k[2] = t.k[3];
      t.v[3] = -1.0; t.k[3] = 0xFFFFFFFFu;
    }
    const bool ok = bv >= 0.0;
    r.a[i] = ok ? bv : 0.0;
    r.K[i] = ok ? (uint16_t)bk : (uint16_t)0;
  }
  const uint32_t K1 = r.K[0];
  // ---- pass 2: lane 0's sequential Q' = alpha sum_{k != K1} What[v][k] (ascending k: the
  //      oracle's order, so Q' is its value bit for bit)
  double acc = 0.0;
  double* qe = d.qexact + (size_t)v * d.nch;
  tcur = 0;
  for (uint32_t c0 = 0; c0 < d.K; c0 += kWbChunk) {
    fill_what_chunk(d, cur, v, c0, ch, tcur);
    if (lane == 0 && K1 >= c0 && K1 < c0 + kWbChunk) ch[K1 - c0] = 0.0;  // What' (Eq 6)
    __syncwarp();
    const uint32_t n = min(kWbChunk, d.K - c0);
    if (lane == 0) {  // strictly sequential; 8 entries loaded ahead of the dependent adds
      double x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = ch[i];
      for (uint32_t i0 = 0; i0 < n; i0 += 8u) {
        double xn[8];
        const uint32_t in = (i0 + 8u < n) ? i0 + 8u : i0;
#pragma unroll
        for (int i = 0; i < 8; ++i) xn[i] = ch[in + i];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i0 + i < n) acc = acc + x[i];
        if ((i0 & 31u) == 24u || i0 + 8u >= n) qe[(c0 + i0) >> 5] = acc;  // exact P_v(32 c + 31)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = xn[i];
      }
    }
    __syncwarp();
  }
  r.Qp = d.alpha * acc;
  if (lane == 0) {
    d.rec[v] = r;
    d.recm[v] = WordRecM{r.a[0], r.a[1], r.a[2], r.Qp};
    d.reck[v] = (uint32_t)r.K[0] | ((uint32_t)r.K[1] << 16);
  }
}

// H1 records of the tail words at large K (K > 4096): one THREAD per word.
//   Top-4: the word's nonzeros (What = (W + beta) / den_k) and its four best ABSENT topics,
//     whose value What = beta / den_k (what0[k], the oracle's (0 + beta) / den_k) is the same
//     for every tail word: they are the first four topics of the iteration's global order of
//     what0 (value desc, topic asc: d.w0ord, sorted once per iteration) that are not in the
//     word's row.  Any later absent topic ranks below them, so the top-4 is exact.
//   Q': the oracle's sequential sum over k != K1 in ascending k, with a checkpoint every 32
//     topics: the 128 words of a block walk the topics in lockstep, what0 staged through
//     shared memory in chunks (one broadcast read per topic), the word's packed row merged
//     with a cursor (only its nonzeros take the division).
constexpr uint32_t kTailChunk = 2048;  // what0 doubles per shared-memory chunk
__device__ __forceinline__ bool row_has(const uint32_t* tr, uint32_t n, uint32_t k) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((tr[mid] >> 16) < k) lo = mid + 1u; else hi = mid;
  }
  return lo < n && (tr[lo] >> 16) == k;
}
__global__ void __launch_bounds__(128) k_word_rec_tail(Dev d, Buf cur) {
  __shared__ double s_w0[kTailChunk];
  const uint32_t Vt = d.V - d.Vd;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t v = d.Vd + t;
  const bool act = t < Vt && d.wtok[v + 1] != d.wtok[v];
  const uint32_t* tr = act ? cur.Wt + d.tofs[t] : nullptr;
  const uint32_t n = act ? cur.tnnz[t] : 0u;
  Top4 tp;
  top4_init(tp);
  WordRec r;
  double* tv = act ? d.twv + d.tofs[t] : nullptr;  // the nonzeros' What, for the lockstep pass
  if (act) {
    // 16 entries per step with their loads and den gathers issued together: the heaviest tail
    // words (thousands of nonzeros) set the kernel's time, and one dependent load pair per
    // entry left them latency-bound
    constexpr uint32_t kU = 16;
    for (uint32_t e0 = 0; e0 < n; e0 += kU) {
      uint32_t pp[kU];
      double dd[kU];
#pragma unroll
      for (uint32_t i = 0; i < kU; ++i) pp[i] = (e0 + i < n) ? __ldg(tr + e0 + i) : 0u;
#pragma unroll
      for (uint32_t i = 0; i < kU; ++i) dd[i] = (e0 + i < n) ? __ldg(d.den + (pp[i] >> 16)) : 1.0;
#pragma unroll
      for (uint32_t i = 0; i < kU; ++i) {
        if (e0 + i < n) {
          const double w = ((double)(pp[i] & 0xFFFFu) + d.beta) / dd[i];
          tv[e0 + i] = w;
          top4_insert(tp, w, pp[i] >> 16);
        }
      }
    }
    uint32_t found = 0;
    for (uint32_t i = 0; found < 4u && i < d.K; ++i) {
      const uint32_t k = __ldg(d.w0ord + i);
      if (!row_has(tr, n, k)) {
        top4_insert(tp, __ldg(d.what0 + k), k);
        ++found;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool ok = tp.v[i] >= 0.0;
    r.a[i] = ok ? tp.v[i] : 0.0;
    r.K[i] = ok ? (uint16_t)tp.k[i] : (uint16_t)0;
  }
  const uint32_t K1 = r.K[0];
  double* qe = d.qexact + (size_t)(act ? v : 0u) * d.nch;
  double acc = 0.0;
  // the nonzeros' values were computed above (independent divisions); the lockstep chain only
  // selects them, with the next nonzero's topic and value loaded one nonzero ahead (a division
  // inside the divergent branch sat on every word's dependent chain: K = 10k 6 -> <1 ms)
  uint32_t e = 0, nk = n ? (tr[0] >> 16) : 0xFFFFFFFFu;
  double nv = n ? tv[0] : 0.0;
  for (uint32_t c0 = 0; c0 < d.Kpad; c0 += kTailChunk) {  // (every thread of the block: barriers)
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kTailChunk; i += blockDim.x)
      s_w0[i] = (c0 + i < d.K) ? __ldg(d.what0 + c0 + i) : 0.0;
    __syncthreads();
    const uint32_t cend = min(c0 + kTailChunk, d.Kpad);
    for (uint32_t k = c0; k < cend; ++k) {
      double w = s_w0[k - c0];
      if (k == nk) {
        w = nv;
        ++e;
        nk = (e < n) ? (tr[e] >> 16) : 0xFFFFFFFFu;
        nv = (e < n) ? tv[e] : 0.0;
      }
      if (k == K1) w = 0.0;  // What' (Eq 6): adds +0, as the oracle skips K1
      acc = acc + w;
      if (act && (k & 31u) == 31u) qe[k >> 5] = acc;  // exact P_v(32 c + 31)
    }
  }
  r.Qp = d.alpha * acc;
  if (act) {
    d.rec[v] = r;
    d.recm[v] = WordRecM{r.a[0], r.a[1], r.a[2], r.Qp};
    d.reck[v] = (uint32_t)r.K[0] | ((uint32_t)r.K[1] << 16);
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

// MPT test of one token j (word v) of a doc of length L.  C(k) = D[d][k].  Writes z^i (K1, or
// the sampler's marker) and returns true if the token failed the test (its run must be flagged).
template <typename LookupF>
__device__ __forceinline__ bool mpt_token(const Dev& d, const Buf& nxt, uint32_t j, uint32_t L, uint32_t iter,
                                          uint32_t v, LookupF C, unsigned long long& n_skip, bool g2,
                                          uint32_t kk_pre = 0xFFFFFFFFu) {
  WordRec r;
  if (g2) {  // g <= 2 (a warp-uniform kernel argument): compact view, one 32-byte load + one 4-byte load
    const WordRecM m = d.recm[v];
    // K1 | K2 << 16, loaded ahead by the caller when it can (the counter lookups wait on it)
    const uint32_t kk = (kk_pre != 0xFFFFFFFFu) ? kk_pre : __ldg(d.reck + v);
    r.a[0] = m.a0;
    r.a[1] = m.a1;
    r.a[2] = m.a2;
    r.a[3] = 0.0;
    r.Qp = m.Qp;
    r.K[0] = (uint16_t)(kk & 0xFFFFu);
    r.K[1] = (uint16_t)(kk >> 16);
    r.K[2] = r.K[3] = 0;
  } else {
    r = d.rec[v];
  }
  const uint32_t C1 = C(r.K[0]);
  const uint32_t C2 = d.geff >= 2 ? C(r.K[1]) : 0u;
  const uint32_t C3 = d.geff >= 3 ? C(r.K[2]) : 0u;
  const double M = mpt_M(r, C1, d.alpha);
  const double den = mpt_den(r, M, C1, C2, C3, L, d.geff);
#ifdef EZLDA_EXP_DOC_NOPHILOX  // diagnostic: a cheap hash instead of Philox in the doc pass
  const double u = (double)((j * 2654435761u) >> 8) * 0x1p-24;
#else
  const double u = philox_u_k(d.pk, iter, d.token_base + j);
#endif
  if (mpt_skip(u, M, den)) {
    nxt.z[j] = r.K[0];
    ++n_skip;
    return false;
  }
  // the sampler draws it; the marker carries C1 when K <= 32768 (see sample_batch)
  nxt.z[j] = d.zmark ? (uint16_t)(0x8000u | min(C1, d.c1_cap)) : kUnsampled;
  return true;
}

// Flag run rid of a token that failed the MPT test (word-major run bitset, L2 resident).  The
// lanes hold consecutive tokens of the doc: a token whose left neighbour is in the same run and
// was flagged too leaves the atomic to it.
__device__ __forceinline__ void flag_run(const Dev& d, bool flagged, uint32_t rid) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t prid = __shfl_up_sync(kFull, rid, 1);
  const bool pflag = __shfl_up_sync(kFull, flagged ? 1u : 0u, 1) != 0u;
  if (flagged && !(lane > 0 && pflag && prid == rid)) atomicOr(&d.flags[rid >> 5], 1u << (rid & 31u));
}

// Per-token MPT test of one doc's tokens (shared by both doc tiers).  C(k) = D[d][k].
template <typename LookupF>
__device__ __forceinline__ void doc_tokens_skip_test(const Dev& d, const Buf& nxt, uint32_t j0, uint32_t L,
                                                     uint32_t iter, uint32_t start, uint32_t stride,
                                                     LookupF C, unsigned long long& n_skip) {
  for (uint32_t i = start; i < L; i += stride) {
    const uint32_t j = j0 + i;
    const uint32_t v = d.twr[j].x;
    const WordRec r = d.rec[v];
    const uint32_t C1 = C(r.K[0]);
    const uint32_t C2 = d.geff >= 2 ? C(r.K[1]) : 0u;
    const uint32_t C3 = d.geff >= 3 ? C(r.K[2]) : 0u;
    const double M = mpt_M(r, C1, d.alpha);
    const double den = mpt_den(r, M, C1, C2, C3, L, d.geff);
    const double u = philox_u_k(d.pk, iter, d.token_base + j);
    if (mpt_skip(u, M, den)) {
      nxt.z[j] = r.K[0];
      ++n_skip;
    } else {
      // the sampler draws it; the marker carries C1 when K <= 32768 (see sample_batch)
      nxt.z[j] = d.zmark ? (uint16_t)(0x8000u | min(C1, d.c1_cap)) : kUnsampled;
      const uint32_t rid = d.twr[j].y;
      atomicOr(&d.flags[rid >> 5], 1u << (rid & 31u));
    }
  }
}

// Warp tier, K <= 4096: one warp per doc with a private dense shared-memory histogram
// (two 16-bit counters per word) and a topic bitmap, C_j read straight from the
// histogram; the packed D row is emitted in topic order from the bitmap (each lane owns
// 32-topic words: popcount prefix + set-bit walk, O(nnz + K/32) per doc) and both are
// re-zeroed as they are read.
// per-warp shared words of k_doc_hist: Kpad / 2 counter words + Kpad / 32 bitmap words, padded
// to 16 bytes (the counters are re-zeroed with 16-byte stores)
__host__ __device__ __forceinline__ uint32_t doc_hist_stride(uint32_t Kpad) {
  return (Kpad / 2u + Kpad / 32u + 3u) & ~3u;
}
template <bool kSkipTest, bool kG2 = true>  // kG2: S_est depth g <= 2 (the compact record view)
#ifndef EZLDA_DOC_PF
#define EZLDA_DOC_PF 1
#endif
#ifndef EZLDA_DOC_KKPF
#define EZLDA_DOC_KKPF 0  // A/B: 10.22 -> 10.38 ms at PubMed (profiles/r02/ab_dperm.log), off
#endif
#ifndef EZLDA_DOC_MINB
#define EZLDA_DOC_MINB 4
#endif
__global__ void __launch_bounds__(kDocWarps * 32, EZLDA_DOC_MINB) k_doc_hist(Dev d, Buf cur, Buf nxt, const uint32_t* docs,
                                                              uint32_t n_docs, uint32_t iter) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t hw = d.Kpad >> 1;   // counter words per warp
  const uint32_t bw = d.Kpad >> 5;   // bitmap words per warp
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem) + warp * doc_hist_stride(d.Kpad);
  uint32_t* bmp = hist + hw;
  for (uint32_t i = lane; i < hw + bw; i += 32) hist[i] = 0;
  __syncwarp();
  unsigned long long n_skip = 0, n_nnz = 0;
#if EZLDA_DOC_PF
  // the next doc's id, token range and D-row base are loaded one doc ahead (the chain
  // docs -> dofs -> tokens otherwise starts every doc with two dependent global loads)
  const uint32_t stride = gridDim.x * kDocWarps;
  uint32_t idx = blockIdx.x * kDocWarps + warp;
  uint32_t n_doc = 0, n_j0 = 0, n_j1 = 0, n_db = 0;
  if (idx < n_docs) {
    n_doc = docs[idx];
    n_j0 = d.dofs[n_doc];
    n_j1 = d.dofs[n_doc + 1];
    n_db = d.ddb[n_doc];
  }
  for (; idx < n_docs; idx += stride) {
    const uint32_t doc = n_doc, j0 = n_j0, L = n_j1 - n_j0, dbase = n_db;
    (void)doc;
    if (idx + stride < n_docs) {
      n_doc = docs[idx + stride];
      n_j0 = d.dofs[n_doc];
      n_j1 = d.dofs[n_doc + 1];
      n_db = d.ddb[n_doc];
    }
#else
  for (uint32_t idx = blockIdx.x * kDocWarps + warp; idx < n_docs; idx += gridDim.x * kDocWarps) {
    const uint32_t doc = docs[idx];
    const uint32_t j0 = d.dofs[doc];
    const uint32_t L = d.dofs[doc + 1] - j0;
    const uint32_t dbase = d.ddb[doc];
#endif
    // the first kPre tokens of each lane: topic, word and run id loaded together (the
    // skip test's word records then depend on one load round instead of two)
    constexpr uint32_t kPre = 4;
    uint32_t pk[kPre], pv[kPre], pr[kPre];
#pragma unroll
    for (uint32_t c = 0; c < kPre; ++c) {
      const uint32_t i = lane + 32u * c;
      pk[c] = (i < L) ? cur.z[j0 + i] : 0u;
      const uint2 wr = (kSkipTest && i < L) ? d.twr[j0 + i] : make_uint2(0u, 0u);  // one 8-byte load
      pv[c] = wr.x;
      pr[c] = wr.y;
    }
#if EZLDA_DOC_KKPF
    // the first rounds' K1 | K2 words requested before the histogram is built, so that their
    // latency overlaps the shared-memory atomics instead of stalling the counter lookups
    uint32_t pkk[kPre];
#pragma unroll
    for (uint32_t c = 0; c < kPre; ++c)
      pkk[c] = (kSkipTest && kG2 && lane + 32u * c < L) ? __ldg(d.reck + pv[c]) : 0xFFFFFFFFu;
#endif
#pragma unroll
    for (uint32_t c = 0; c < kPre; ++c) {
      if (lane + 32u * c < L) {
        const uint32_t k = pk[c];
        atomicAdd(&hist[k >> 1], 1u << ((k & 1u) << 4));
        atomicOr(&bmp[k >> 5], 1u << (k & 31u));
      }
    }
    for (uint32_t i = lane + 32u * kPre; i < L; i += 32) {
      const uint32_t k = cur.z[j0 + i];
      atomicAdd(&hist[k >> 1], 1u << ((k & 1u) << 4));
      atomicOr(&bmp[k >> 5], 1u << (k & 31u));
    }
    __syncwarp();
    if (kSkipTest) {
      auto C = [&](uint32_t k) { return (hist[k >> 1] >> ((k & 1u) << 4)) & 0xFFFFu; };
#pragma unroll
      for (uint32_t c = 0; c < kPre; ++c) {
        if (32u * c >= L) break;  // warp-uniform
        bool f = false;
#if EZLDA_DOC_KKPF
        if (lane + 32u * c < L) f = mpt_token(d, nxt, j0 + lane + 32u * c, L, iter, pv[c], C, n_skip, kG2, pkk[c]);
#else
        if (lane + 32u * c < L) f = mpt_token(d, nxt, j0 + lane + 32u * c, L, iter, pv[c], C, n_skip, kG2);
#endif
#ifndef EZLDA_EXP_DOC_NOFLAG  // diagnostic: no flag atomics (the sampler then sees no flagged run)
        flag_run(d, f, pr[c]);
#endif
      }
      for (uint32_t i0 = 32u * kPre; i0 < L; i0 += 32u) {  // warp-uniform rounds
        const uint32_t i = i0 + lane;
        bool f = false;
        uint32_t rid = 0;
        if (i < L) {
          const uint2 wr = d.twr[j0 + i];
          rid = wr.y;
          f = mpt_token(d, nxt, j0 + i, L, iter, wr.x, C, n_skip, kG2);
        }
        flag_run(d, f, rid);
      }
      __syncwarp();
    }
    uint32_t* Drow = d.D + dbase + kDHdr;
    uint32_t nnz = 0;
#ifdef EZLDA_EXP_DOC_NOWALK  // diagnostic: no D-row emission (counters re-zeroed wholesale)
    for (uint32_t i = lane; i < hw + bw; i += 32) hist[i] = 0;
    if (false)
#endif
    for (uint32_t base = 0; base < bw; base += 32) {
      const uint32_t wi = base + lane;
      const uint32_t b = (wi < bw) ? bmp[wi] : 0u;
      const uint32_t cnt = __popc(b);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      uint32_t pos = nnz + incl - cnt;
      for (uint32_t m = b; m; m &= m - 1u) {
        const uint32_t k = wi * 32u + (__ffs(m) - 1u);
        Drow[d_at(d.dperm, pos++)] = d_entry(k, (hist[k >> 1] >> ((k & 1u) << 4)) & 0xFFFFu, d.dt);
      }
      if (b) bmp[wi] = 0u;
      nnz += __shfl_sync(kFull, incl, 31);
    }
    if (nnz + lane < ((nnz + 7u) & ~7u)) Drow[d_at(d.dperm, nnz + lane)] = 0u;  // pad to 8 (< 8 entries)
    if (lane == 0) {
      Drow[-(int)kDHdr] = (L << 16) | nnz;
      Drow[1 - (int)kDHdr] = j0;
    }
    __syncwarp();  // every lane's counter reads above precede the wholesale re-zeroing
    // re-zero the counters with 16-byte stores (cheaper than a second set-bit walk)
    for (uint32_t i = 4u * lane; i < hw; i += 128u) *reinterpret_cast<uint4*>(hist + i) = make_uint4(0u, 0u, 0u, 0u);
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
    Drow[kDHdr + p] = d_entry(ukey[p], cnt, d.dt);
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
  const uint32_t nnz = block_compact(hist, d.K, Drow + kDHdr, s_wsum, &s_run, d.dt, d.dperm);
  for (uint32_t p = nnz + tid; p < ((nnz + 7u) & ~7u); p += nt) Drow[kDHdr + d_at(d.dperm, p)] = 0u;  // pad to 8
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
// H5+H6: the residual three-branch sampler + W/n_k rebuild.
// ---------------------------------------------------------------------------------
//
// Work item = (word v, a range of its (doc, word) runs).  The item's fixed-point What' row
// m_v (Eq 6, K1 entry 0), the fixed-point Q' prefix table and their scales are staged in a
// shared-memory slot with ONE TMA bulk copy (cp.async.bulk + mbarrier) of the word's wrow
// head (tail rows word-prep did not precompute are staged by a warp).  Persistent blocks
// own 2-3 slots and pipeline items through them (k_sampler below).  Warps take groups of
// 32 runs from the item's cursor, queue the flagged ones (a token of the run failed the doc
// pass's MPT test) and process them in batches (P:546 steps 4-6):
//
//  A (lane per run)      run table + D-row header; the row is cut into segments of kSegW
//                        entries (16 = two 32-byte sectors); a batch admits runs while
//                        the segment total fits the checkpoint array;
//  B (lane per segment)  consecutive lanes read consecutive sectors of a row (coalesced)
//                        and accumulate the exact integer products D[d][k] m_v[k]
//                        (IMAD.WIDE); a segmented warp scan (+ carry across rounds) turns
//                        segment sums into run prefixes, stored as checkpoints (two per
//                        16-entry segment); S' = the run's last checkpoint;
//  D (lane per token)    C1 from the doc pass's z marker, M (Eq 8), Philox u, Z = (M + S')
//                        + Q', x = u Z in [M | S' | Q']; S' descent: binary search over the
//                        checkpoints, then a walk of one sector from registers; Q' descent:
//                        binary search over the fixed-point prefix table.  Each decision
//                        is certified against the fixed-point error bound or the token is
//                        redrawn by exact_draw with the oracle's fp64 operations, so the
//                        topics equal the oracle's.
#ifdef EZLDA_EXP_FAKEROW
__device__ uint32_t g_fake[1024 + 16];  // (topic << 18) | 1, topics spread over [0, 1000)
#endif
#ifndef EZLDA_SCAN_DYN
#define EZLDA_SCAN_DYN 1
#endif
#ifndef EZLDA_B_PF
#define EZLDA_B_PF 1
#endif
#ifndef EZLDA_QSWZ
#define EZLDA_QSWZ 1
#endif
// The fixed-point Q' table is stored XOR-swizzled within each 32-topic chunk (topic i at
// i ^ (chunk & 31)): the lanes of a warp search different chunks in step, so an unswizzled
// table sends them all to the same bank (e.g. every lane's first probe is entry 15 of its chunk)
__device__ __forceinline__ uint32_t q_swz(uint32_t i) { return EZLDA_QSWZ ? (i ^ ((i >> 5) & 31u)) : i; }
#ifndef EZLDA_ZPRE2
#define EZLDA_ZPRE2 0  // A/B: 72.7-73.0 -> 73.4-73.6 ms at PubMed (spills), off
#endif
#ifndef EZLDA_QG_VEC
#define EZLDA_QG_VEC 0  // A/B at K = 10k: 42.91 -> 43.02 ms (profiles/r02/ab_dperm.log), off
#endif
#ifndef EZLDA_LARGEK_1BLK
#define EZLDA_LARGEK_1BLK 0  // A/B: 1 block x 3-4 slots at K = 10k 42.5 -> 57-59 ms (profiles/r02/ab_dperm.log)
#endif
#ifndef EZLDA_SPIN_MAX
#define EZLDA_SPIN_MAX 256  // longest nanosleep (ns) of the sampler's slot wait
#endif
#ifndef EZLDA_RED_SHARED
#define EZLDA_RED_SHARED 1
#endif
#ifndef EZLDA_HDR_PF
#define EZLDA_HDR_PF 0
#endif
#ifndef EZLDA_WALK2
#define EZLDA_WALK2 1
#endif
#ifndef EZLDA_SEGW_SMALL
#define EZLDA_SEGW_SMALL 16u  // S' segment width when K <= kSegCap x 16 (16 or 32 entries per lane and round)
#endif
struct RunCounters {
  uint32_t sampled, hitM, runs, words, exact;
};

constexpr int kQueue = 64;  // one batch + one refill group

struct WarpScratch {  // per-warp shared memory (d.ws_bytes): checkpoints | queue (32-bit shared addresses)
  uint32_t P;     // u64 fixed-point prefix checkpoints of the batch's runs (see sample_batch)
  uint32_t q;     // ring of kQueue flagged runs
  uint32_t head;  // ring position of the queue's first entry
};
__device__ __forceinline__ unsigned long long lds_u64(uint32_t addr) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_u64x2(uint32_t addr, unsigned long long a, unsigned long long b) {
  asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(addr), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void sts_u64(uint32_t addr, unsigned long long a) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(addr), "l"(a) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32v(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t a) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(a) : "memory");
}
__device__ __forceinline__ uint32_t ws_q_at(const WarpScratch& ws, uint32_t i) {
  return ws.q + 4u * ((ws.head + i) & (uint32_t)(kQueue - 1));
}

// 32-byte (one sector) read-only load
__device__ __forceinline__ void ldg256(const uint32_t* p, uint4& a, uint4& b) {
  asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// acc + D[d][k] m_v[k] for one packed entry (topic << 18 | count): m_v is the word's
// fixed-point What' row (What' ~ m 2^-s), the product and the sum are exact 64-bit integers
// (IMAD.WIDE.U32); padding (0) adds 0.
template <uint32_t kDTs>
__device__ __forceinline__ unsigned long long entry_mac(uint32_t w, uint32_t row_s, unsigned long long acc) {
  // dt = 18: w >> 16 = 4 topic (one LEA.HI); dt = 16: 4 topic = (w >> 14) & ~3
  const uint32_t off = (kDTs == 18u) ? (w >> 16) : ((w >> 14) & ~3u);
#ifdef EZLDA_EXP_NOCONFLICT  // diagnostic: every lane gathers one address (no bank conflicts)
  return acc + (unsigned long long)(w & 0xFFFFu) * lds_u32(row_s + (off & 4u));
#endif
  return acc + (unsigned long long)(w & 0xFFFFu) * lds_u32(row_s + off);
}

#ifndef EZLDA_MAC2
#define EZLDA_MAC2 0
#endif
template <uint32_t kDTs>
__device__ __forceinline__ unsigned long long sector_mac(unsigned long long acc, const uint4& a, const uint4& b,
                                                         uint32_t row_s) {
#if EZLDA_MAC2  // two independent IMAD.WIDE chains (half the dependent latency per sector)
  unsigned long long t = entry_mac<kDTs>(a.y, row_s, 0ull);
  acc = entry_mac<kDTs>(a.x, row_s, acc);
  t = entry_mac<kDTs>(a.w, row_s, t);
  acc = entry_mac<kDTs>(a.z, row_s, acc);
  t = entry_mac<kDTs>(b.y, row_s, t);
  acc = entry_mac<kDTs>(b.x, row_s, acc);
  t = entry_mac<kDTs>(b.w, row_s, t);
  acc = entry_mac<kDTs>(b.z, row_s, acc);
  return acc + t;
#endif
  acc = entry_mac<kDTs>(a.x, row_s, acc);
  acc = entry_mac<kDTs>(a.y, row_s, acc);
  acc = entry_mac<kDTs>(a.z, row_s, acc);
  acc = entry_mac<kDTs>(a.w, row_s, acc);
  acc = entry_mac<kDTs>(b.x, row_s, acc);
  acc = entry_mac<kDTs>(b.y, row_s, acc);
  acc = entry_mac<kDTs>(b.z, row_s, acc);
  acc = entry_mac<kDTs>(b.w, row_s, acc);
  return acc;
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst_s, const void* src, uint32_t bytes, uint32_t mbar_s) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar_s), "r"(bytes) : "memory");
  const uint64_t g = (uint64_t)__cvta_generic_to_global(src);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_s),
               "l"(g), "r"(bytes), "r"(mbar_s)
               : "memory");
}

// bulk copy completing on an mbarrier whose expect_tx was already posted
__device__ __forceinline__ void bulk_copy_tx(uint32_t dst_s, const void* src, uint32_t bytes, uint32_t mbar_s) {
  const uint64_t g = (uint64_t)__cvta_generic_to_global(src);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_s),
               "l"(g), "r"(bytes), "r"(mbar_s)
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
__device__ __forceinline__ uint32_t packed_count(const uint32_t* E, uint32_t nnz, uint32_t k, uint32_t shift) {
  uint32_t lo = 0, hi = nnz;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((__ldg(E + mid) >> shift) < k) lo = mid + 1u; else hi = mid;
  }
  if (lo < nnz) {
    const uint32_t w = __ldg(E + lo);
    if ((w >> shift) == k) return w & 0xFFFFu;
  }
  return 0u;
}
// D[d][k] of a packed D row (logical index -> address by d_at) / W[v][k] of a packed tail row
__device__ __forceinline__ uint32_t row_count(const Dev& d, const uint32_t* E, uint32_t nnz, uint32_t k) {
  uint32_t lo = 0, hi = nnz;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((__ldg(E + d_at(d.dperm, mid)) >> d.dt) < k) lo = mid + 1u; else hi = mid;
  }
  if (lo < nnz) {
    const uint32_t w = __ldg(E + d_at(d.dperm, lo));
    if ((w >> d.dt) == k) return w & 0xFFFFu;
  }
  return 0u;
}
__device__ __forceinline__ uint32_t tail_count(const uint32_t* E, uint32_t nnz, uint32_t k) {
  return packed_count(E, nnz, k, 16u);
}

// The oracle's per-token draw in fp64 with its summation orders:
// S' = ascending sequential sum over the row's topics != K1 of D[d][k] What[v][k], Z = (M +
// S') + Q', x = u Z, [M | S' | Q'] descents.  Used for the (rare) tokens whose fast
// path could not certify its decision.
// W[v][k] for the ascending topics of a walk over a D row: dense rows by index, tail rows by a
// cursor merged along the sorted packed row (one pass instead of a binary search per entry)
struct WCursor {
  const int32_t* wr;
  const uint32_t* tr;
  uint32_t tn, te;
  __device__ __forceinline__ uint32_t at(uint32_t k) {
    if (wr) return (uint32_t)wr[k];
    while (te < tn && (tr[te] >> 16) < k) ++te;
    return (te < tn && (tr[te] >> 16) == k) ? (tr[te] & 0xFFFFu) : 0u;
  }
};
__device__ __forceinline__ WCursor wcursor(const Dev& d, const Buf& cur, uint32_t v) {
  WCursor c;
  if (v < d.Vd) {
    c.wr = cur.Wd + (size_t)v * d.K;
    c.tr = nullptr;
    c.tn = 0;
  } else {
    c.wr = nullptr;
    c.tr = cur.Wt + d.tofs[v - d.Vd];
    c.tn = cur.tnnz[v - d.Vd];
  }
  c.te = 0;
  return c;
}

// What[v][k] in fp64 exactly as word-prep / the oracle form it: (W[v][k] + beta) / den_k.
__device__ __forceinline__ double what_exact(const Dev& d, const Buf& cur, uint32_t v, uint32_t k) {
  uint32_t c;
  if (v < d.Vd) {
    c = (uint32_t)cur.Wd[(size_t)v * d.K + k];
  } else {
    const uint32_t t = v - d.Vd;
    c = tail_count(cur.Wt + d.tofs[t], cur.tnnz[t], k);
  }
  return ((double)c + d.beta) / d.den[k];
}

// kMerge (large K, where tail words carry a large share of the exact redraws): W[v][k] along the
// D row by a cursor merged with the packed tail row; else a binary search per entry (fewer live
// registers in the sampler's token loop)
template <bool kMerge>
__device__ uint32_t exact_draw(const Dev& d, const Buf& cur, uint32_t v, const WordRec& rec, const uint32_t* E,
                               uint32_t nnz, double M, double u, bool& hitM) {
  const uint32_t K1 = rec.K[0];
  double Sp = 0.0;
  {
    WCursor wc = wcursor(d, cur, v);
    for (uint32_t e = 0; e < nnz; ++e) {
      const uint32_t w = __ldg(E + d_at(d.dperm, e));
      const uint32_t k = d_topic(w, d.dt);
      if (kMerge) {
        const uint32_t c = wc.at(k);
        if (k != K1) Sp = Sp + (double)(w & 0xFFFFu) * (((double)c + d.beta) / d.den[k]);
      } else if (k != K1) {
        Sp = Sp + (double)(w & 0xFFFFu) * what_exact(d, cur, v, k);
      }
    }
  }
  const double Z = (M + Sp) + rec.Qp;
  const double x = u * Z;
  hitM = false;
  if (x < M) {
    hitM = true;
    return K1;
  }
  if (x < M + Sp) {
    const double y = x - M;
    double acc = 0.0;
    uint32_t last = K1;
    WCursor wc = wcursor(d, cur, v);
    for (uint32_t e = 0; e < nnz; ++e) {
      const uint32_t w = __ldg(E + d_at(d.dperm, e));
      const uint32_t k = d_topic(w, d.dt);
      const uint32_t c = kMerge ? wc.at(k) : 0u;
      if (k == K1) continue;
      acc = acc + (double)(w & 0xFFFFu) * (kMerge ? (((double)c + d.beta) / d.den[k]) : what_exact(d, cur, v, k));
      last = k;
      if (acc > y) return k;
    }
    return last;
  }
  // Q': the first k != K1 (ascending) with alpha P_v(k) > y, P_v the oracle's running sum of
  // What over j <= k, j != K1; past the end -> last k != K1.  The word-prep kept the exact
  // running sum at every 32nd topic (qe[c] = P_v(32 c + 31)): the first chunk whose end
  // passes y is found by binary search, then the oracle's additions are replayed from the
  // previous checkpoint through that chunk (same operands, same order: bit-identical)
  const double y = (x - M) - Sp;
  const double* qe = d.qexact + (size_t)v * d.nch;
  uint32_t ca = 0, cb = d.nch;
  while (ca < cb) {
    const uint32_t mid = (ca + cb) >> 1;
    if (d.alpha * qe[mid] > y) cb = mid; else ca = mid + 1u;
  }
  if (ca >= d.nch) return (d.K - 1 != K1) ? d.K - 1 : d.K - 2;
  const bool dense = v < d.Vd;
  const int32_t* wr = cur.Wd + (size_t)v * d.K;
  const uint32_t* tr = dense ? nullptr : cur.Wt + d.tofs[v - d.Vd];
  const uint32_t tn = dense ? 0u : cur.tnnz[v - d.Vd];
  const uint32_t k0 = 32u * ca;
  uint32_t te = 0;
  if (!dense) {  // first tail entry with topic >= k0
    uint32_t lo = 0, hi = tn;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if ((tr[mid] >> 16) < k0) lo = mid + 1u; else hi = mid;
    }
    te = lo;
  }
  double acc = ca ? qe[ca - 1u] : 0.0;
  for (uint32_t k = k0; k < d.K; ++k) {
    uint32_t c;
    if (dense) {
      c = (uint32_t)wr[k];
    } else {
      while (te < tn && (tr[te] >> 16) < k) ++te;
      c = (te < tn && (tr[te] >> 16) == k) ? (tr[te] & 0xFFFFu) : 0u;
    }
    if (k == K1) continue;
    acc = acc + ((double)c + d.beta) / d.den[k];
    if (d.alpha * acc > y) return k;
  }
  return (d.K - 1 != K1) ? d.K - 1 : d.K - 2;
}

// One batch of flagged runs (warp-uniform control flow).  Returns the number of queue
// entries consumed.  kSegW: entries per segment (8, or a power of two >= 16); the per-run
// state lives in the registers of the run's lane and is fetched by shuffles.
//
// Precision: the S' sums are exact 64-bit integer sums of counts times the word's
// fixed-point What' row (m = rint(What' 2^s), |m 2^-s - What'| <= 2^-s).  Every decision
// of the fast path (x vs M, x vs M + S', the S' and Q' descents) is taken only if it holds
// with a margin bounding that error (2 L_d 2^-s + 4e-15 Z); otherwise the token is redrawn
// by exact_draw.  Either way the topic equals the oracle's fp64 decision.
template <uint32_t kSegW, uint32_t kSub, uint32_t kDTs, bool kQG>
__device__ __forceinline__ uint32_t sample_batch(const Dev& d, const Buf& cur, const Buf& nxt, const WordRec& rec,
                                                 uint32_t v, uint32_t row_s, const uint32_t* qfx, const uint32_t* ce,
                                                 const double* scl,
                                                 uint32_t* hist, WarpScratch& ws,
                                                 uint32_t qn, uint32_t iter, RunCounters& rc) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t K1 = rec.K[0];
  // ---- A: lane per run: run table + header, segment admission
  const uint32_t nc = min(qn, 32u);
  uint32_t j0 = 0, ebase = 0, len = 0, nnz = 0, nseg = 0, Ld = 0;
  if (lane < nc) {
    const uint32_t r = lds_u32v(ws_q_at(ws, lane));
    j0 = d.run_j0[r];
    const uint32_t dbase = d.run_dbase[r];
    len = d.run_len[r];
    const uint32_t hdr = d.D[dbase];
    nnz = hdr & 0xFFFFu;
    Ld = hdr >> 16;
    ebase = dbase + kDHdr;
    nseg = (nnz + kSegW - 1u) / kSegW;
  }
  uint32_t sincl = nseg, tincl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, sincl, o);
    if (lane >= (uint32_t)o) sincl += y;
  }
  // checkpoints per segment: one per kSub-entry chunk (kSub = 8: one per 32-byte sector, so a
  // descent walks one sector from registers; kSub = kSegW: one per segment)
  constexpr uint32_t kCk = kSegW / kSub;
  constexpr uint32_t kCap = (kSub == 8u ? 2u * kSegCap : kSegCap) / kCk;  // segments per batch
  const uint32_t nb = __popc(__ballot_sync(kFull, lane < nc && sincl <= kCap));
  if (nb == 0) return 0;  // the first run alone exceeds a batch: the caller takes its wide-segment path
#if EZLDA_HDR_PF
  // the D-row bases of the runs already queued for the next batch, loaded now; their header
  // lines are prefetched into L2 once phase B is done (the next phase A then hits L2)
  uint32_t pf_dbase = 0xFFFFFFFFu;
  if (nb + lane < qn) pf_dbase = __ldg(d.run_dbase + lds_u32v(ws_q_at(ws, nb + lane)));
#endif
  const uint32_t T = __shfl_sync(kFull, sincl, nb - 1u);
  const uint32_t soff = sincl - nseg;
#if EZLDA_SCAN_DYN
  // the segmented scan of phase B needs offsets below the longest admitted run (<= 32 lanes)
  const uint32_t smax = __reduce_max_sync(kFull, lane < nb ? nseg : 0u);
#else
  const uint32_t smax = 32u;
#endif
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
  // the z^i markers of D's first round are requested now, hidden behind phase B
  uint32_t zpre = 0;
  {
    const uint32_t slot = slot_of(0u, tofs);
    const uint32_t j = __shfl_sync(kFull, j0, slot) + (lane - __shfl_sync(kFull, tofs, slot));
    if (lane < ntb) zpre = nxt.z[j];
  }
#if EZLDA_ZPRE2
  // ... and those of the second round (a batch of ~32 short runs holds 33-64 tokens)
  uint32_t zpre2 = 0;
  if (ntb > 32u) {
    const uint32_t slot = slot_of(32u, tofs);
    const uint32_t j = __shfl_sync(kFull, j0, slot) + (32u + lane - __shfl_sync(kFull, tofs, slot));
    if (32u + lane < ntb) zpre2 = nxt.z[j];
  }
#endif
  // ---- B: lane per segment (kSegW entries = kSegW / 8 sectors); consecutive lanes read
  //      consecutive sectors of a row.  Exact integer sums of D[d][k] m_v[k] (m_v the word's
  //      fixed-point What' row), combined by a segmented warp scan (+ carry across rounds).
  //      Checkpoints: P[kCk g + i] = P(before g) + (chunks 0..i of g); the last one is
  //      P(end of g), and S' = the run's last checkpoint.
  static_assert(kCk == 1u || kCk == 2u || kCk == 4u, "checkpoints per segment");
  unsigned long long carry = 0ull;
#if EZLDA_B_PF
  // software pipeline (kSegW == 16): the two sectors of round B0 + 32 are requested before
  // round B0 is accumulated, so a warp keeps two rounds of D-row loads in flight
  constexpr bool kPf = (kSegW == 16u);
#else
  constexpr bool kPf = false;
#endif
  // sector-interleaved D rows (kernels.h d_phys): the K <= 4096 kernel, 16-entry segments
  // (runtime: create picks the layout per shard, dperm_of)
  const bool kPerm = kDPermOn && kSub == 8u && d.dperm;
  static_assert(!(kDPermOn && kSub == 8u) || (kSegW == 16u && kPf), "interleaved D rows assume 16-entry segments, prefetched");
  uint4 fa = make_uint4(0u, 0u, 0u, 0u), fb = fa, fc = fa, fd = fa;  // prefetched round (kPf)
  uint32_t f_soff = 0;
  auto round_load = [&](uint32_t B0, uint32_t& o_soff, uint4& qa, uint4& qb, uint4& qc, uint4& qd) {
    const uint32_t g = B0 + lane;
    const uint32_t slot = slot_of(B0, soff);
    o_soff = __shfl_sync(kFull, soff, slot);
    const uint32_t s_ebase = __shfl_sync(kFull, ebase, slot);
    const uint32_t s_nnz = __shfl_sync(kFull, nnz, slot);
    const uint32_t sg = g - o_soff, e0 = sg * 16u;  // segment of the row, its first logical entry
    // interleaved rows: the segment's two sectors are physical sectors g%4 and 4 + g%4 of its
    // 64-entry block (consecutive lanes fill whole lines); else consecutive
    const uint32_t* p = d.D + s_ebase + (kPerm ? ((sg >> 2) * 64u + (sg & 3u) * 8u) : e0);
    const uint32_t kSec2 = kPerm ? 32u : 8u;
    qa = qb = qc = qd = make_uint4(0u, 0u, 0u, 0u);
    if (g < T && e0 < s_nnz) ldg256(p, qa, qb);
    if (g < T && e0 + 8u < s_nnz) ldg256(p + kSec2, qc, qd);
  };
  if (kPf) round_load(0u, f_soff, fa, fb, fc, fd);
  for (uint32_t B0 = 0; B0 < T; B0 += 32u) {
    const uint32_t g = B0 + lane;
    unsigned long long acc = 0ull;
    unsigned long long part[4] = {0ull, 0ull, 0ull, 0ull};  // running sums after each sector (kSub == 8)
    uint32_t s_soff;
    if (kPf) {
      const uint4 ca = fa, cb = fb, cc = fc, cd = fd;
      s_soff = f_soff;
      if (B0 + 32u < T) round_load(B0 + 32u, f_soff, fa, fb, fc, fd);
      acc = sector_mac<kDTs>(acc, ca, cb, row_s);
      part[0] = acc;
      acc = sector_mac<kDTs>(acc, cc, cd, row_s);
    } else {
    const uint32_t slot = slot_of(B0, soff);
    s_soff = __shfl_sync(kFull, soff, slot);
    const uint32_t s_ebase = __shfl_sync(kFull, ebase, slot);
    const uint32_t s_nnz = __shfl_sync(kFull, nnz, slot);
    const uint32_t e0 = (g - s_soff) * kSegW;
#ifdef EZLDA_EXP_FAKEROW  // diagnostic: D-row memory traffic removed (entries from a 4 KB table)
    const uint32_t* p = g_fake + ((s_ebase + e0) & 0x3F0u);
#else
    const uint32_t* p = d.D + s_ebase + e0;
#endif
    if (g < T) {
      {
#pragma unroll(kSegW <= 64u ? 4 : 2)
        for (uint32_t b = 0; b < kSegW; b += 16u) {
          uint4 qa = make_uint4(0u, 0u, 0u, 0u), qb = qa, qc = qa, qd = qa;
          if (e0 + b < s_nnz) ldg256(p + b, qa, qb);
          if (e0 + b + 8u < s_nnz) ldg256(p + b + 8u, qc, qd);
          acc = sector_mac<kDTs>(acc, qa, qb, row_s);
          if (kSub == 8u) part[(b >> 3) & 3u] = acc;
          acc = sector_mac<kDTs>(acc, qc, qd, row_s);
          if (kSub == 8u) part[((b >> 3) + 1u) & 3u] = acc;
        }
      }
    }
    }
    const unsigned long long tot = acc;
    // segmented inclusive scan over the lanes of one run (lanes >= rs belong to it)
    const uint32_t rs = (s_soff > B0) ? s_soff - B0 : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      if ((uint32_t)o >= smax) break;
      const unsigned long long y = __shfl_up_sync(kFull, acc, o);
      if (lane >= rs + (uint32_t)o) acc += y;
    }
    if (s_soff < B0) acc += carry;  // the run started in an earlier round
    if (g < T) {
      if (kCk == 1u) {
        sts_u64(ws.P + 8u * g, acc);
      } else if (kCk == 2u) {
        const unsigned long long excl = acc - tot;  // prefix before segment g
        // the two checkpoints of a segment are adjacent: one 16-byte store
        ulonglong2 pr;
        pr.x = excl + part[0];
        pr.y = acc;
        sts_u64x2(ws.P + 16u * g, pr.x, pr.y);
      } else {
        const unsigned long long excl = acc - tot;
        ulonglong2 p0, p1;
        p0.x = excl + part[0];
        p0.y = excl + part[1];
        p1.x = excl + part[2];
        p1.y = acc;
        sts_u64x2(ws.P + 32u * g, p0.x, p0.y);
        sts_u64x2(ws.P + 32u * g + 16u, p1.x, p1.y);
      }
    }
    carry = __shfl_sync(kFull, acc, 31);
  }
  __syncwarp();
#if EZLDA_HDR_PF
  if (pf_dbase != 0xFFFFFFFFu) asm volatile("prefetch.global.L2 [%0];" ::"l"(d.D + pf_dbase));
#endif
  // ---- D: lane per token.  The doc pass left a marker in z^i for the tokens that failed
  //      the MPT test (the others already hold K1): 0x8000 | min(C1, 0x7FFF) when K <=
  //      32768 (d.zmark), else 0xFFFF.
  const double Qp = rec.Qp;
  for (uint32_t B0 = 0; B0 < ntb; B0 += 32u) {
    const double inv_s = scl[0];  // fixed-point scale of m (shared memory, broadcast)
    const uint32_t slot = slot_of(B0, tofs);
    const uint32_t s_j0 = __shfl_sync(kFull, j0, slot);
    const uint32_t s_tofs = __shfl_sync(kFull, tofs, slot);
    const uint32_t s_soff = __shfl_sync(kFull, soff, slot);
    const uint32_t s_nseg = __shfl_sync(kFull, nseg, slot);
    const uint32_t s_ebase = __shfl_sync(kFull, ebase, slot);
    const uint32_t s_nnz = __shfl_sync(kFull, nnz, slot);
    const uint32_t s_L = __shfl_sync(kFull, Ld, slot);
    const uint32_t i = B0 + lane;
    if (i >= ntb) continue;
    const uint32_t j = s_j0 + (i - s_tofs);
    const uint32_t* E = d.D + s_ebase;
#if EZLDA_ZPRE2
    const uint32_t zm = B0 == 0u ? zpre : B0 == 32u ? zpre2 : (uint32_t)nxt.z[j];
#else
    const uint32_t zm = B0 ? (uint32_t)nxt.z[j] : zpre;
#endif
    uint32_t C1;
    if (d.zmark) {
      if (!(zm & 0x8000u)) continue;  // skipped by the MPT test (z^i = K1 < 0x8000)
      C1 = zm & 0x7FFFu;
      if (C1 == d.c1_cap) C1 = row_count(d, E, s_nnz, K1);  // saturated marker: look C1 up
    } else {
      if (zm != kUnsampled) continue;
      C1 = row_count(d, E, s_nnz, K1);
    }
    const uint32_t c0 = kCk * s_soff, nck = kCk * s_nseg;
    const unsigned long long Spi = nck ? lds_u64(ws.P + 8u * (c0 + nck - 1u)) : 0ull;
    const double Sp = (double)Spi * inv_s;  // exact: Spi < 2^48
    const double M = mpt_M(rec, C1, d.alpha);
    const double Z = (M + Sp) + Qp;
    const double u = philox_u_k(d.pk, iter, d.token_base + j);
    const double x = u * Z;
    // certification margin: m_v[k] = rint(What'~ 2^s) with What'~ within 2^-52 relative of
    // What'[v][k] (the reciprocal), so |m 2^-s - What'| <= (1/2 + 2^-20) 2^-s and every
    // fixed-point prefix (exact integer sums) is within delta = 0.500001 (L_d - C1) 2^-s of the exact
    // real prefix; x and y inherit it at most twice (2 delta); the oracle's own sequential fp64
    // sums of nnz terms are within nnz 2^-53 of exact (1.2e-16 nnz Z), and 4e-15 Z covers the
    // roundings of M, Z and x
    // (the K1 entry of m is 0, exact: only the other L_d - C1 counts carry the error)
    const double mg = 1.000002 * (double)(s_L - C1) * inv_s + (4e-15 + 1.2e-16 * (double)s_nnz) * Z;
    uint32_t topic = 0xFFFFFFFFu;
    bool hit = false;
    if (!d.exact_all && fabs(x - M) > mg && fabs(x - (M + Sp)) > mg) {
      if (x < M) {
        topic = K1;  // second chance: u < M / (M + S' + Q')
        hit = true;
      } else if (x < M + Sp) {
        // S' branch: first checkpoint with P > y, then the walk from the previous one, all
        // in exact integers against Yf = floor(y 2^s)  (P > y  <=>  P > Yf for integer P)
        const double y = x - M;
        const unsigned long long Yf = (unsigned long long)(y * scl[1]);
        uint32_t a = c0, b = c0 + nck - 1u;
        while (a < b) {
          const uint32_t mid = (a + b) >> 1;
          if (lds_u64(ws.P + 8u * mid) > Yf) b = mid; else a = mid + 1u;
        }
        const unsigned long long base = (a > c0) ? lds_u64(ws.P + 8u * (a - 1u)) : 0ull;
        unsigned long long pb = base, pa = base;  // prefixes before / after the candidate
        if (kSub == 8u) {  // one sector (8 entries; zero padding past nnz) from registers
          uint4 qa, qb;
#ifdef EZLDA_EXP_FAKEROW
          ldg256(g_fake + ((s_ebase + 16u * ((a - c0) >> 1)) & 0x3F0u) + 8u * ((a - c0) & 1u), qa, qb);
#else
          ldg256(E + (kPerm ? d_phys((a - c0) * 8u) : (a - c0) * 8u), qa, qb);
#endif
          const uint32_t wv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#if EZLDA_WALK2
          // the candidate is the first entry whose running prefix passes Yf.  No K1 or padding
          // test is needed: m[K1] = 0 and padding (w = 0) add 0, and the prefix before the chunk
          // (base) is <= Yf, so neither can be the first to pass.  Branch-free: pb = the last
          // prefix <= Yf, wsel = the entry where the prefix crosses; pa = pb + its product.
          {
            unsigned long long q = pa;
            uint32_t wsel = 0u;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const unsigned long long qn = entry_mac<kDTs>(wv[e], row_s, q);
              const bool le = qn <= Yf;
              if (le) pb = qn;
              if (!le && q <= Yf) wsel = wv[e];
              q = qn;
            }
            topic = d_topic(wsel, kDTs);
            pa = entry_mac<kDTs>(wsel, row_s, pb);
          }
#else
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const uint32_t w = wv[e];
            if (topic == 0xFFFFFFFFu && w != 0u) {
              const unsigned long long q = entry_mac<kDTs>(w, row_s, pa);
              if (d_topic(w, kDTs) != K1 && q > Yf) topic = d_topic(w, kDTs);
              else pb = q;
              pa = q;
            }
          }
#endif
        } else {
          // walk the chunk two sectors (16 entries) at a time from registers: one memory
          // round trip per 16 entries instead of one per entry
          const uint32_t e0 = (a - c0) * kSub;
          for (uint32_t eb = e0; eb < e0 + kSub && eb < s_nnz && topic == 0xFFFFFFFFu; eb += 16u) {
            uint4 qa, qb, qc = make_uint4(0u, 0u, 0u, 0u), qd = qc;
            ldg256(E + eb, qa, qb);
            if (eb + 8u < s_nnz) ldg256(E + eb + 8u, qc, qd);
            const uint32_t wv[16] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w,
                                     qc.x, qc.y, qc.z, qc.w, qd.x, qd.y, qd.z, qd.w};
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const uint32_t w = wv[e];
              if (topic == 0xFFFFFFFFu && w != 0u) {  // w == 0: zero padding past nnz
                const unsigned long long q = entry_mac<kDTs>(w, row_s, pa);
                if (d_topic(w, kDTs) != K1 && q > Yf) topic = d_topic(w, kDTs);
                else pb = q;
                pa = q;
              }
            }
          }
        }
        // certify: the candidate's interval [pb, pa) holds y with margin on both sides
        if (topic != 0xFFFFFFFFu && !((double)pa * inv_s - y > mg && y - (double)pb * inv_s > mg))
          topic = 0xFFFFFFFFu;  // uncertified: exact redraw
      } else {
        // Q' branch: first topic k != K1 with alpha P(k) > y, searched over the fixed-point
        // copy qfx = rint(QP 2^t) of the oracle's prefix table (flat across K1) against
        // Yq = floor(y 2^t); certified with the margin widened by qfx's one-ulp error
        const double y = (x - M) - Sp;
        if (y >= 0.0) {
          const double inv_t = scl[2];
          const uint32_t Yq = (uint32_t)fmin(y * scl[3], 4294967295.0);  // past the end: uncertified
          uint32_t a = 0, b = d.Kpad - 1u;
          // the table is in the slot (shared memory) or, for large K (kQG), in HBM
          // (chunk ends ce in the slot either way: the HBM search touches one 128-byte line)
          // (HBM table: L1-cached loads, coherent within the SM -- a warp-staged item's table is
          // written inside this kernel by a warp of the same block, published by the slot's
          // release / acquire)
          auto qv = [&](uint32_t i) -> uint32_t { return kQG ? __ldca(qfx + q_swz(i)) : qfx[q_swz(i)]; };
          {  // first the 32-topic chunk from the contiguous chunk ends
            uint32_t ca = 0, cb = d.nch - 1u;
            while (ca < cb) {
              const uint32_t mid = (ca + cb) >> 1;
              if (ce[mid] > Yq) cb = mid; else ca = mid + 1u;
            }
            a = 32u * ca;
            b = a + 31u;
          }
          if (kQG && EZLDA_QG_VEC) {
            // HBM table (large K): the chunk's 32 entries (one 128-byte line) with 8 independent
            // 16-byte loads instead of 5 dependent probes; qfx is non-decreasing, so the first
            // entry > Yq sits at the count of entries <= Yq (the swizzle only permutes the line)
            const uint4* q4 = reinterpret_cast<const uint4*>(qfx + a);
            uint32_t cnt = 0;
#pragma unroll 1
            for (int h2 = 0; h2 < 8; h2 += 4) {  // two groups of four loads (register budget)
              uint4 x[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) x[q] = __ldca(q4 + h2 + q);
#pragma unroll
              for (int q = 0; q < 4; ++q) cnt += (x[q].x <= Yq) + (x[q].y <= Yq) + (x[q].z <= Yq) + (x[q].w <= Yq);
            }
            a += min(cnt, 31u);
          } else {
            while (a < b) {
              const uint32_t mid = (a + b) >> 1;
              if (qv(mid) > Yq) b = mid; else a = mid + 1u;
            }
          }
          // + one qfx ulp + the bound (K + 4) 2^-52 Q' on the difference between the staged
          // chunked prefix and the oracle's sequential one (stage_row_warp)
          const double mq = mg + inv_t + (double)(d.K + 4u) * 0x1p-52 * Qp;
          const double qa = (double)qv(a) * inv_t, qp = a ? (double)qv(a - 1u) * inv_t : 0.0;
          if (a != K1 && a < d.K && qa - y > mq && y - qp > mq) topic = a;
        }
      }
    }
    if (topic == 0xFFFFFFFFu) {
      topic = exact_draw<(kSub == 16u)>(d, cur, v, rec, E, s_nnz, M, u, hit);
      rc.exact += 1;
    }
    if (hit) rc.hitM += 1;
    nxt.z[j] = (uint16_t)topic;
    if (d.hist_bitmap) {
      if (atomicAdd(&hist[topic], 1u) == 0u)  // first token of this topic in the item: mark it
        atomicOr(&hist[d.Kpad + (topic >> 5)], 1u << (topic & 31u));
    } else if (EZLDA_RED_SHARED && !d.hist_global) {  // shared-space reduction (not a generic atomic)
      asm volatile("red.shared.add.u32 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(hist + topic)) : "memory");
    } else {
      atomicAdd(&hist[topic], 1u);
    }
    rc.sampled += 1;
  }
  __syncwarp();
  return nb;
}

// ---------------------------------------------------------------------------------
// Persistent, slot-pipelined sampler.  One block per SM (kSampWarps warps) loops over the
// global heavy-first item list.  The block's k-th item lives in slot k % kSlots (What'
// row + QP, topic histogram, cursor, counters).  Every warp walks the block's items in
// order and leaves an item as soon as its run cursor is exhausted; the LAST warp to leave
// item k writes its W row / n_k (warp-level epilogue) and re-arms the slot with block
// item k + kSlots (claim from the global counter, TMA bulk copy of a dense What' row or a
// warp-staged tail row).  No block-wide barrier after the prologue: a warp is never idle
// while another warp finishes the previous item.
// ---------------------------------------------------------------------------------
#ifndef EZLDA_SLOTS
#define EZLDA_SLOTS 3
#endif
constexpr uint32_t kMaxSlots = EZLDA_SLOTS;  // slots per block when they fit (d.nslots: 1 for large K)
constexpr uint32_t kExit = 0x80000000u;

struct __align__(16) SlotCtl {
  WordRec rec;
  uint64_t mbar;
  uint32_t v, r0, r1, ntok;
  uint32_t cursor, done;
  uint32_t sampled, hitM, runs, words, exact;
  uint32_t state;  // block item number held by the slot (| kExit: no item left)
  const uint32_t* qfx; // fixed-point Q' prefix table (slot shared memory, or HBM scratch if d.qfx_global)
};

__device__ __forceinline__ uint32_t ld_acquire_s(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}

__device__ __forceinline__ void st_release_s(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v)
               : "memory");
}

// per-slot dynamic shared memory: m u32 [Kpad] | qfx u32 [Kpad] | scales f64 [4] (one bulk
// copy of the word's wrow record head) | hist u32 [Kpad] when it fits (else in HBM scratch)
__host__ __device__ __forceinline__ uint32_t slot_head_bytes(uint32_t Kpad, uint32_t qfx_global) {
  // m | scales | ce (qfx searched in HBM), or m | scales | qfx | ce
  return qfx_global ? 4u * Kpad + 32u + 4u * ce_words(Kpad) : 8u * Kpad + 32u + 4u * ce_words(Kpad);
}

// The item word's sampler head staged by one warp straight from W (no precomputed table):
//   m[k]   = rint(What'[v][k] 2^s), What' = (W[v][k] + beta) * (1 / den_k) with the K1 entry 0
//            (Eq 6); one rounding more than the oracle's quotient, so |m 2^-s - What'| < 2^-s
//            still holds (the S' certification margin);
//   qfx[k] = rint(alpha P'(k) 2^t), P' the fp64 prefix of What' in chunks of 32 topics (warp
//            scan + running carry) -- another summation order than the oracle's sequential
//            P_v, within (K + 4) 2^-52 Q' of it (standard fp64 summation bound, included in the
//            Q' certification margin); ce[c] = qfx[32 c + 31] (chunk ends, in the slot);
//   sc     = {2^-s, 2^s, 2^-t, 2^t} from a2 = max What' and Q' of the word record.
// Tail words: the packed row's counts are first scattered into m (used as a count array).
__device__ void stage_row_warp(const Dev& d, const Buf& cur, uint32_t v, const WordRec& rec, uint32_t* m,
                               uint32_t* qfx, uint32_t* ce, double* sc) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t K1 = rec.K[0];
  int e = 0;
  frexp(rec.a[1], &e);
  const int sh = 32 - e;  // max What' 2^sh in [2^31, 2^32)
  const double two_s = ldexp(1.0, sh);
  int et = 0;
  frexp(rec.Qp, &et);
  const double two_t = ldexp(1.0, 32 - et);  // Q' 2^t in [2^31, 2^32)
  const bool dense = v < d.Vd;
  const int32_t* wr = cur.Wd + (size_t)v * d.K;
  if (!dense) {
    for (uint32_t k = lane; k < d.Kpad; k += 32u) m[k] = 0u;
    __syncwarp();
    const uint32_t t = v - d.Vd;
    const uint32_t* tr = cur.Wt + d.tofs[t];
    const uint32_t n = cur.tnnz[t];
    for (uint32_t i = lane; i < n; i += 32u) {
      const uint32_t p = tr[i];
      m[p >> 16] = p & 0xFFFFu;
    }
    __syncwarp();
  }
  // 128 topics per step, four consecutive topics per lane: local prefix of the four, one warp
  // scan of the lane totals (exclusive prefix by a shifted read, no subtraction), 16-byte m /
  // qfx stores; the chunk ends ce[c] = qfx[32 c + 31] fall on lanes 7, 15, 23, 31
  double carry = 0.0;
  for (uint32_t c0 = 0; c0 < d.Kpad; c0 += 128u) {
    const uint32_t kb = c0 + 4u * lane;  // a multiple of 4; Kpad too: all four in or all out
    const bool in4 = kb < d.Kpad;
    double w[4];
    if (in4) {
      uint32_t cnt[4];
      if (dense) {
#pragma unroll
        for (int i = 0; i < 4; ++i) cnt[i] = (kb + i < d.K) ? (uint32_t)__ldg(wr + kb + i) : 0u;
      } else {
        const uint4 c4 = *reinterpret_cast<const uint4*>(m + kb);
        cnt[0] = c4.x; cnt[1] = c4.y; cnt[2] = c4.z; cnt[3] = c4.w;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t k = kb + i;
        w[i] = (k < d.K && k != K1) ? ((double)cnt[i] + d.beta) * __ldg(d.inv_den + k) : 0.0;
      }
      uint4 mm;
      mm.x = __double2uint_rn(fmin(w[0] * two_s, 4294967295.0));
      mm.y = __double2uint_rn(fmin(w[1] * two_s, 4294967295.0));
      mm.z = __double2uint_rn(fmin(w[2] * two_s, 4294967295.0));
      mm.w = __double2uint_rn(fmin(w[3] * two_s, 4294967295.0));
      *reinterpret_cast<uint4*>(m + kb) = mm;
    } else {
      w[0] = w[1] = w[2] = w[3] = 0.0;
    }
    const double p0 = w[0], p1 = p0 + w[1], p2 = p1 + w[2], p3 = p2 + w[3];
    double incl = p3;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(kFull, incl, o);
      if (lane >= (uint32_t)o) incl = incl + y;
    }
    const double prev = __shfl_up_sync(kFull, incl, 1);
    const double base = carry + (lane ? prev : 0.0);
    if (in4) {
      uint4 q4;
      q4.x = __double2uint_rn(fmin(d.alpha * (base + p0) * two_t, 4294967295.0));
      q4.y = __double2uint_rn(fmin(d.alpha * (base + p1) * two_t, 4294967295.0));
      q4.z = __double2uint_rn(fmin(d.alpha * (base + p2) * two_t, 4294967295.0));
      q4.w = __double2uint_rn(fmin(d.alpha * (base + p3) * two_t, 4294967295.0));
      if ((lane & 7u) == 7u) ce[(kb + 3u) >> 5] = q4.w;
#if EZLDA_QSWZ
      {  // swizzled store (q_swz): topic kb + t at (kb ^ (x & ~3)) + (t ^ (x & 3)), x = chunk & 31
        const uint32_t x = (kb >> 5) & 31u;
        uint32_t t;  // element p of the stored vector = topic kb + (p ^ (x & 3)): swap pairs, then halves
        if (x & 1u) { t = q4.x; q4.x = q4.y; q4.y = t; t = q4.z; q4.z = q4.w; q4.w = t; }
        if (x & 2u) { t = q4.x; q4.x = q4.z; q4.z = t; t = q4.y; q4.y = q4.w; q4.w = t; }
        *reinterpret_cast<uint4*>(qfx + (kb ^ (x & ~3u))) = q4;
      }
#else
      *reinterpret_cast<uint4*>(qfx + kb) = q4;
#endif
    }
    carry = carry + __shfl_sync(kFull, incl, 31);
  }
  for (uint32_t c = d.nch + lane; c < ce_words(d.Kpad); c += 32u) ce[c] = 0xFFFFFFFFu;
  if (lane == 0) {
    sc[0] = 1.0 / two_s;
    sc[1] = two_s;
    sc[2] = 1.0 / two_t;
    sc[3] = two_t;
  }
  __syncwarp();
}

// Sampler head of word v in the wrow table (v < Vw; k_word_heads): m | scales | qfx | ce.
struct HeadPtrs {
  uint32_t* m;
  double* sc;
  uint32_t* qfx;
  uint32_t* ce;
};
__device__ __forceinline__ HeadPtrs head_ptrs(const Dev& d, uint32_t v) {
  unsigned char* b = d.wrow + (size_t)v * d.rs_bytes;
  HeadPtrs o;
  o.m = reinterpret_cast<uint32_t*>(b);
  o.sc = reinterpret_cast<double*>(b + 4u * d.Kpad);
  o.qfx = reinterpret_cast<uint32_t*>(b + 4u * d.Kpad + 32u);
  o.ce = o.qfx + d.Kpad;
  return o;
}

// Arm slot `sl` with block item k (one warp): claim the next global item, publish its
// description and fill the slot with the word's head: ONE TMA bulk copy (cp.async.bulk,
// completing on the slot's mbarrier) of the precomputed head (v < Vw), else staged by this
// warp (stage_row_warp) followed by a plain arrive.  The slot's histogram is zero on entry.
__device__ void arm_slot(const Dev& d, const Buf& cur, SlotCtl& c, unsigned char* sbase, uint32_t* qfx_scratch,
                         uint32_t k, uint32_t n_items) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t i = 0;
  if (lane == 0) i = (uint32_t)atomicAdd(&d.ctr->item_ctr, 1ull);
  i = __shfl_sync(kFull, i, 0);
  if (i >= (d.n_act ? *d.n_act : n_items)) {
    if (lane == 0) st_release_s(&c.state, k | kExit);
    return;
  }
  if (d.item_act) i = d.item_act[i];  // this iteration's schedule (H4): items with a flagged run
  const uint32_t v = d.item_word[i];
  if (lane == 0) atomicAdd(&d.ctr->items, 1ull);
  uint32_t* mrow = reinterpret_cast<uint32_t*>(sbase);
  const uint32_t mbar_s = (uint32_t)__cvta_generic_to_shared(&c.mbar);
  if (lane < 6) reinterpret_cast<uint64_t*>(&c.rec)[lane] = reinterpret_cast<const uint64_t*>(d.rec + v)[lane];
  if (lane == 0) {
    c.v = v;
    c.r0 = d.item_r0[i];
    c.r1 = d.item_r1[i];
    c.ntok = d.item_ntok[i];
    c.cursor = 0;
    c.done = 0;
    c.sampled = 0;
    c.hitM = 0;
    c.runs = 0;
    c.words = 0;
    c.exact = 0;
  }
  if (v < d.Vw) {  // precomputed by k_word_heads
    if (lane == 0) {
      const HeadPtrs o = head_ptrs(d, v);
      const uint32_t ms = (uint32_t)__cvta_generic_to_shared(mrow);
      if (!d.qfx_global) {  // m | scales | qfx | ce: one contiguous bulk copy
        c.qfx = mrow + d.Kpad + 8u;
        bulk_g2s(ms, o.m, slot_head_bytes(d.Kpad, 0u), mbar_s);
      } else {  // m | scales, then the chunk ends ce (the qfx table itself stays in HBM)
        c.qfx = o.qfx;
        const uint32_t b1 = 4u * d.Kpad + 32u, b2 = 4u * ce_words(d.Kpad);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar_s), "r"(b1 + b2) : "memory");
        bulk_copy_tx(ms, o.m, b1, mbar_s);
        bulk_copy_tx(ms + b1, o.ce, b2, mbar_s);
      }
    }
  } else {
    __syncwarp();
    // slot: m | scales | qfx | ce, or m | scales | ce with qfx in the slot's HBM scratch
    uint32_t* qfx = d.qfx_global ? qfx_scratch : mrow + d.Kpad + 8u;
    uint32_t* ce = d.qfx_global ? mrow + d.Kpad + 8u : qfx + d.Kpad;
    if (lane == 0) c.qfx = qfx;
    stage_row_warp(d, cur, v, c.rec, mrow, qfx, ce, reinterpret_cast<double*>(mrow + d.Kpad));
    if (d.qfx_global) __threadfence_block();  // the HBM qfx table before the arrive / release
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar_s) : "memory");
  }
  __syncwarp();
  if (lane == 0) st_release_s(&c.state, k);
}

// H1 (second half): the sampler heads of this iteration's words (the words of the live items
// when the per-iteration schedule runs, else every word; v < Vw) into the wrow table, one
// warp per word -- the same staging as an in-kernel item (stage_row_warp), written to HBM
// for the sampler's bulk copies.
__global__ void __launch_bounds__(128) k_word_heads(Dev d, Buf cur) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t v = blockIdx.x * 4u + (threadIdx.x >> 5);
  if (v >= d.Vw || d.wtok[v + 1] == d.wtok[v]) return;
  if (d.word_live && !d.word_live[v]) return;
  (void)lane;
  const WordRec r = d.rec[v];
  const HeadPtrs o = head_ptrs(d, v);
  stage_row_warp(d, cur, v, r, o.m, o.qfx, o.ce, o.sc);
}

// Warp-level epilogue of a finished item: skipped tokens at K1, W row / n_k from the
// histogram (dense: atomics; tail: ordered compaction into the packed row), histogram
// re-zeroed for the slot's next item.
__device__ void item_epilogue_warp(const Dev& d, const Buf& nxt, SlotCtl& c, uint32_t* hist) {
  // hist[Kpad] counts + bitmap [Kpad / 32] of the topics present: only the marked topics are
  // visited (O(K/32 + nnz) per item), in ascending order, and re-zeroed
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t v = c.v;
  uint32_t* bmp = hist + d.Kpad;
  const uint32_t bw = d.Kpad >> 5;
  if (lane == 0) {  // skipped tokens stay at K1
    const uint32_t K1 = c.rec.K[0], n = c.ntok - c.sampled;
    if (n) {
      const uint32_t old = hist[K1];
      hist[K1] = old + n;
      if (!old && d.hist_bitmap) bmp[K1 >> 5] |= 1u << (K1 & 31u);
    }
  }
  __syncwarp();
  const bool dense = v < d.Vd;
  int32_t* Wrow = dense ? nxt.Wd + (size_t)v * d.K : nullptr;
  uint32_t* out = dense ? nullptr : nxt.Wt + d.tofs[v - d.Vd];
  uint32_t nz = 0;
  if (!d.hist_bitmap) {  // small K: visit all K counters (no per-token bitmap maintenance)
    for (uint32_t base = 0; base < d.Kpad; base += 32u) {
      const uint32_t k = base + lane;
      const uint32_t n = hist[k];  // zero past K
      const uint32_t m = __ballot_sync(kFull, n != 0);
      if (n) {
        if (dense) atomicAdd(&Wrow[k], (int32_t)n);
        else out[nz + __popc(m & lanemask_lt())] = (k << 16) | n;
        hist[k] = 0;
      }
      nz += __popc(m);
    }
  }
  for (uint32_t base = 0; d.hist_bitmap && base < bw; base += 32u) {
    const uint32_t wi = base + lane;
    const uint32_t b = (wi < bw) ? bmp[wi] : 0u;
    const uint32_t cnt = __popc(b);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    uint32_t pos = nz + incl - cnt;
    for (uint32_t m = b; m; m &= m - 1u) {
      const uint32_t k = wi * 32u + (__ffs(m) - 1u);
      const uint32_t n = hist[k];
      if (dense) atomicAdd(&Wrow[k], (int32_t)n);
      else out[pos++] = (k << 16) | n;
      hist[k] = 0;
    }
    if (b) bmp[wi] = 0;
    nz += __shfl_sync(kFull, incl, 31);
  }
  if (!dense && lane == 0) nxt.tnnz[v - d.Vd] = nz;
  if (lane == 0) {
    atomicAdd(&d.ctr->sampled, (unsigned long long)c.sampled);
    atomicAdd(&d.ctr->skip_M, (unsigned long long)c.hitM);
    atomicAdd(&d.ctr->active_runs, (unsigned long long)c.runs);
    atomicAdd(&d.ctr->drow_words, (unsigned long long)c.words);
    if (c.exact) atomicAdd(&d.ctr->exact, (unsigned long long)c.exact);
  }
  __syncwarp();
}

#ifndef EZLDA_SAMP_WARPS
#define EZLDA_SAMP_WARPS 14
#endif
constexpr int kSampWarpsP = EZLDA_SAMP_WARPS;

__host__ __device__ __forceinline__ uint32_t sampler_ctl_bytes() {
  return (uint32_t)((sizeof(SlotCtl) * kMaxSlots + 15u) & ~15u);
}

#ifndef EZLDA_SAMP_MINB
#define EZLDA_SAMP_MINB 2  // resident sampler blocks per SM the register allocation must allow
#endif

// one kernel per (S' segment width, Q' table placement): each gets the register allocation
// of its own path only
template <uint32_t kSegW, uint32_t kSub, uint32_t kFbW, uint32_t kDTs, bool kQG>
__global__ void __launch_bounds__(kSampWarpsP * 32, EZLDA_SAMP_MINB) k_sampler(Dev d, Buf cur, Buf nxt, uint32_t iter,
                                                                  uint32_t n_items) {
  extern __shared__ __align__(16) unsigned char smem[];
  SlotCtl* ctl = reinterpret_cast<SlotCtl*>(smem);
  unsigned char* slots = smem + sampler_ctl_bytes();
  const uint32_t sb = d.slot_bytes;
  const uint32_t nsl = d.nslots;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  WarpScratch ws;
  {
    unsigned char* wb = slots + nsl * sb + warp * d.ws_bytes;
    ws.P = (uint32_t)__cvta_generic_to_shared(wb);
    ws.q = ws.P + d.ws_bytes - 4u * kQueue;
    ws.head = 0;
  }
  // histogram of slot sl: shared memory after the slot head, or this block's HBM scratch
  auto hist_of = [&](uint32_t sl) -> uint32_t* {
    return d.hist_global ? d.hist_scratch + ((size_t)blockIdx.x * nsl + sl) * (d.Kpad + d.Kpad / 32u)
                         : reinterpret_cast<uint32_t*>(slots + sl * sb + slot_head_bytes(d.Kpad, d.qfx_global));
  };
  // fixed-point Q' table of slot sl in HBM (d.qfx_global: large K)
  auto qfs_of = [&](uint32_t sl) -> uint32_t* {
    return d.qfx_global ? d.qfx_scratch + ((size_t)blockIdx.x * nsl + sl) * d.Kpad : nullptr;
  };
  const uint32_t nw = blockDim.x >> 5;
  // prologue: barriers, zero histograms, warp 0 arms the first kSlots items
  if (tid == 0) {
    for (uint32_t sl = 0; sl < nsl; ++sl) {
      const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&ctl[sl].mbar);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(1u) : "memory");
      ctl[sl].state = 0xFFFFFFFFu;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (!d.hist_global)  // (the HBM scratch histograms are zeroed at create and by every epilogue)
    for (uint32_t sl = 0; sl < nsl; ++sl) {
      uint32_t* hist = hist_of(sl);
      for (uint32_t k = tid; k < d.Kpad + d.Kpad / 32u; k += blockDim.x) hist[k] = 0;  // counts + bitmap
    }
  __syncthreads();
  if (warp == 0)
    for (uint32_t sl = 0; sl < nsl; ++sl) arm_slot(d, cur, ctl[sl], slots + sl * sb, qfs_of(sl), sl, n_items);
  for (uint32_t k = 0;; ++k) {
    const uint32_t sl = k % nsl;
    SlotCtl& c = ctl[sl];
    uint32_t st = 0;
    if (lane == 0) {
#if EZLDA_SPIN_MAX > 32
      uint32_t ns = 32u;  // exponential backoff: fewer spin instructions competing for issue
      while (((st = ld_acquire_s(&c.state)) & ~kExit) != k) {
        __nanosleep(ns);
        ns = min(2u * ns, (uint32_t)EZLDA_SPIN_MAX);
      }
#else
      while (((st = ld_acquire_s(&c.state)) & ~kExit) != k) __nanosleep(32);
#endif
    }
    st = __shfl_sync(kFull, st, 0);
    __syncwarp();  // orders lane 0's acquire before the other lanes' reads of the slot
    if (st & kExit) break;
    mbar_wait((uint32_t)__cvta_generic_to_shared(&c.mbar), (k / nsl) & 1u);
    // fixed-point Q' table: in the slot right after the scales, or in HBM (kQG, large K)
    const uint32_t* qfx = kQG ? c.qfx : reinterpret_cast<const uint32_t*>(slots + sl * sb + 4u * d.Kpad + 32u);
    const uint32_t* ce = kQG ? reinterpret_cast<const uint32_t*>(slots + sl * sb + 4u * d.Kpad + 32u) : qfx + d.Kpad;
    const double* scl = reinterpret_cast<const double*>(slots + sl * sb + 4u * d.Kpad);
    uint32_t* hist = hist_of(sl);
    const WordRec rec = c.rec;
    const uint32_t v = c.v, r0 = c.r0, r1 = c.r1;
    const uint32_t row_s = (uint32_t)__cvta_generic_to_shared(slots + sl * sb);
    RunCounters rc{0, 0, 0, 0, 0};
    uint32_t qn = 0;
    bool exhausted = false;
    bool pf_ok = false;  // a claimed run group (pf_rb) whose flag words (pf_fw) are in flight
    uint32_t pf_rb = 0, pf_fw = 0;
    while (true) {
      // refill the queue with flagged runs (warp-uniform control flow throughout): groups of
      // G = d.grp runs are claimed from the item's cursor (G = 32, or fewer at large K so that
      // an item's long rows spread over more warps), the next group one refill ahead
      const uint32_t G = d.grp;
      while (qn < G && !exhausted) {
        uint32_t rb, fw;
        if (pf_ok) {
          rb = pf_rb;
          fw = pf_fw;
          pf_ok = false;
        } else {
          uint32_t grp = 0;
          if (lane == 0) grp = atomicAdd(&c.cursor, 1u);
          rb = r0 + __shfl_sync(kFull, grp, 0) * G;
          fw = (lane < G && rb + lane < r1) ? d.flags[(rb + lane) >> 5] : 0u;
        }
        if (rb >= r1) {
          exhausted = true;
          break;
        }
        const uint32_t r = rb + lane;
        const bool act = lane < G && (r < r1) && ((fw >> (r & 31u)) & 1u);
        const uint32_t m = __ballot_sync(kFull, act);
        if (act) sts_u32(ws_q_at(ws, qn + __popc(m & lanemask_lt())), r);
        qn += __popc(m);
        __syncwarp();
      }
      if (qn == 0) break;
      if (!exhausted && !pf_ok) {
        uint32_t grp = 0;
        if (lane == 0) grp = atomicAdd(&c.cursor, 1u);
        pf_rb = r0 + __shfl_sync(kFull, grp, 0) * G;
        pf_fw = (lane < G && pf_rb + lane < r1) ? d.flags[(pf_rb + lane) >> 5] : 0u;
        pf_ok = true;
      }
      uint32_t nb = sample_batch<kSegW, kSub, kDTs, kQG>(d, cur, nxt, rec, v, row_s, qfx, ce, scl, hist, ws,
                                                         qn, iter, rc);
      if (kFbW && nb == 0)  // a run with more than kSegCap x 16 nonzeros (large K only): wide segments
        nb = sample_batch<kFbW ? kFbW : 16u, kFbW ? kFbW : 16u, kDTs, kQG>(d, cur, nxt, rec, v, row_s, qfx, ce, scl,
                                                                          hist, ws, qn, iter, rc);

      // drop the processed runs from the queue (ring)
      ws.head += nb;
      qn -= nb;
      __syncwarp();
    }
    const uint32_t smp = warp_sum(rc.sampled), hm = warp_sum(rc.hitM);
    const uint32_t nr = warp_sum(rc.runs), nwd = warp_sum(rc.words), nex = warp_sum(rc.exact);
    uint32_t last = 0;
    if (lane == 0) {
      if (nex) atomicAdd(&c.exact, nex);
      if (smp) atomicAdd(&c.sampled, smp);
      if (hm) atomicAdd(&c.hitM, hm);
      if (nr) atomicAdd(&c.runs, nr);
      if (nwd) atomicAdd(&c.words, nwd);
      __threadfence_block();
      last = (atomicAdd(&c.done, 1u) == nw - 1u);
      if (last) __threadfence_block();
    }
    last = __shfl_sync(kFull, last, 0);
    if (last) {
      item_epilogue_warp(d, nxt, c, hist);
      arm_slot(d, cur, c, slots + sl * sb, qfs_of(sl), k + nsl, n_items);
    }
  }
}

// W / n_k of one item from its topic histogram, block-wide (dense rows: atomics, the item
// may be one of several regions of the word; tail rows: ordered compaction).
__device__ void item_epilogue(const Dev& d, const Buf& nxt, uint32_t v, const uint32_t* hist, uint32_t* s_wsum,
                              uint32_t* s_run) {
  const uint32_t tid = threadIdx.x;
  if (v < d.Vd) {
    int32_t* Wrow = nxt.Wd + (size_t)v * d.K;
    for (uint32_t k = tid; k < d.K; k += blockDim.x) {
      const uint32_t c = hist[k];
      if (c) atomicAdd(&Wrow[k], (int32_t)c);
    }
  } else {
    const uint32_t t = v - d.Vd;
    const uint32_t nz = block_compact(hist, d.K, nxt.Wt + d.tofs[t], s_wsum, s_run, 16u);
    if (tid == 0) nxt.tnnz[t] = nz;
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

// H6: n_k = sum_v W[v][k] once W is complete (after the sampler, and after the H7 merge
// when world > 1): column sums of the dense block (consecutive threads read consecutive
// topics of a row: coalesced) and the tail rows' packed entries, reduced per block in shared
// memory, then one atomic per (block, topic) -- no per-(item, topic) global atomics.
constexpr uint32_t kNkBlocks = 296;
__global__ void __launch_bounds__(256) k_nk(Dev d, Buf b) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* s_nk = reinterpret_cast<uint32_t*>(smem);
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  for (uint32_t k = tid; k < d.Kpad; k += blockDim.x) s_nk[k] = 0u;
  __syncthreads();
  const uint32_t rpb = (d.Vd + gridDim.x - 1u) / gridDim.x;  // dense rows of this block
  const uint32_t v0 = min(d.Vd, blockIdx.x * rpb), v1 = min(d.Vd, v0 + rpb);
  for (uint32_t k = tid; k < d.K; k += blockDim.x) {  // thread-owned topics: plain adds
    uint32_t acc = 0;
    const int32_t* col = b.Wd + k;
    uint32_t v = v0;
    for (; v + 4u <= v1; v += 4u)
      acc += (uint32_t)col[(size_t)v * d.K] + (uint32_t)col[(size_t)(v + 1u) * d.K] +
             (uint32_t)col[(size_t)(v + 2u) * d.K] + (uint32_t)col[(size_t)(v + 3u) * d.K];
    for (; v < v1; ++v) acc += (uint32_t)col[(size_t)v * d.K];
    s_nk[k] = acc;
  }
  __syncthreads();
  const uint32_t Vt = d.V - d.Vd;
  const uint32_t tpb = (Vt + gridDim.x - 1u) / gridDim.x;  // tail words of this block
  const uint32_t t0 = min(Vt, blockIdx.x * tpb), t1 = min(Vt, t0 + tpb);
  for (uint32_t t = t0 + warp; t < t1; t += blockDim.x >> 5) {
    const uint32_t* tr = b.Wt + d.tofs[t];
    const uint32_t n = b.tnnz[t];
    for (uint32_t e = lane; e < n; e += 32u) {
      const uint32_t p = tr[e];
      atomicAdd(&s_nk[p >> 16], p & 0xFFFFu);
    }
  }
  __syncthreads();
  for (uint32_t k = tid; k < d.K; k += blockDim.x) {
    const uint32_t n = s_nk[k];
    if (n) atomicAdd(&b.nk[k], (int32_t)n);
  }
}

// H7 (world > 1): global packed tail row of tail word t from every rank's word-major tail
// topics (all-gathered): segment r of word t is tz_all[r * tail_max + off_r[t] .. off_r[t+1]).
// Block per tail word: shared histogram, ordered compaction (integer: identical on all ranks).
__global__ void __launch_bounds__(256) k_tail_rebuild(Dev d, Buf nxt, const uint16_t* tz_all, const uint32_t* off,
                                                      uint32_t world, uint64_t tail_max) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
  __shared__ uint32_t s_wsum[32], s_run;
  const uint32_t t = blockIdx.x, Vt = d.V - d.Vd;
  uint32_t tot = 0;
  for (uint32_t r = 0; r < world; ++r) tot += off[(size_t)r * (Vt + 1) + t + 1] - off[(size_t)r * (Vt + 1) + t];
  if (tot == 0) {  // no token of the word on any rank
    if (threadIdx.x == 0) nxt.tnnz[t] = 0;
    return;
  }
  for (uint32_t k = threadIdx.x; k < d.Kpad; k += blockDim.x) hist[k] = 0;
  __syncthreads();
  for (uint32_t r = 0; r < world; ++r) {
    const uint32_t o0 = off[(size_t)r * (Vt + 1) + t], o1 = off[(size_t)r * (Vt + 1) + t + 1];
    const uint16_t* src = tz_all + (size_t)r * tail_max;
    for (uint32_t i = o0 + threadIdx.x; i < o1; i += blockDim.x) atomicAdd(&hist[src[i]], 1u);
  }
  __syncthreads();
  const uint32_t nz = block_compact(hist, d.K, nxt.Wt + d.tofs[t], s_wsum, &s_run, 16u);
  if (threadIdx.x == 0) nxt.tnnz[t] = nz;
}

// H4 per iteration: warp per item, flagged runs of the item counted from the flag bitset.
// An item without a flagged run holds only skipped tokens (z^i = K1 for all of them): its W
// row / n_k contribution is written here and the sampler never stages it.
__global__ void __launch_bounds__(256) k_item_schedule(Dev d, Buf nxt, uint32_t n_items) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t item = blockIdx.x * 8u + (threadIdx.x >> 5);
  if (item >= n_items) return;
  const uint32_t r0 = d.item_r0[item], r1 = d.item_r1[item];
  uint32_t f = 0;
  const uint32_t w0 = r0 >> 5, w1 = (r1 - 1u) >> 5;
  for (uint32_t wb = w0 + lane; wb <= w1; wb += 32u) {
    uint32_t x = d.flags[wb];
    if (wb == w0) x &= 0xFFFFFFFFu << (r0 & 31u);
    if (wb == w1 && (r1 & 31u) != 0u) x &= 0xFFFFFFFFu >> (32u - (r1 & 31u));
    f |= x;
  }
  const uint32_t any = __any_sync(kFull, f != 0u) ? 1u : 0u;
  if (lane == 0) {
    d.item_live[item] = (uint8_t)any;
    if (any && d.word_live) d.word_live[d.item_word[item]] = 1u;  // its head is needed (k_word_heads)
    if (!any) {
      const uint32_t v = d.item_word[item], n = d.item_ntok[item], K1 = d.rec[v].K[0];
      if (v < d.Vd) {
        atomicAdd(&nxt.Wd[(size_t)v * d.K + K1], (int32_t)n);
      } else {  // a tail word has exactly one item: its row is the single entry (K1, n)
        nxt.Wt[d.tofs[v - d.Vd]] = (K1 << 16) | n;
        nxt.tnnz[v - d.Vd] = 1u;
      }
    }
  }
}

// ---------------------------------------------------------------------------------
// H8: LLPT, Eq (5) via sum_k (D+alpha) What = S_full + Q_full, one value per (d, v) run.
// ---------------------------------------------------------------------------------
// kG (large K): the row / chunk prefix live in a per-block HBM scratch (the fp64 row of K =
// 32768 does not fit shared memory) and the blocks loop over the items.
template <bool kG>
__global__ void __launch_bounds__(kLlptWarps * 32) k_llpt(Dev d, Buf cur, double* partial, uint32_t n_items,
                                                          double* scratch) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* row = kG ? scratch + (size_t)blockIdx.x * (d.Kpad + 2u * d.nch + 1u) : reinterpret_cast<double*>(smem);
  double* T = row + d.Kpad;
  double* CP = T + d.nch;
  __shared__ double s_acc[kLlptWarps];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  for (uint32_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const uint32_t v = d.item_word[item], r0 = d.item_r0[item], r1 = d.item_r1[item];
    __syncthreads();  // the previous item's row is no longer read
    stage_row(d, cur, v, row);
    chunk_prefix(row, d.nch, T, CP);
    const double Qfull = d.alpha * CP[d.nch];
    const double Kalpha = (double)d.K * d.alpha;
    // lane per run: the run's packed D row walked sector by sector (8 entries per 32-byte load,
    // zero padded) with the fp64 products summed in the lane (any order is within the 1e-10
    // the LLPT parity asks: ~nnz ulps)
    double acc = 0.0;
    (void)lane;
    for (uint32_t r = r0 + tid; r < r1; r += blockDim.x) {
      const uint32_t dbase = d.run_dbase[r], len = d.run_len[r];
      const uint32_t hdr = __ldg(d.D + dbase);
      const uint32_t L = hdr >> 16, nnz = hdr & 0xFFFFu;
      const uint32_t* Drow = d.D + dbase + kDHdr;
      double S = 0.0;
      for (uint32_t e0 = 0; e0 < nnz; e0 += 8u) {
        uint4 qa, qb;
        ldg256(Drow + d_at(d.dperm, e0), qa, qb);
        const uint32_t ev[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)  // padding entries are 0: count 0 adds +0
          S = S + u2d(ev[i] & 0xFFFFu) * row[d_topic(ev[i], d.dt)];
      }
      const double p = (S + Qfull) / ((double)L + Kalpha);
      acc = acc + (double)len * log2(p);
    }
    acc = warp_sum(acc);
    if (lane == 0) s_acc[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kLlptWarps; ++w) s = s + s_acc[w];
      partial[item] = s;
    }
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
// Two-branch (ESCA) sampler mode (NEXT-1 of SURVEY 8(f); Eq (3)-(4) P:344-402, Alg
// P:1481-1507, reading #11 of SURVEY 8(c)): the paper's own baseline, with neither the MPT
// skip test nor the K1 split; it runs on the same D rebuild (doc pass without the skip
// test) and W rebuild (item histograms of the new topics).
//   k_tb_prep  block per word: What row (Eq 1-2) and the Q tree prefix
//              QP2(k) = sum_{j<=k} alpha What_j (ascending, fp64, thread 0) in HBM
//   k_tb_draw  warp per doc, lane per token: S = ascending sum over the packed D row of
//              D[d][k] What[v][k], Z = S + Q; the S tree if u <= S / Z with u' = u Z,
//              else the Q tree with u' = (1 - u) Z (the Fig 2 text)
// Every operation is the oracle's, in its order (build flag -fmad=false), so the topics
// are bit-identical without a certification step.  Not tuned: it exists to compare.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_tb_prep(Dev d, Buf cur) {
  const uint32_t v = blockIdx.x;
  double* row = d.tbw + (size_t)v * d.Kpad;
  stage_row(d, cur, v, row);  // ends with __syncthreads: the row is visible block-wide
  if (threadIdx.x == 0) {
    double* q = d.tbq + (size_t)v * d.Kpad;
    double acc = 0.0;
#pragma unroll 8
    for (uint32_t k = 0; k < d.K; ++k) {
      acc = acc + d.alpha * row[k];
      q[k] = acc;
    }
  }
}

__global__ void __launch_bounds__(256) k_tb_draw(Dev d, Buf nxt, uint32_t iter) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t doc = blockIdx.x * 8u + (threadIdx.x >> 5);
  if (doc >= d.Dn) return;
  const uint32_t base = __ldg(d.ddb + doc);
  const uint32_t nnz = __ldg(d.D + base) & 0xFFFFu;
  const uint32_t* E = d.D + base + kDHdr;
  const uint32_t j0 = __ldg(d.dofs + doc), j1 = __ldg(d.dofs + doc + 1);
  for (uint32_t j = j0 + lane; j < j1; j += 32u) {
    const uint32_t v = __ldg(d.tw + j);
    const double* wh = d.tbw + (size_t)v * d.Kpad;
    const double* qp = d.tbq + (size_t)v * d.Kpad;
    double S = 0.0;
    for (uint32_t e = 0; e < nnz; ++e) {
      const uint32_t w = __ldg(E + d_at(d.dperm, e));
      S = S + (double)(w & 0xFFFFu) * __ldg(wh + d_topic(w, d.dt));
    }
    const double Q = __ldg(qp + d.K - 1u);
    const double Z = S + Q;
    const double u = philox_u_k(d.pk, iter, d.token_base + j);
    uint32_t topic = d.K - 1u;
    if (u <= S / Z) {  // S tree: first topic of the row whose prefix exceeds u Z, else the last
      const double up = u * Z;
      double acc = 0.0;
      for (uint32_t e = 0; e < nnz; ++e) {
        const uint32_t w = __ldg(E + d_at(d.dperm, e));
        const uint32_t k = d_topic(w, d.dt);
        acc = acc + (double)(w & 0xFFFFu) * __ldg(wh + k);
        topic = k;
        if (acc > up) break;
      }
    } else {  // Q tree: first k with QP2(k) > (1 - u) Z (QP2 is non-decreasing), else K - 1
      const double up = (1.0 - u) * Z;
      uint32_t a = 0, b = d.K - 1u;
      while (a < b) {
        const uint32_t mid = (a + b) >> 1;
        if (__ldg(qp + mid) > up) b = mid; else a = mid + 1u;
      }
      topic = a;
    }
    nxt.z[j] = (uint16_t)topic;
  }
  if (lane == 0) atomicAdd(&d.ctr->sampled, (unsigned long long)(j1 - j0));
}

// Word-major form (the paper's ESCA layout, K <= kTbItemMaxK): block per work item (word,
// run range): the word's What row and Q prefix in shared memory, thread per (doc, word) run
// (S once per run from the packed D row, then the run's tokens), the new topics into the
// item's histogram and W / n_k rebuilt from it in the same kernel (as the three-branch
// sampler does).  Same operations and orders as k_tb_draw.
__global__ void __launch_bounds__(256) k_tb_item(Dev d, Buf cur, Buf nxt, uint32_t iter) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* wh = reinterpret_cast<double*>(smem);
  double* qp = wh + d.Kpad;
  uint32_t* hist = reinterpret_cast<uint32_t*>(qp + d.Kpad);
  __shared__ uint32_t s_wsum[32], s_run;
  const uint32_t tid = threadIdx.x;
  const uint32_t item = blockIdx.x;
  const uint32_t v = d.item_word[item], r0 = d.item_r0[item], r1 = d.item_r1[item];
  for (uint32_t k = tid; k < d.Kpad; k += blockDim.x) hist[k] = 0;
  stage_row(d, cur, v, wh);  // ends with __syncthreads
  if (tid == 0) {
    double acc = 0.0;
#pragma unroll 8
    for (uint32_t k = 0; k < d.K; ++k) {
      acc = acc + d.alpha * wh[k];
      qp[k] = acc;
    }
  }
  __syncthreads();
  const double Q = qp[d.K - 1u];
  for (uint32_t r = r0 + tid; r < r1; r += blockDim.x) {
    const uint32_t j0 = __ldg(d.run_j0 + r), len = __ldg(d.run_len + r), base = __ldg(d.run_dbase + r);
    const uint32_t nnz = __ldg(d.D + base) & 0xFFFFu;
    const uint32_t* E = d.D + base + kDHdr;
    double S = 0.0;
    for (uint32_t e = 0; e < nnz; ++e) {
      const uint32_t w = __ldg(E + d_at(d.dperm, e));
      S = S + (double)(w & 0xFFFFu) * wh[d_topic(w, d.dt)];
    }
    const double Z = S + Q;
    for (uint32_t t = 0; t < len; ++t) {
      const uint32_t j = j0 + t;
      const double u = philox_u_k(d.pk, iter, d.token_base + j);
      uint32_t topic = d.K - 1u;
      if (u <= S / Z) {
        const double up = u * Z;
        double acc = 0.0;
        for (uint32_t e = 0; e < nnz; ++e) {
          const uint32_t w = __ldg(E + d_at(d.dperm, e));
          const uint32_t k = d_topic(w, d.dt);
          acc = acc + (double)(w & 0xFFFFu) * wh[k];
          topic = k;
          if (acc > up) break;
        }
      } else {
        const double up = (1.0 - u) * Z;
        uint32_t a = 0, b = d.K - 1u;
        while (a < b) {
          const uint32_t mid = (a + b) >> 1;
          if (qp[mid] > up) b = mid; else a = mid + 1u;
        }
        topic = a;
      }
      nxt.z[j] = (uint16_t)topic;
      atomicAdd(&hist[topic], 1u);
    }
  }
  __syncthreads();
  item_epilogue(d, nxt, v, hist, s_wsum, &s_run);
  if (tid == 0) atomicAdd(&d.ctr->sampled, (unsigned long long)d.item_ntok[item]);
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

constexpr size_t kLlptSmemMax = 96u * 1024u;  // larger rows: HBM scratch (k_llpt<true>)
constexpr uint32_t kLlptGrid = 148u * 4u;
size_t llpt_scratch_doubles(uint32_t K) {
  const size_t nch = (K + 31) / 32;
  return kLlptGrid * (nch * 32 + 2 * nch + 1);
}
size_t llpt_smem_bytes(uint32_t K) {  // row | T | CP
  const uint32_t nch = (K + 31) / 32;
  return (size_t)nch * 32 * 8 + (size_t)nch * 8 + (size_t)(nch + 1) * 8;
}
#ifndef EZLDA_SEG_MIN
#define EZLDA_SEG_MIN 16
#endif
// S' segment layout of K: 16-entry segments (two 32-byte sectors per lane and round) with a
// checkpoint per sector (K <= 4096: every row fits one batch of kSegCap segments) or per
// segment (K > 4096: the descent walks two sectors from registers); runs longer than kSegCap x
// 16 nonzeros (large K only) take a fallback with fb-entry segments, fb a power of two with
// K <= kSegCap x fb.
static_assert(kDPermMaxK == kSegCap * 16u, "interleaved D rows iff the <16, 8> sampler kernel (K <= kSegCap x 16)");
void seg_config(uint32_t K, uint32_t* segw, uint32_t* sub, uint32_t* fb) {
  *segw = 16u;
  if (K <= kSegCap * 16u) {
    *segw = EZLDA_SEGW_SMALL;
    *sub = 8u;
    *fb = 0u;
    return;
  }
  *sub = 16u;
  uint32_t w = 32u;
  while (w * kSegCap < K) w <<= 1;
  *fb = w;
}
#ifndef EZLDA_GRP_LARGEK
#define EZLDA_GRP_LARGEK 16  // runs per work claim when K > 4096 (A/B at NYTimes K=5k/10k: 8 55.2/91.7, 16 53.0/90.7, 32 53.9/93.8 ms)
#endif
uint32_t sampler_group_runs(uint32_t K) { return K <= kSegCap * 16u ? 32u : (uint32_t)EZLDA_GRP_LARGEK; }

constexpr size_t kMaxSmem = 227u * 1024u;
// shared-memory layout of the sampler block: kMaxSlots SlotCtl | nslots x (slot head [+ hist])
// | kSampWarpsP x warp scratch.  kMaxSlots (3) slots with the histograms and the Q' table in
// shared memory when they fit, else with the histograms / Q' table in HBM, else fewer slots.
SamplerLayout sampler_layout(uint32_t K) {
  SamplerLayout L{};
  const uint32_t Kpad = (K + 31) / 32 * 32;
  uint32_t segw, sub, fb;
  seg_config(K, &segw, &sub, &fb);
  L.ws_bytes = (sub == 8u ? 2u * kSegCap : kSegCap) * 8u + 4u * kQueue;
  const size_t fixed = sampler_ctl_bytes() + (size_t)kSampWarpsP * L.ws_bytes;
  // prefer layouts that keep EZLDA_SAMP_MINB blocks per SM (the register budget assumes it)
  // with >= 2 slots, the most slots first (A/B: 3 slots vs 2 -- PubMed 77.1 -> 76.0 ms,
  // NYTimes K=5k 60.0 -> 46.0 ms; 4 slots slower); per slot count: histograms and the Q'
  // table in shared memory, else the histograms in HBM scratch, else also the Q' table in
  // HBM; last resort one block per SM
  const size_t budgets[2] = {(228u * 1024u) / EZLDA_SAMP_MINB - 1024u, kMaxSmem};
  for (size_t budget : budgets) {
    // large K (EZLDA_LARGEK_1BLK): one block per SM with more slots rather than two blocks with
    // two -- a block's warps can run at most nslots - 1 items ahead of its slowest warp
    if (EZLDA_LARGEK_1BLK && K > kSegCap * 16u && budget != kMaxSmem) continue;
    for (uint32_t n = kMaxSlots; n >= 1; --n) {
      if (n < 2u && budget != kMaxSmem) break;  // keep >= 2 slots when blocks share the SM
      for (uint32_t mode = 0; mode < 3; ++mode) {
        const uint32_t qg = mode == 2 ? 1u : 0u, hg = mode >= 1 ? 1u : 0u;
        const uint32_t head = slot_head_bytes(Kpad, qg);
        const uint32_t sb = hg ? head : ((head + 4u * (Kpad + Kpad / 32u) + 15u) & ~15u);
        if (fixed + (size_t)n * sb <= budget) {
          L.nslots = n;
          L.hist_global = hg;
          L.qfx_global = qg;
          L.slot_bytes = sb;
          L.smem_bytes = fixed + (size_t)n * sb;
          return L;
        }
      }
    }
  }
  return L;
}
uint32_t sampler_slots(uint32_t K) { return sampler_layout(K).nslots; }
size_t sampler_smem_bytes(uint32_t K) { return sampler_layout(K).smem_bytes; }
size_t wcount_smem_bytes(uint32_t K) { return (size_t)((K + 31) / 32) * 32 * 4; }
static size_t tb_item_smem_bytes(uint32_t K) {
  const size_t Kpad = (K + 31) / 32 * 32;
  return Kpad * 8 * 2 + Kpad * 4;
}
bool two_branch_word_major(uint32_t K) { return tb_item_smem_bytes(K) <= 200u * 1024u; }

size_t doc_block_smem_bytes(uint32_t K) { return (size_t)((K + 31) / 32) * 32 * 4; }

template <uint32_t kFbW, uint32_t kDTs>
static const void* sampler_kernel_fb(uint32_t qg) {
  return qg ? (const void*)k_sampler<16u, 16u, kFbW, kDTs, true> : (const void*)k_sampler<16u, 16u, kFbW, kDTs, false>;
}
static const void* sampler_kernel(uint32_t K, uint32_t qg) {
  uint32_t segw, sub, fb;
  seg_config(K, &segw, &sub, &fb);
  if (fb == 0u)
    return qg ? (const void*)k_sampler<EZLDA_SEGW_SMALL, 8u, 0u, kDTSmall, true>
              : (const void*)k_sampler<EZLDA_SEGW_SMALL, 8u, 0u, kDTSmall, false>;
  switch (fb) {  // K > 4096: fallback segment width 32 .. 256 (K <= 65535)
    case 32u: return sampler_kernel_fb<32u, kDTSmall>(qg);
    case 64u: return sampler_kernel_fb<64u, kDTSmall>(qg);
    case 128u: return sampler_kernel_fb<128u, kDTLarge>(qg);
    default: return sampler_kernel_fb<256u, kDTLarge>(qg);
  }
}

size_t word_prep_smem_bytes(uint32_t K) { return (size_t)kWpWarps * ((K + 31) / 32) * 32 * 8; }  // row per warp

// The dynamic shared-memory limit of a kernel is process-wide state of the device: it is
// only ever RAISED here (to the largest size any live or past handle asked for), so a handle
// with a small K never invalidates the launches of a live handle with a large K.
static std::mutex g_attr_m;
static std::map<std::pair<int, const void*>, int> g_attr;  // (device, kernel) -> limit set

static cudaError_t raise_smem(int dev, const void* k, int bytes) {
  int& cur = g_attr[{dev, k}];
  if (bytes <= cur) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

cudaError_t configure_kernels(uint32_t K, uint32_t* grid) {
  std::lock_guard<std::mutex> lk(g_attr_m);
  cudaError_t e;
#ifdef EZLDA_EXP_FAKEROW
  {
    std::vector<uint32_t> f(1040);
    for (uint32_t i = 0; i < 1040; ++i) f[i] = ((((i * 37u) % 61u) + 16u * (i % 16u)) % K) << 18 | 1u;
    for (uint32_t i = 0; i < 1040; i += 16)  // ascending topics within each 16-entry segment
      std::sort(f.begin() + i, f.begin() + std::min<uint32_t>(i + 16, 1040));
    if ((e = cudaMemcpyToSymbol(g_fake, f.data(), 4 * f.size()))) return e;
  }
#endif
  int dev = 0, nsm = 0, nb = 0;
  if ((e = cudaGetDevice(&dev))) return e;
  if (K <= kWpSmallK && (e = raise_smem(dev, (const void*)k_word_prep_w, (int)word_prep_smem_bytes(K)))) return e;
  const int sp = (int)sampler_smem_bytes(K), db = (int)doc_block_smem_bytes(K);
  if (llpt_smem_bytes(K) <= kLlptSmemMax && (e = raise_smem(dev, (const void*)k_llpt<false>, (int)llpt_smem_bytes(K))))
    return e;
  const void* ks = sampler_kernel(K, sampler_layout(K).qfx_global);
  if ((e = raise_smem(dev, ks, sp))) return e;
  if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev))) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, ks, kSampWarpsP * 32, (size_t)sp))) return e;
  if (nb < 1) return cudaErrorInvalidConfiguration;
  *grid = (uint32_t)(nsm * nb);
  if ((e = raise_smem(dev, (const void*)k_wcount, (int)wcount_smem_bytes(K)))) return e;
  if ((e = raise_smem(dev, (const void*)k_nk, (int)wcount_smem_bytes(K)))) return e;
  if ((e = raise_smem(dev, (const void*)k_tail_rebuild, (int)wcount_smem_bytes(K)))) return e;
  if (two_branch_word_major(K) && (e = raise_smem(dev, (const void*)k_tb_item, (int)tb_item_smem_bytes(K))))
    return e;
  if ((e = raise_smem(dev, (const void*)k_doc_block<false>, db))) return e;
  if ((e = raise_smem(dev, (const void*)k_doc_block<true>, db))) return e;
  if (K <= 4096) {
    const int dh = kDocWarps * (int)doc_hist_stride((K + 31) / 32 * 32) * 4;
    if ((e = raise_smem(dev, (const void*)k_doc_hist<false>, dh))) return e;
    if ((e = raise_smem(dev, (const void*)k_doc_hist<true>, dh))) return e;
    if ((e = raise_smem(dev, (const void*)k_doc_hist<true, false>, dh))) return e;
  }
  return cudaSuccess;
}

void launch_den(const Dev& d, const Buf& cur, cudaStream_t s) {
  k_den<<<(d.K + 255) / 256, 256, 0, s>>>(d, cur);
}

void launch_word_heads(const Dev& d, const Buf& cur, cudaStream_t s) {
  if (d.Vw) k_word_heads<<<(d.Vw + 3u) / 4u, 128, 0, s>>>(d, cur);
}
uint32_t head_bytes(uint32_t K) {  // m | scales | qfx | ce of one word (a multiple of 16 bytes)
  const uint32_t Kpad = (K + 31u) / 32u * 32u;
  return 8u * Kpad + 32u + 4u * ce_words(Kpad);
}

void launch_word_prep(const Dev& d, const Buf& cur, cudaStream_t s) {
  if (d.K <= kWpSmallK) {
    k_word_prep_w<<<(d.V + kWpWarps - 1) / kWpWarps, kWpWarps * 32, word_prep_smem_bytes(d.K), s>>>(d, cur);
  } else {  // dense words: warp per word (256-topic chunks); tail words: thread per word
    if (d.Vd) k_word_prep_big<<<(d.Vd + kWbWarps - 1) / kWbWarps, kWbWarps * 32, 0, s>>>(d, cur);
    if (d.V > d.Vd) k_word_rec_tail<<<(d.V - d.Vd + 127) / 128, 128, 0, s>>>(d, cur);
  }
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
    const size_t smem = (size_t)kDocWarps * doc_hist_stride(d.Kpad) * 4;
    if (skip_test && d.geff <= 2)
      k_doc_hist<true><<<grid, kDocWarps * 32, smem, s>>>(d, cur, nxt, docs_w, n_w, iteration);
    else if (skip_test)
      k_doc_hist<true, false><<<grid, kDocWarps * 32, smem, s>>>(d, cur, nxt, docs_w, n_w, iteration);
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
    {
      const void* ks = sampler_kernel(d.K, d.qfx_global);
      const uint32_t grid = std::min<uint32_t>(n_items, d.sampler_grid);
      void* args[] = {(void*)&d, (void*)&cur, (void*)&nxt, (void*)&iteration, (void*)&n_items};
      cudaLaunchKernel(ks, dim3(grid), dim3(kSampWarpsP * 32), args, sampler_smem_bytes(d.K), s);
    }
}

void launch_item_schedule(const Dev& d, const Buf& nxt, uint32_t n_items, cudaStream_t s) {
  if (n_items) k_item_schedule<<<(n_items + 7) / 8, 256, 0, s>>>(d, nxt, n_items);
}

void launch_two_branch(const Dev& d, const Buf& cur, const Buf& nxt, uint32_t n_items, uint32_t iteration,
                       cudaStream_t s) {
  if (two_branch_word_major(d.K)) {
    if (n_items) k_tb_item<<<n_items, 256, tb_item_smem_bytes(d.K), s>>>(d, cur, nxt, iteration);
    return;
  }
  k_tb_prep<<<d.V, 256, 0, s>>>(d, cur);
  k_tb_draw<<<(d.Dn + 7) / 8, 256, 0, s>>>(d, nxt, iteration);
  if (n_items) k_wcount<<<n_items, 256, wcount_smem_bytes(d.K), s>>>(d, nxt, nxt);
}

void launch_nk(const Dev& d, const Buf& b, cudaStream_t s) {
  k_nk<<<kNkBlocks, 256, 4u * d.Kpad, s>>>(d, b);
}

void launch_tail_rebuild(const Dev& d, const Buf& nxt, const uint16_t* tz_all, const uint32_t* off, uint32_t world,
                         uint64_t tail_max, cudaStream_t s) {
  const uint32_t Vt = d.V - d.Vd;
  if (Vt) k_tail_rebuild<<<Vt, 256, wcount_smem_bytes(d.K), s>>>(d, nxt, tz_all, off, world, tail_max);
}

void launch_llpt(const Dev& d, const Buf& cur, uint32_t n_items, double* partial, double* out, double* scratch,
                 cudaStream_t s) {
  if (n_items && llpt_smem_bytes(d.K) <= kLlptSmemMax)
    k_llpt<false><<<n_items, kLlptWarps * 32, llpt_smem_bytes(d.K), s>>>(d, cur, partial, n_items, nullptr);
  else if (n_items)
    k_llpt<true><<<std::min(n_items, kLlptGrid), kLlptWarps * 32, 0, s>>>(d, cur, partial, n_items, scratch);
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
