// ezlda.cu -- C ABI (include/ezlda.h) and host orchestration of the ezLDA hot path.
//
// create:  inputs -> device; doc-major order (doc, word, input position) by a CUB radix
//          sort; words relabelled by count; (doc, word) runs; word-major run
//          order (the word-sorted token list T of P:845, at run granularity); the
//          sampler's work list with large-word dissection; z^0 from
//          Philox; W^0 / n_k^0.  All on the device except O(V) / O(items) host sorts.
// iterate: den + word-prep -> doc pass -> sampler (+ W all-reduce when world > 1),
//          one stream, no host round trip.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <condition_variable>
#include <cub/cub.cuh>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/ezlda.h"
#include "kernels.h"

using ezl::Buf;
using ezl::Dev;

namespace {

thread_local std::string g_create_error;

// ----------------------------------------------------------------------------
// NCCL, loaded at run time (only when world > 1).
// ----------------------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
      api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
      api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.AllGather && api.CommDestroy &&
               api.GetErrorString && api.GroupStart && api.GroupEnd;
    }
  }
  return api;
}

// ----------------------------------------------------------------------------
// setup kernels
// ----------------------------------------------------------------------------
__global__ void k_max_u32(const uint32_t* a, uint64_t n, uint32_t* out) {
  uint32_t m = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    m = max(m, a[i]);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_max_u16(const uint16_t* a, uint64_t n, uint32_t* out) {
  uint32_t m = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    m = max(m, (uint32_t)a[i]);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// D-row capacity of doc d in words: an 8-word header + min(L_d, K) entries padded to 8
// Sector-interleaved D rows (kernels.h d_phys) when K <= 4096 and the docs are long: every row
// then pays a header line of its own (the entries start on a line), which costs more L2 / DRAM
// than the coalesced phase-B loads save when rows are short (A/B, profiles/r02/ab_dperm.log:
// NYTimes-shaped (332 tokens per doc) sampler 19.8 -> 18.4 ms, PubMed-shaped (90) 73.0 -> 75.0 ms
// with DRAM reads 187 -> 235 GB).  debug_flags force it on / off.
#ifndef EZLDA_DPERM_MIN_MEAN_L
#define EZLDA_DPERM_MIN_MEAN_L 192
#endif
#ifndef EZLDA_POOL
#define EZLDA_POOL 0  // A/B (profiles/r02/ab_dperm.log): create time and e2e within the run-to-run noise either way
#endif
static uint32_t dperm_of(uint32_t K, uint64_t N, uint32_t Dn, uint32_t flags) {
  if (!ezl::kDPermOn || K > ezl::kDPermMaxK || (flags & EZLDA_DEBUG_DPERM_OFF)) return 0u;
  if (flags & EZLDA_DEBUG_DPERM_ON) return 1u;
  return (Dn && N >= (uint64_t)EZLDA_DPERM_MIN_MEAN_L * Dn) ? 1u : 0u;
}
// D-row capacity: an 8-word header + min(L_d, K) entries padded to a multiple of 8 (one 32-byte
// sector per 8 entries); sector-interleaved rows (perm): whole 64-entry blocks, and the header
// sector preceded by 24 unused words so that every row's entries start on a 128-byte line
__global__ void k_rowcap(const uint32_t* L, uint32_t n, uint32_t K, uint32_t perm, uint64_t* cap) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < n) cap[d] = perm ? 32ull + ((min(L[d], K) + 63u) & ~63u) : 8ull + ((min(L[d], K) + 7u) & ~7u);
}
__global__ void k_u64_to_u32(const uint64_t* a, uint32_t n, uint32_t add, uint32_t* b) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (uint32_t)a[i] + add;
}
// doc tiers: 1 iff L_d <= 512 (warp tier) / > 512 (block tier); key of the block tier = L_d
__global__ void k_tier_flags(const uint32_t* L, uint32_t n, uint8_t* fw, uint8_t* fb) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < n) {
    fw[d] = L[d] <= 512u ? 1u : 0u;
    fb[d] = L[d] > 512u ? 1u : 0u;
  }
}
__global__ void k_gather_u32(const uint32_t* src, const uint32_t* idx, uint32_t n, uint32_t* dst) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

// keys / topics of the absent-pair order (positive doubles order like their bit patterns)
__global__ void k_w0_keys(const double* what0, uint32_t K, unsigned long long* key, uint32_t* topic) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < K) {
    key[k] = (unsigned long long)__double_as_longlong(what0[k]);
    topic[k] = k;
  }
}

__global__ void k_hist(const uint32_t* a, uint64_t n, uint32_t* h) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[a[i]], 1u);
}

// sort key (doc << vbits) | word: a stable radix sort over the vbits + dbits significant bits
// gives (doc, original word id, input position) order
__global__ void k_make_keys(const uint32_t* word, const uint32_t* doc, uint32_t n, uint32_t vbits, uint64_t* key,
                            uint32_t* idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    key[i] = ((uint64_t)doc[i] << vbits) | word[i];
    idx[i] = i;
  }
}

// tw[j] = newword[word(j)]; head[j] = 1 iff a (doc, word) run starts at j
__global__ void k_tw_heads(const uint64_t* key, uint32_t n, uint32_t vbits, const uint32_t* newword, uint32_t* tw,
                           uint32_t* head) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) {
    const uint64_t k = key[j];
    tw[j] = newword[(uint32_t)(k & ((1ull << vbits) - 1ull))];
    head[j] = (j == 0 || key[j - 1] != k) ? 1u : 0u;
  }
}

// per doc-major run q (qidx = inclusive scan of heads - 1)
__global__ void k_run_heads(const uint64_t* key, const uint32_t* head, const uint32_t* qinc, const uint32_t* tw,
                            uint32_t n, uint32_t vbits, uint32_t* q_j0, uint32_t* q_v, uint32_t* q_doc) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n && head[j]) {
    const uint32_t q = qinc[j] - 1;
    q_j0[q] = j;
    q_v[q] = tw[j];
    q_doc[q] = (uint32_t)(key[j] >> vbits);
  }
}

__global__ void k_iota(uint32_t* a, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

// word-major run tables from the sorted run permutation
__global__ void k_run_tables(const uint32_t* rperm, uint32_t R, uint32_t N, const uint32_t* q_j0, const uint32_t* q_doc,
                             const uint32_t* ddb, uint32_t* run_j0, uint32_t* run_dbase, uint16_t* run_len,
                             uint32_t* len32, uint32_t* rid_of_q) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) {
    const uint32_t q = rperm[r];
    const uint32_t j0 = q_j0[q];
    const uint32_t j1 = (q + 1 < R) ? q_j0[q + 1] : N;
    const uint32_t d = q_doc[q];
    run_j0[r] = j0;
    run_dbase[r] = ddb[d];
    run_len[r] = (uint16_t)(j1 - j0);
    len32[r] = j1 - j0;
    rid_of_q[q] = r;
  }
}

// (word, run id) of every doc-major token, packed for one 8-byte load in the doc pass
__global__ void k_twr(const uint32_t* qinc, const uint32_t* rid_of_q, const uint32_t* tw, uint32_t n, uint2* twr) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) twr[j] = make_uint2(tw[j], rid_of_q[qinc[j] - 1]);
}

// wrun[v] = first run of word v (lower bound in the sorted run words), v in [0, V]
__global__ void k_wrun(const uint32_t* vs, uint32_t R, uint32_t V, uint32_t* wrun) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v <= V) {
    uint32_t lo = 0, hi = R;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (vs[mid] < v) lo = mid + 1; else hi = mid;
    }
    wrun[v] = lo;
  }
}

// item heads: first run of each word; for dense words also region boundaries every `split`
// tokens and, for hot words (>= cut_min tokens), doc-window boundaries
// (run_dbase / blk_words changes)
__global__ void k_item_heads(const uint32_t* vs, const uint32_t* wrun, const uint32_t* tokpre,
                             const uint32_t* run_dbase, uint32_t R, uint32_t Vd, uint32_t split, uint32_t blk_words,
                             uint32_t cut_min, uint32_t* head) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) {
    const uint32_t v = vs[r];
    const uint32_t first = wrun[v];
    uint32_t h = (r == first);
    if (!h && v < Vd) {
      const uint32_t b = tokpre[first];
      h = ((tokpre[r] - b) / split) != ((tokpre[r - 1] - b) / split);
      if (tokpre[wrun[v + 1]] - b >= cut_min) h |= (run_dbase[r] / blk_words) != (run_dbase[r - 1] / blk_words);
    }
    head[r] = h;
  }
}

__global__ void k_items(const uint32_t* r0s, uint32_t NI, uint32_t R, const uint32_t* vs, const uint32_t* tokpre,
                        const uint32_t* run_dbase, uint32_t blk_words, uint32_t* item5) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < NI) {
    const uint32_t r0 = r0s[i];
    const uint32_t r1 = (i + 1 < NI) ? r0s[i + 1] : R;
    item5[5 * i + 0] = vs[r0];
    item5[5 * i + 1] = r0;
    item5[5 * i + 2] = r1;
    item5[5 * i + 3] = tokpre[r1] - tokpre[r0];
    item5[5 * i + 4] = run_dbase[r0] / blk_words;
  }
}

// word-major run order key: relabelled word; the stable sort keeps doc order within a word,
// so concurrently running items sweep the D rows in the same (ascending) direction -- the L2
// temporal locality the sampler relies on (measured: ordering runs by doc length instead cost
// 1.7x on PubMed)

inline unsigned blocks(uint64_t n, unsigned t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

// ----------------------------------------------------------------------------
// the handle
// ----------------------------------------------------------------------------
struct ezlda {
  void* lgroup = nullptr;  // LocalGroup* of the in-process rank group (options.local_group), else NCCL
  uint64_t lgroup_key = 0;
  bool multi = false;      // multi-rank path: world > 1, or a one-rank NCCL group (world == 1 + nccl id)
  Dev dev{};
  Buf buf[2]{};
  int cur = 0;
  std::vector<void*> allocs;  // device allocations owned by the handle
  uint64_t N = 0;
  uint32_t Dn = 0, V = 0, K = 0, R = 0, Vd = 0, Vt = 0;
  uint32_t n_items = 0, n_docs_w = 0, n_docs_b = 0;
  uint64_t tail_cap = 0;
  uint64_t Dwords = 0;
  uint32_t dperm = 0;                 // sector-interleaved D rows (dperm_of)
  uint32_t cut_min = 0;
  double alpha = 0, beta = 0;
  uint64_t seed = 0;
  uint32_t g = 2;
  int rank = 0, world = 1;
  uint64_t N_global = 0;
  // tail-W exchange (world > 1): every rank all-gathers the new topics of its
  // tail-word tokens in word-major order; each rank rebuilds the global tail rows from them
  uint32_t rt0 = 0;                 // first word-major run of a tail word
  uint64_t tail_max = 0;            // max over ranks of the local tail-token count (gather slot)
  uint16_t* tz_local = nullptr;     // [tail_max] this rank's tail topics, word-major
  uint16_t* tz_all = nullptr;       // [world * tail_max] gathered
  uint32_t* tail_run_tok = nullptr; // [R - rt0] word-major offset of a tail run's tokens in tz_local
  uint32_t* tail_off = nullptr;     // [world * (Vt + 1)] per-rank prefix of local tail counts
  double exchange_bytes = 0;        // collective payload of the last exchange
  // dense-block deltas (world > 1): this rank's local counts of the last exchange, the packed
  // 16-bit deltas, and a device flag "some |delta| does not fit"
  int32_t* wloc_prev = nullptr;     // [Vd * K]
  uint32_t* wpack = nullptr;        // [ceil(Vd * K / 2)]
  int32_t* wover = nullptr;         // [1]
  bool wloc_valid = false;          // wloc_prev holds the local counts of the previous exchange
  uint64_t delta_exchanges = 0;     // exchanges that took the packed path (diagnostics)
  uint32_t* docs_w = nullptr;
  uint32_t* docs_b = nullptr;
  uint32_t* perm = nullptr;
  std::vector<uint32_t> newword, origword;  // orig -> relabelled, relabelled -> orig
  uint32_t iteration = 0;
  bool D_fresh = false;  // D rows describe buf[cur].z
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool timing = true;
  // per-iteration records (events + pinned counter copies), folded lazily into stats
  static constexpr int kSlots = 256;
  struct Slot {
    cudaEvent_t ev[7];  // start | word records | doc pass | schedule | heads | sampler | end
    uint32_t iteration;
    uint32_t launches;
  };
  std::vector<Slot> slots;
  std::vector<int> pending;  // FIFO of slot indices not yet folded
  uint64_t slot_counter = 0;
  ezl::Counters* ctr_host = nullptr;  // pinned, kSlots entries
  uint32_t exact_all = 0;             // options.exact_draws
  uint32_t branches = 3;              // options.sampler (2: two-branch ESCA mode)
  uint32_t debug_flags = 0;           // options.debug_flags (EZLDA_DEBUG_*)
  uint32_t schedule = 0;              // options.schedule
  // H4 per-iteration schedule: CUB select of the live items (static order preserved)
  uint32_t* item_iota = nullptr;
  uint32_t* item_act = nullptr;
  unsigned long long *w0_key_in = nullptr, *w0_key_out = nullptr;  // absent-pair order (large K)
  uint32_t* w0_top_in = nullptr;
  unsigned char* w0_tmp = nullptr;
  size_t w0_tmp_bytes = 0;
  uint32_t* n_act = nullptr;
  void* sel_tmp = nullptr;
  size_t sel_tmp_bytes = 0;
  ezlda_iter_stats sum{};
  uint32_t sum_n = 0;
  double* llpt_partial = nullptr;
  double* llpt_out = nullptr;
  double* llpt_scratch = nullptr;  // large K: per-block fp64 rows of the LLPT kernel (lazily allocated)
  ncclComm_t comm = nullptr;
  ezlda_status sticky = EZLDA_OK;
  std::string err;
  ezlda_iter_stats last{};

  ezlda_status fail(ezlda_status s, const char* fmt, ...) {
    char b[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(b, sizeof b, fmt, ap);
    va_end(ap);
    err = b;
    if (s == EZLDA_E_CUDA || s == EZLDA_E_NCCL) sticky = s;
    return s;
  }

  // Optional (EZLDA_POOL build switch, off): device memory from a private stream-ordered pool,
  // so that create's many GB of transients are reused instead of mapped and unmapped by
  // cudaMalloc / cudaFree; trimmed when create ends, destroyed with the handle.  Measured within
  // the (large) run-to-run noise of create, so the default stays cudaMalloc.
  cudaMemPool_t pool = nullptr;
  template <typename T>
  T* alloc(size_t n) {
    void* p = nullptr;
    const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
    if (pool) {
      if (cudaMallocFromPoolAsync(&p, bytes, pool, stream) != cudaSuccess) return nullptr;
    } else if (cudaMalloc(&p, bytes) != cudaSuccess) {
      return nullptr;
    }
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  void release(void* p) {
    auto it = std::find(allocs.begin(), allocs.end(), p);
    if (it != allocs.end()) {
      if (pool) cudaFreeAsync(p, stream); else cudaFree(p);
      allocs.erase(it);
    }
  }

};

#define EZ_CUDA(h, call)                                                                                   \
  do {                                                                                                     \
    cudaError_t e_ = (call);                                                                               \
    if (e_ != cudaSuccess) return (h)->fail(EZLDA_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,       \
                                            cudaGetErrorString(e_));                                       \
  } while (0)
#define EZ_ALLOC(h, ptr, T, n)                                                                             \
  do {                                                                                                     \
    (ptr) = (h)->alloc<T>(n);                                                                              \
    if (!(ptr)) return (h)->fail(EZLDA_E_NOMEM, "cudaMalloc of %zu x %zu bytes failed (%s)", (size_t)(n),  \
                                 sizeof(T), #ptr);                                                         \
  } while (0)
#define EZ_NCCL(h, call)                                                                                   \
  do {                                                                                                     \
    ncclResult_t r_ = (call);                                                                              \
    if (r_ != ncclSuccess) return (h)->fail(EZLDA_E_NCCL, "%s: %s", #call, nccl().GetErrorString(r_));     \
  } while (0)

namespace {

// CUB wrappers (setup only)
template <typename F>
ezlda_status cub_call(ezlda* h, F f) {
  size_t bytes = 0;
  if (f(nullptr, bytes) != cudaSuccess) return h->fail(EZLDA_E_CUDA, "cub size query failed");
  void* tmp = h->alloc<unsigned char>(bytes);
  if (!tmp) return h->fail(EZLDA_E_NOMEM, "cub temp alloc");
  cudaError_t e = f(tmp, bytes);
  h->release(tmp);
  if (e != cudaSuccess) return h->fail(EZLDA_E_CUDA, "cub call failed: %s", cudaGetErrorString(e));
  return EZLDA_OK;
}

// ---- in-process rank group (options.local_group != 0; test hook): the ranks are handles of
// one process on one device, each driven by its own host thread; the all-reduce is a sum of
// the ranks' device buffers in rank order (integer sums are exact, so W is bit-identical to
// the NCCL path).  Everything else of the multi-rank path (relabelling from global counts,
// all-dense W, token bases, doc shards) runs unchanged, so it can be tested on one GPU.
struct LocalGroup {
  std::mutex m;
  std::condition_variable cv;
  int world = 0, arrived = 0, members = 0;
  uint64_t gen = 0;
  bool broken = false;  // a barrier timed out: every later barrier fails at once
  std::vector<const void*> bufs;
};
std::mutex g_groups_m;
std::map<uint64_t, LocalGroup*> g_groups;

// Join the group of `key` (created by its first member with `world` ranks); nullptr if the
// key already names a group with a different world.
LocalGroup* local_group_join(uint64_t key, int world) {
  std::lock_guard<std::mutex> lk(g_groups_m);
  LocalGroup*& g = g_groups[key];
  if (!g) {
    g = new LocalGroup();
    g->world = world;
    g->bufs.assign(world, nullptr);
  } else if (g->world != world) {
    return nullptr;
  }
  g->members += 1;
  return g;
}

// Leave the group; the last member frees it (the key can then be reused with any world).
void local_group_leave(uint64_t key) {
  std::lock_guard<std::mutex> lk(g_groups_m);
  auto it = g_groups.find(key);
  if (it == g_groups.end()) return;
  if (--it->second->members == 0) {
    delete it->second;
    g_groups.erase(it);
  }
}

template <typename T>
__global__ void k_sum_ranks(const T* const* src, int n, size_t count, T* dst) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    T acc = src[0][i];
    for (int r = 1; r < n; ++r) acc = acc + src[r][i];
    dst[i] = acc;
  }
}

// Barrier of the group.  A rank that failed never arrives: the others give up after 600 s
// (and the group is marked broken) instead of blocking forever.
bool group_barrier(LocalGroup* g) {
  std::unique_lock<std::mutex> lk(g->m);
  if (g->broken) return false;
  const uint64_t my = g->gen;
  if (++g->arrived == g->world) {
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
    return true;
  }
  if (!g->cv.wait_for(lk, std::chrono::seconds(600), [&] { return g->gen != my || g->broken; }) || g->broken) {
    g->broken = true;
    g->cv.notify_all();
    return false;
  }
  return true;
}

ezlda_status local_allreduce(ezlda* h, void* buf, size_t count, ncclDataType_t dt) {
  LocalGroup* g = static_cast<LocalGroup*>(h->lgroup);
  const size_t esz = (dt == ncclInt32 || dt == ncclUint32) ? 4 : 8;
  EZ_CUDA(h, cudaStreamSynchronize(h->stream));
  {
    std::lock_guard<std::mutex> lk(g->m);
    g->bufs[h->rank] = buf;
  }
  if (!group_barrier(g)) return h->fail(EZLDA_E_STATE, "local group barrier timed out (a rank failed)");
  void* tmp = nullptr;
  const size_t src_off = (count * esz + 15) & ~(size_t)15;  // the pointer table 16-byte aligned
  EZ_CUDA(h, cudaMalloc(&tmp, src_off + sizeof(void*) * g->world));
  const void** d_src = reinterpret_cast<const void**>(static_cast<char*>(tmp) + src_off);
  EZ_CUDA(h, cudaMemcpyAsync(d_src, g->bufs.data(), sizeof(void*) * g->world, cudaMemcpyHostToDevice, h->stream));
  const unsigned nb = (unsigned)std::min<size_t>((count + 255) / 256, 4096);
  if (dt == ncclInt32)
    k_sum_ranks<int32_t><<<nb, 256, 0, h->stream>>>(reinterpret_cast<const int32_t* const*>(d_src), g->world, count,
                                                     static_cast<int32_t*>(tmp));
  else if (dt == ncclUint32)
    k_sum_ranks<uint32_t><<<nb, 256, 0, h->stream>>>(reinterpret_cast<const uint32_t* const*>(d_src), g->world, count,
                                                      static_cast<uint32_t*>(tmp));
  else if (dt == ncclUint64)
    k_sum_ranks<unsigned long long><<<nb, 256, 0, h->stream>>>(
        reinterpret_cast<const unsigned long long* const*>(d_src), g->world, count,
        static_cast<unsigned long long*>(tmp));
  else
    k_sum_ranks<double><<<nb, 256, 0, h->stream>>>(reinterpret_cast<const double* const*>(d_src), g->world, count,
                                                   static_cast<double*>(tmp));
  EZ_CUDA(h, cudaStreamSynchronize(h->stream));
  if (!group_barrier(g)) return h->fail(EZLDA_E_STATE, "local group barrier timed out (a rank failed)");
  EZ_CUDA(h, cudaMemcpyAsync(buf, tmp, count * esz, cudaMemcpyDeviceToDevice, h->stream));
  EZ_CUDA(h, cudaStreamSynchronize(h->stream));
  cudaFree(tmp);
  return EZLDA_OK;
}

ezlda_status allreduce(ezlda* h, void* buf, size_t count, ncclDataType_t dt) {
  if (!h->multi || count == 0) return EZLDA_OK;
  if (h->lgroup) return local_allreduce(h, buf, count, dt);
  EZ_NCCL(h, nccl().AllReduce(buf, buf, count, dt, ncclSum, h->comm, h->stream));
  return EZLDA_OK;
}

ezlda_status local_allgather(ezlda* h, const void* send, void* recv, size_t bytes) {
  LocalGroup* g = static_cast<LocalGroup*>(h->lgroup);
  EZ_CUDA(h, cudaStreamSynchronize(h->stream));
  {
    std::lock_guard<std::mutex> lk(g->m);
    g->bufs[h->rank] = send;
  }
  if (!group_barrier(g)) return h->fail(EZLDA_E_STATE, "local group barrier timed out (a rank failed)");
  for (int r = 0; r < g->world; ++r)
    if (bytes)
      EZ_CUDA(h, cudaMemcpyAsync(static_cast<char*>(recv) + (size_t)r * bytes, g->bufs[r], bytes,
                                 cudaMemcpyDeviceToDevice, h->stream));
  EZ_CUDA(h, cudaStreamSynchronize(h->stream));
  if (!group_barrier(g)) return h->fail(EZLDA_E_STATE, "local group barrier timed out (a rank failed)");
  return EZLDA_OK;
}

// recv[r * bytes .. (r + 1) * bytes) = rank r's send (device buffers, every rank the same size)
ezlda_status allgather(ezlda* h, const void* send, void* recv, size_t bytes) {
  if (!h->multi) return EZLDA_OK;
  if (h->lgroup) return local_allgather(h, send, recv, bytes);
  if (bytes) EZ_NCCL(h, nccl().AllGather(send, recv, bytes, ncclUint8, h->comm, h->stream));
  return EZLDA_OK;
}

// word-major copy of the tail tokens' topics: run r (a tail word's run) -> tz[tail_run_tok[r]..]
__global__ void k_tail_gather(const uint32_t* run_j0, const uint16_t* run_len, const uint32_t* run_tok, uint32_t rt0,
                              uint32_t R, const uint16_t* z, uint16_t* tz) {
  const uint32_t r = rt0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) {
    const uint32_t j0 = run_j0[r], n = run_len[r], o = run_tok[r - rt0];
    for (uint32_t t = 0; t < n; ++t) tz[o + t] = z[j0 + t];
  }
}

__global__ void k_tail_run_tok(const uint32_t* tokpre, uint32_t rt0, uint32_t R, uint32_t* out) {
  const uint32_t r = rt0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) out[r - rt0] = tokpre[r] - tokpre[rt0];
}

// Dense-block deltas (SURVEY 8(e) "int16 deltas with an overflow guard").  delta = local -
// prev (this rank's local counts now vs at the last exchange), packed two per u32 as 16-bit
// fields delta + b, b = 32768 / world: every term lies in [1, 2b - 1] when |delta| < b, so the
// u32 sum over the ranks of each field stays below 2^16 and never carries into its neighbour.
// prev <- local.  *over is set if some |delta| >= b (then the exchange takes the int32 path).
__global__ void k_wdelta_pack(const int32_t* loc, int32_t* prev, size_t n, int32_t b, uint32_t* pack, int32_t* over) {
  bool bad = false;
  const size_t np = (n + 1) / 2;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < np; i += (size_t)gridDim.x * blockDim.x) {
    const size_t e = 2 * i;
    const int32_t l0 = loc[e], l1 = (e + 1 < n) ? loc[e + 1] : 0;
    const int32_t d0 = l0 - prev[e], d1 = (e + 1 < n) ? l1 - prev[e + 1] : 0;
    bad |= (d0 >= b || d0 <= -b || d1 >= b || d1 <= -b);
    pack[i] = (uint32_t)(d0 + b) | ((uint32_t)(d1 + b) << 16);
    prev[e] = l0;
    if (e + 1 < n) prev[e + 1] = l1;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31u) == 0) atomicOr(over, 1);
}
// out = gprev + (sum over ranks of the packed fields) - world * b
__global__ void k_wdelta_apply(const int32_t* gprev, const uint32_t* sum, size_t n, int32_t wb, int32_t* out) {
  const size_t np = (n + 1) / 2;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < np; i += (size_t)gridDim.x * blockDim.x) {
    const size_t e = 2 * i;
    const uint32_t v = sum[i];
    out[e] = gprev[e] + ((int32_t)(v & 0xFFFFu) - wb);
    if (e + 1 < n) out[e + 1] = gprev[e + 1] + ((int32_t)(v >> 16) - wb);
  }
}

// H7 (world > 1): the W merge.  The tail tokens' topics are gathered word-major
// (k_tail_gather); the int32 all-reduce of the dense block and the u16 all-gather of the tail
// topics are issued as ONE NCCL group, so the two collectives run concurrently; then every
// rank rebuilds the global packed tail rows (integer sums: W is identical on every rank).
// The dense block goes as packed 16-bit deltas against the previous global W (gprev, the
// other buffer) when every rank's deltas fit (one int32 all-reduce of the overflow flags
// decides), else as the int32 local counts; gprev == nullptr forces the int32 path.
ezlda_status exchange_w(ezlda* h, Buf& b, const Buf* gprev) {
  if (!h->multi) return EZLDA_OK;
  const bool tail = h->Vt != 0;
  const size_t dn = (size_t)h->Vd * h->K;
  const int32_t bias = 32768 / h->world;
  bool delta = false;
  if (dn && h->wpack) {  // always refresh wloc_prev; the packed deltas are usable iff it was valid
    const bool want = gprev && h->wloc_valid && !(h->debug_flags & EZLDA_DEBUG_NO_W_DELTA);
    EZ_CUDA(h, cudaMemsetAsync(h->wover, 0, 4, h->stream));
    const unsigned nb = (unsigned)std::min<size_t>(((dn + 1) / 2 + 255) / 256, 148u * 16u);
    k_wdelta_pack<<<nb, 256, 0, h->stream>>>(b.Wd, h->wloc_prev, dn, bias, h->wpack, h->wover);
    EZ_CUDA(h, cudaGetLastError());
    h->wloc_valid = true;
    if (want) {
      ezlda_status st0 = allreduce(h, h->wover, 1, ncclInt32);
      if (st0) return st0;
      int32_t over = 1;
      EZ_CUDA(h, cudaMemcpyAsync(&over, h->wover, 4, cudaMemcpyDeviceToHost, h->stream));
      EZ_CUDA(h, cudaStreamSynchronize(h->stream));
      delta = over == 0;
    }
  }
  void* dbuf = delta ? (void*)h->wpack : (void*)b.Wd;
  const size_t dcount = delta ? (dn + 1) / 2 : dn;
  const ncclDataType_t dtype = delta ? ncclUint32 : ncclInt32;
  if (tail && h->R > h->rt0) {
    k_tail_gather<<<(unsigned)((h->R - h->rt0 + 255) / 256), 256, 0, h->stream>>>(
        h->dev.run_j0, h->dev.run_len, h->tail_run_tok, h->rt0, h->R, b.z, h->tz_local);
    EZ_CUDA(h, cudaGetLastError());
  }
  const size_t tbytes = tail ? 2ull * h->tail_max : 0;
  ezlda_status st;
  if (h->lgroup) {  // in-process test hook: the same sums / concatenation, one after the other
    if ((st = allreduce(h, dbuf, dcount, dtype))) return st;
    if (tail && (st = allgather(h, h->tz_local, h->tz_all, tbytes))) return st;
  } else {
    EZ_NCCL(h, nccl().GroupStart());
    if (dcount) EZ_NCCL(h, nccl().AllReduce(dbuf, dbuf, dcount, dtype, ncclSum, h->comm, h->stream));
    if (tbytes) EZ_NCCL(h, nccl().AllGather(h->tz_local, h->tz_all, tbytes, ncclUint8, h->comm, h->stream));
    EZ_NCCL(h, nccl().GroupEnd());
  }
  if (delta) {
    const unsigned nb = (unsigned)std::min<size_t>(((dn + 1) / 2 + 255) / 256, 148u * 16u);
    k_wdelta_apply<<<nb, 256, 0, h->stream>>>(gprev->Wd, h->wpack, dn, bias * h->world, b.Wd);
    EZ_CUDA(h, cudaGetLastError());
    ++h->delta_exchanges;
  }
  h->exchange_bytes = 4.0 * (double)dcount + (double)h->world * (double)tbytes;
  if (tail) {
    ezl::launch_tail_rebuild(h->dev, b, h->tz_all, h->tail_off, (uint32_t)h->world, h->tail_max, h->stream);
    EZ_CUDA(h, cudaGetLastError());
  }
  return EZLDA_OK;
}

void fill_dev(ezlda* h) {
  Dev& d = h->dev;
  d.N = (uint32_t)h->N;
  d.Dn = h->Dn;
  d.V = h->V;
  d.K = h->K;
  d.nch = (h->K + 31) / 32;
  d.Kpad = d.nch * 32;
  d.Vd = h->Vd;
  ezl::seg_config(h->K, &d.segw, &d.segsub, &d.segfb);
  d.dt = ezl::d_shift(h->K);
  d.dperm = h->dperm;
  d.grp = ezl::sampler_group_runs(h->K);
  d.zmark = h->K <= 32768u ? 1u : 0u;
  d.c1_cap = (h->debug_flags & EZLDA_DEBUG_C1_LOOKUP) ? 0u : 0x7FFFu;
  {
    const ezl::SamplerLayout L = ezl::sampler_layout(h->K);
    d.nslots = L.nslots;
    d.hist_global = L.hist_global;
    d.qfx_global = L.qfx_global;
    d.hist_bitmap = h->K >= 2048u ? 1u : 0u;
    d.slot_bytes = L.slot_bytes;
    d.ws_bytes = L.ws_bytes;
  }
  d.exact_all = h->exact_all;
  d.branches = h->branches;
  d.geff = std::min<uint32_t>(h->g, h->K - 1);
  d.alpha = h->alpha;
  d.beta = h->beta;
  d.Vbeta = (double)h->V * h->beta;
  d.seed = h->seed;
  d.pk = ezl::philox_keys(h->seed);
}

// W^cur and n_k^cur from buf[cur].z (init / set_topics), + all-reduce
ezlda_status rebuild_counts(ezlda* h) {
  Buf& b = h->buf[h->cur];
  EZ_CUDA(h, cudaMemsetAsync(b.Wd, 0, sizeof(int32_t) * (size_t)h->Vd * h->K, h->stream));
  EZ_CUDA(h, cudaMemsetAsync(b.nk, 0, sizeof(int32_t) * h->K, h->stream));
  EZ_CUDA(h, cudaMemsetAsync(b.tnnz, 0, sizeof(uint32_t) * std::max<uint32_t>(h->Vt, 1), h->stream));
  EZ_CUDA(h, cudaMemsetAsync(h->dev.ctr, 0, sizeof(ezl::Counters), h->stream));
  ezl::launch_sampler(h->dev, b, b, h->n_items, 0, true, h->stream);
  EZ_CUDA(h, cudaGetLastError());
  ezlda_status s;
  if ((s = exchange_w(h, b, nullptr))) return s;  // int32 path (no previous exchange to delta against)
  ezl::launch_nk(h->dev, b, h->stream);  // n_k of the global W (identical on every rank)
  EZ_CUDA(h, cudaGetLastError());
  h->D_fresh = false;
  return EZLDA_OK;
}

ezlda_status ensure_D(ezlda* h) {
  if (h->D_fresh) return EZLDA_OK;
  Buf& b = h->buf[h->cur];
  ezl::launch_doc_pass(h->dev, b, b, h->docs_w, h->n_docs_w, h->docs_b, h->n_docs_b, h->iteration, false, h->stream);
  EZ_CUDA(h, cudaGetLastError());
  h->D_fresh = true;
  return EZLDA_OK;
}

ezlda_status do_create(ezlda* h, const uint32_t* word_ids, const uint32_t* doc_ids, const ezlda_options& o) {
  // EZLDA_CREATE_TIMING=1: per-phase wall time of create on stderr (stream synchronized at each mark)
  static const bool s_tm = std::getenv("EZLDA_CREATE_TIMING") != nullptr;
  auto t_prev = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!s_tm) return;
    cudaStreamSynchronize(h->stream);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ezlda create] %-40s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t - t_prev).count());
    t_prev = t;
  };
  const uint32_t N = (uint32_t)h->N;
  cudaStream_t s = h->stream;
  mark("before: inputs on device");
  // ---- inputs on device
  uint32_t *d_word, *d_doc;
  EZ_ALLOC(h, d_word, uint32_t, N);
  EZ_ALLOC(h, d_doc, uint32_t, N);
  const cudaMemcpyKind kind = o.input_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  EZ_CUDA(h, cudaMemcpyAsync(d_word, word_ids, sizeof(uint32_t) * N, kind, s));
  EZ_CUDA(h, cudaMemcpyAsync(d_doc, doc_ids, sizeof(uint32_t) * N, kind, s));
  mark("before: validate ids");
  // ---- validate ids
  uint32_t* d_max;
  EZ_ALLOC(h, d_max, uint32_t, 2);
  EZ_CUDA(h, cudaMemsetAsync(d_max, 0, 8, s));
  k_max_u32<<<1184, 256, 0, s>>>(d_word, N, d_max);
  k_max_u32<<<1184, 256, 0, s>>>(d_doc, N, d_max + 1);
  uint32_t mx[2];
  EZ_CUDA(h, cudaMemcpyAsync(mx, d_max, 8, cudaMemcpyDeviceToHost, s));
  EZ_CUDA(h, cudaStreamSynchronize(s));
  if (mx[0] >= h->V) return h->fail(EZLDA_E_INVALID, "word id %u >= V = %u", mx[0], h->V);
  if (mx[1] >= h->Dn) return h->fail(EZLDA_E_INVALID, "doc id %u >= n_docs = %u", mx[1], h->Dn);
  mark("before: doc lengths, word counts");
  // ---- doc lengths, word counts
  // (all per-doc tables are built on the device: doc offsets and D-row bases by scans, the
  // doc tiers by selections; only the V word counts come to the host, for the relabelling)
  uint32_t *d_L, *d_cnt, *d_dofs, *d_ddb;
  uint64_t *d_cap, *d_ddb64;
  EZ_ALLOC(h, d_L, uint32_t, h->Dn + 1);
  EZ_ALLOC(h, d_cnt, uint32_t, h->V);
  EZ_CUDA(h, cudaMemsetAsync(d_L, 0, sizeof(uint32_t) * (h->Dn + 1), s));
  EZ_CUDA(h, cudaMemsetAsync(d_cnt, 0, sizeof(uint32_t) * h->V, s));
  k_hist<<<2368, 256, 0, s>>>(d_doc, N, d_L);
  k_hist<<<2368, 256, 0, s>>>(d_word, N, d_cnt);
  std::vector<uint32_t> cnt_local(h->V);
  EZ_CUDA(h, cudaMemcpyAsync(cnt_local.data(), d_cnt, sizeof(uint32_t) * h->V, cudaMemcpyDeviceToHost, s));
  EZ_CUDA(h, cudaMemsetAsync(d_max, 0, 4, s));
  k_max_u32<<<1184, 256, 0, s>>>(d_L, h->Dn, d_max);
  // doc offsets (exclusive scan of L over Dn + 1 entries: dofs[Dn] = N) and D-row bases: an
  // 8-word header + min(L_d, K) entries padded to a multiple of 8 (one 32-byte sector per 8
  // entries; rows start sector aligned)
  EZ_ALLOC(h, d_dofs, uint32_t, h->Dn + 1);
  EZ_ALLOC(h, d_cap, uint64_t, h->Dn + 1);
  EZ_ALLOC(h, d_ddb64, uint64_t, h->Dn + 1);
  EZ_ALLOC(h, d_ddb, uint32_t, h->Dn);
  EZ_CUDA(h, cudaMemsetAsync(d_cap + h->Dn, 0, 8, s));
  const uint32_t dperm = dperm_of(h->K, N, h->Dn, h->debug_flags);
  h->dperm = dperm;
  k_rowcap<<<blocks(h->Dn), 256, 0, s>>>(d_L, h->Dn, h->K, dperm, d_cap);
  {
    ezlda_status st0 = cub_call(h, [&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, d_L, d_dofs, (int)(h->Dn + 1), s);
    });
    if (st0) return st0;
    st0 = cub_call(h, [&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, d_cap, d_ddb64, (int)(h->Dn + 1), s);
    });
    if (st0) return st0;
  }
  // (perm: bases 24 mod 32 words, so that the entries after the 8-word header start on a line)
  k_u64_to_u32<<<blocks(h->Dn), 256, 0, s>>>(d_ddb64, h->Dn, dperm ? 24u : 0u, d_ddb);
  uint64_t dwords = 0;
  uint32_t maxL = 0;
  EZ_CUDA(h, cudaMemcpyAsync(&dwords, d_ddb64 + h->Dn, 8, cudaMemcpyDeviceToHost, s));
  EZ_CUDA(h, cudaMemcpyAsync(&maxL, d_max, 4, cudaMemcpyDeviceToHost, s));
  EZ_CUDA(h, cudaStreamSynchronize(s));
  h->release(d_cap);
  h->release(d_ddb64);
  if (maxL > 65535) return h->fail(EZLDA_E_RANGE, "a doc has %u tokens (> 65535, P:753)", maxL);
  if (dwords + 24u >= (1ull << 32)) return h->fail(EZLDA_E_RANGE, "D storage >= 2^32 words per shard");
  h->Dwords = dwords + (dperm ? 24u : 0u);
  // global word counts (the dense/tail split and relabelling must agree on all ranks)
  std::vector<uint64_t> cnt(h->V);
  for (uint32_t v = 0; v < h->V; ++v) cnt[v] = cnt_local[v];
  if (h->multi) {
    uint64_t* d_c64;
    EZ_ALLOC(h, d_c64, uint64_t, h->V);
    EZ_CUDA(h, cudaMemcpyAsync(d_c64, cnt.data(), sizeof(uint64_t) * h->V, cudaMemcpyHostToDevice, s));
    ezlda_status st = allreduce(h, d_c64, h->V, ncclUint64);
    if (st) return st;
    EZ_CUDA(h, cudaMemcpyAsync(cnt.data(), d_c64, sizeof(uint64_t) * h->V, cudaMemcpyDeviceToHost, s));
    uint64_t nl = N, ng = 0;
    uint64_t* d_n;
    EZ_ALLOC(h, d_n, uint64_t, 1);
    EZ_CUDA(h, cudaMemcpyAsync(d_n, &nl, 8, cudaMemcpyHostToDevice, s));
    if ((st = allreduce(h, d_n, 1, ncclUint64))) return st;
    EZ_CUDA(h, cudaMemcpyAsync(&ng, d_n, 8, cudaMemcpyDeviceToHost, s));
    EZ_CUDA(h, cudaStreamSynchronize(s));
    h->N_global = ng;
    h->release(d_c64);
    h->release(d_n);
  } else {
    h->N_global = N;
  }
  mark("before: relabel words by count desc, ties by");
  // ---- relabel words by count desc, ties by id
  h->origword.resize(h->V);
  std::iota(h->origword.begin(), h->origword.end(), 0u);
  std::stable_sort(h->origword.begin(), h->origword.end(),
                   [&](uint32_t a, uint32_t b) { return cnt[a] > cnt[b]; });
  h->newword.resize(h->V);
  for (uint32_t i = 0; i < h->V; ++i) h->newword[h->origword[i]] = i;
  // dense iff c_v > threshold ("larger than the topic number"); counts > 65535 must be dense
  // (words are sorted by count, so the dense set is a prefix of the relabelled ids)
  uint64_t thr = o.dense_threshold ? o.dense_threshold : h->K;
  if (o.w_mode == EZLDA_W_ALL_SPARSE) thr = 65535;  // tail counts must fit 16 bits
  uint32_t Vd = 0;
  while (Vd < h->V && (cnt[h->origword[Vd]] > thr || cnt[h->origword[Vd]] > 65535)) ++Vd;
  if (o.w_mode == EZLDA_W_ALL_DENSE) Vd = h->V;
  h->Vd = Vd;
  h->Vt = h->V - Vd;
  std::vector<uint32_t> tofs(h->Vt + 1, 0);
  for (uint32_t t = 0; t < h->Vt; ++t)
    tofs[t + 1] = tofs[t] + (uint32_t)std::min<uint64_t>(cnt[h->origword[Vd + t]], h->K);
  h->tail_cap = tofs[h->Vt];
  std::vector<uint32_t> wtok(h->V + 1, 0);
  for (uint32_t v = 0; v < h->V; ++v) wtok[v + 1] = wtok[v] + cnt_local[h->origword[v]];
  mark("before: doc-major order: sort (doc, word, in");
  // ---- doc-major order: sort (doc, word, input position)
  uint64_t *k_in, *k_out;
  uint32_t *i_in, *i_out;
  EZ_ALLOC(h, k_in, uint64_t, N);
  EZ_ALLOC(h, k_out, uint64_t, N);
  EZ_ALLOC(h, i_in, uint32_t, N);
  EZ_ALLOC(h, i_out, uint32_t, N);
  int dbits = 1, vbits = 1;
  while (dbits < 32 && ((h->Dn - 1) >> dbits)) ++dbits;
  while (vbits < 32 && ((h->V - 1) >> vbits)) ++vbits;
  k_make_keys<<<blocks(N), 256, 0, s>>>(d_word, d_doc, N, (uint32_t)vbits, k_in, i_in);
  ezlda_status st;
  st = cub_call(h, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, k_in, k_out, i_in, i_out, (int)N, 0, vbits + dbits, s);
  });
  if (st) return st;
  h->release(k_in);
  h->release(i_in);
  h->release(d_word);
  h->release(d_doc);
  h->perm = i_out;
  mark("before: relabelled word per token, run heads");
  // ---- relabelled word per token, run heads
  uint32_t *d_newword, *tw, *head, *qinc;
  EZ_ALLOC(h, d_newword, uint32_t, h->V);
  EZ_CUDA(h, cudaMemcpyAsync(d_newword, h->newword.data(), sizeof(uint32_t) * h->V, cudaMemcpyHostToDevice, s));
  EZ_ALLOC(h, tw, uint32_t, N);
  EZ_ALLOC(h, head, uint32_t, N);
  EZ_ALLOC(h, qinc, uint32_t, N);
  k_tw_heads<<<blocks(N), 256, 0, s>>>(k_out, N, (uint32_t)vbits, d_newword, tw, head);
  st = cub_call(h, [&](void* t, size_t& b) { return cub::DeviceScan::InclusiveSum(t, b, head, qinc, (int)N, s); });
  if (st) return st;
  uint32_t R = 0;
  EZ_CUDA(h, cudaMemcpyAsync(&R, qinc + N - 1, 4, cudaMemcpyDeviceToHost, s));
  EZ_CUDA(h, cudaStreamSynchronize(s));
  h->R = R;
  uint32_t *q_j0, *q_v, *q_doc;
  EZ_ALLOC(h, q_j0, uint32_t, R);
  EZ_ALLOC(h, q_v, uint32_t, R);
  EZ_ALLOC(h, q_doc, uint32_t, R);
  k_run_heads<<<blocks(N), 256, 0, s>>>(k_out, head, qinc, tw, N, (uint32_t)vbits, q_j0, q_v, q_doc);
  h->release(k_out);
  h->release(head);
  mark("before: word-major run order (stable by word");
  // ---- word-major run order (stable by word => docs ascending within a word)
  // (the relabelled word is the key: a stable radix sort over its vbits bits keeps the runs of a
  // word in doc-major order)
  uint32_t *q_iota, *rperm, *vs;
  EZ_ALLOC(h, q_iota, uint32_t, R);
  EZ_ALLOC(h, rperm, uint32_t, R);
  EZ_ALLOC(h, vs, uint32_t, R);
  k_iota<<<blocks(R), 256, 0, s>>>(q_iota, R);
  st = cub_call(h, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, q_v, vs, q_iota, rperm, (int)R, 0, vbits, s);
  });
  if (st) return st;
  h->release(q_iota);
  h->release(q_v);
  uint32_t *run_j0, *run_dbase, *len32, *rid_of_q;
  uint2* twr;
  uint16_t* run_len;
  EZ_ALLOC(h, run_j0, uint32_t, R);
  EZ_ALLOC(h, run_dbase, uint32_t, R);
  EZ_ALLOC(h, run_len, uint16_t, R);
  EZ_ALLOC(h, len32, uint32_t, R + 1);
  EZ_ALLOC(h, rid_of_q, uint32_t, R);
  k_run_tables<<<blocks(R), 256, 0, s>>>(rperm, R, N, q_j0, q_doc, d_ddb, run_j0, run_dbase, run_len, len32, rid_of_q);
  h->release(q_j0);
  h->release(q_doc);
  h->release(rperm);
  EZ_ALLOC(h, twr, uint2, N);
  k_twr<<<blocks(N), 256, 0, s>>>(qinc, rid_of_q, tw, N, twr);
  h->release(qinc);
  h->release(rid_of_q);
  mark("before: items: per word, split dense words e");
  // ---- items: per word, split dense words every split_threshold tokens
  uint32_t *wrun, *tokpre, *ihead, *r_iota, *r0s, *d_ni;
  EZ_ALLOC(h, wrun, uint32_t, h->V + 1);
  k_wrun<<<blocks(h->V + 1), 256, 0, s>>>(vs, R, h->V, wrun);
  EZ_ALLOC(h, tokpre, uint32_t, R + 1);
  EZ_CUDA(h, cudaMemsetAsync(len32 + R, 0, 4, s));
  st = cub_call(h, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, len32, tokpre, (int)(R + 1), s); });
  if (st) return st;
  h->release(len32);
  const uint32_t split = (o.schedule == 2) ? 0xFFFFFFFFu : (o.split_threshold ? o.split_threshold : 10000u);
  EZ_ALLOC(h, ihead, uint32_t, R);
  // L2 doc windows of doc_block_kb KiB of D rows (0 = 32 MiB): the items of hot words (at
  // least EZLDA_WIN_TOK tokens per window on average) are cut at window boundaries and run
  // window-major, heavy first -- every D row of the window is then read by many items
  // while it is L2 resident; the other words' items (too few runs per window to amortise
  // the staged What' row) run uncut after them
  const uint64_t blk_kb = (o.schedule == 2) ? 0xFFFFFFFFull : (o.doc_block_kb ? o.doc_block_kb : 32768ull);
  const uint32_t blk_words = (uint32_t)std::min<uint64_t>(blk_kb * 256ull, 0xFFFFFFFFull);
  const uint64_t nwin = (h->Dwords + blk_words - 1) / blk_words;
#ifndef EZLDA_WIN_TOK
#define EZLDA_WIN_TOK 512  // window-cut only words with >= 512 tokens per D window on average (A/B: 256 .. 16384)
#endif
  const uint32_t cut_min = (uint32_t)std::min<uint64_t>((uint64_t)EZLDA_WIN_TOK * nwin, 0xFFFFFFFFull);
  h->cut_min = cut_min;
  k_item_heads<<<blocks(R), 256, 0, s>>>(vs, wrun, tokpre, run_dbase, R, h->Vd, split, blk_words, cut_min, ihead);
  EZ_ALLOC(h, r_iota, uint32_t, R);
  EZ_ALLOC(h, r0s, uint32_t, R);
  EZ_ALLOC(h, d_ni, uint32_t, 1);
  k_iota<<<blocks(R), 256, 0, s>>>(r_iota, R);
  st = cub_call(h, [&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, r_iota, ihead, r0s, d_ni, (int)R, s);
  });
  if (st) return st;
  uint32_t NI = 0;
  EZ_CUDA(h, cudaMemcpyAsync(&NI, d_ni, 4, cudaMemcpyDeviceToHost, s));
  EZ_CUDA(h, cudaStreamSynchronize(s));
  h->release(r_iota);
  h->release(ihead);
  uint32_t* item5;
  EZ_ALLOC(h, item5, uint32_t, 5ull * NI);
  k_items<<<blocks(NI), 256, 0, s>>>(r0s, NI, R, vs, tokpre, run_dbase, blk_words, item5);
  std::vector<uint32_t> it5(5ull * NI);
  EZ_CUDA(h, cudaMemcpyAsync(it5.data(), item5, sizeof(uint32_t) * 5ull * NI, cudaMemcpyDeviceToHost, s));
  EZ_CUDA(h, cudaStreamSynchronize(s));
  h->release(item5);
  h->release(r0s);
  h->release(d_ni);
  h->release(vs);
  if (h->multi && h->Vt) {  mark("before: tail-W exchange layout (static): wor");
  // ---- tail-W exchange layout (static): word-major tail runs, per-rank counts
    EZ_CUDA(h, cudaMemcpyAsync(&h->rt0, wrun + h->Vd, 4, cudaMemcpyDeviceToHost, s));
    EZ_CUDA(h, cudaStreamSynchronize(s));
    EZ_ALLOC(h, h->tail_run_tok, uint32_t, std::max<uint32_t>(R - h->rt0, 1));
    if (R > h->rt0) k_tail_run_tok<<<blocks(R - h->rt0), 256, 0, s>>>(tokpre, h->rt0, R, h->tail_run_tok);
    std::vector<uint32_t> tc(h->Vt), tc_all((size_t)h->world * h->Vt);
    for (uint32_t t = 0; t < h->Vt; ++t) tc[t] = cnt_local[h->origword[h->Vd + t]];
    uint32_t *d_tc, *d_tc_all;
    EZ_ALLOC(h, d_tc, uint32_t, h->Vt);
    EZ_ALLOC(h, d_tc_all, uint32_t, (size_t)h->world * h->Vt);
    EZ_CUDA(h, cudaMemcpyAsync(d_tc, tc.data(), 4ull * h->Vt, cudaMemcpyHostToDevice, s));
    if ((st = allgather(h, d_tc, d_tc_all, 4ull * h->Vt))) return st;
    EZ_CUDA(h, cudaMemcpyAsync(tc_all.data(), d_tc_all, 4ull * h->world * h->Vt, cudaMemcpyDeviceToHost, s));
    EZ_CUDA(h, cudaStreamSynchronize(s));
    h->release(d_tc);
    h->release(d_tc_all);
    std::vector<uint32_t> off((size_t)h->world * (h->Vt + 1));
    h->tail_max = 1;
    for (int r = 0; r < h->world; ++r) {
      uint64_t acc = 0;
      for (uint32_t t = 0; t < h->Vt; ++t) {
        off[(size_t)r * (h->Vt + 1) + t] = (uint32_t)acc;
        acc += tc_all[(size_t)r * h->Vt + t];
      }
      off[(size_t)r * (h->Vt + 1) + h->Vt] = (uint32_t)acc;
      h->tail_max = std::max<uint64_t>(h->tail_max, acc);
    }
    EZ_ALLOC(h, h->tail_off, uint32_t, off.size());
    EZ_CUDA(h, cudaMemcpyAsync(h->tail_off, off.data(), 4ull * off.size(), cudaMemcpyHostToDevice, s));
    EZ_ALLOC(h, h->tz_local, uint16_t, h->tail_max);
    EZ_ALLOC(h, h->tz_all, uint16_t, (size_t)h->world * h->tail_max);
    EZ_CUDA(h, cudaStreamSynchronize(s));
  }
  if (h->multi) h->exchange_bytes = 4.0 * (double)h->Vd * h->K + 2.0 * h->world * (h->Vt ? h->tail_max : 0);
  if (h->multi && (size_t)h->Vd * h->K) {
    const size_t dn = (size_t)h->Vd * h->K;
    EZ_ALLOC(h, h->wloc_prev, int32_t, dn);
    EZ_ALLOC(h, h->wpack, uint32_t, (dn + 1) / 2);
    EZ_ALLOC(h, h->wover, int32_t, 1);
  }
  h->release(tokpre);
  h->release(wrun);
  // order: hot-word items window-major, heavy first within a window; then the other items
  // heavy first; the hardware block scheduler balances the tail
  std::vector<uint32_t> order(NI);
  std::iota(order.begin(), order.end(), 0u);
  auto key = [&](uint32_t a) {
    const uint32_t v = it5[5 * a];
    const uint64_t cold = (v >= h->Vd || cnt_local[h->origword[v]] < cut_min) ? 1u : 0u;
    const uint64_t blk = cold ? 0u : it5[5 * a + 4];
    return (cold << 63) | (blk << 32) | (uint64_t)(0xFFFFFFFFu - it5[5 * a + 3]);
  };
  if (o.schedule != 2)  // schedule 2 (ablation): items stay in word order
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return key(a) < key(b); });
  std::vector<uint32_t> iw(NI), ir0(NI), ir1(NI), int_(NI);
  for (uint32_t i = 0; i < NI; ++i) {
    const uint32_t q = order[i];
    iw[i] = it5[5 * q];
    ir0[i] = it5[5 * q + 1];
    ir1[i] = it5[5 * q + 2];
    int_[i] = it5[5 * q + 3];
  }
  h->n_items = NI;
  uint32_t *item_word, *item_r0, *item_r1, *item_ntok;
  EZ_ALLOC(h, item_word, uint32_t, NI);
  EZ_ALLOC(h, item_r0, uint32_t, NI);
  EZ_ALLOC(h, item_r1, uint32_t, NI);
  EZ_ALLOC(h, item_ntok, uint32_t, NI);
  EZ_CUDA(h, cudaMemcpyAsync(item_word, iw.data(), 4ull * NI, cudaMemcpyHostToDevice, s));
  EZ_CUDA(h, cudaMemcpyAsync(item_r0, ir0.data(), 4ull * NI, cudaMemcpyHostToDevice, s));
  EZ_CUDA(h, cudaMemcpyAsync(item_r1, ir1.data(), 4ull * NI, cudaMemcpyHostToDevice, s));
  EZ_CUDA(h, cudaMemcpyAsync(item_ntok, int_.data(), 4ull * NI, cudaMemcpyHostToDevice, s));
  mark("before: doc tiers (static: L_d does not chan");
  // ---- doc tiers (static: L_d does not change)
  // warp tier: docs with L_d <= 512 in doc order; block tier: the others by L_d descending
  // (stable: ties in doc order)
  {
    uint8_t *fw, *fb;
    uint32_t *d_iota, *d_nsel, *b_unsorted, *b_key, *b_key_sorted;
    EZ_ALLOC(h, fw, uint8_t, h->Dn);
    EZ_ALLOC(h, fb, uint8_t, h->Dn);
    EZ_ALLOC(h, d_iota, uint32_t, h->Dn);
    EZ_ALLOC(h, d_nsel, uint32_t, 2);
    EZ_ALLOC(h, h->docs_w, uint32_t, h->Dn);
    EZ_ALLOC(h, b_unsorted, uint32_t, h->Dn);
    k_tier_flags<<<blocks(h->Dn), 256, 0, s>>>(d_L, h->Dn, fw, fb);
    k_iota<<<blocks(h->Dn), 256, 0, s>>>(d_iota, h->Dn);
    ezlda_status st1 = cub_call(h, [&](void* t, size_t& b) {
      return cub::DeviceSelect::Flagged(t, b, d_iota, fw, h->docs_w, d_nsel, (int)h->Dn, s);
    });
    if (st1) return st1;
    st1 = cub_call(h, [&](void* t, size_t& b) {
      return cub::DeviceSelect::Flagged(t, b, d_iota, fb, b_unsorted, d_nsel + 1, (int)h->Dn, s);
    });
    if (st1) return st1;
    uint32_t nsel[2];
    EZ_CUDA(h, cudaMemcpyAsync(nsel, d_nsel, 8, cudaMemcpyDeviceToHost, s));
    EZ_CUDA(h, cudaStreamSynchronize(s));
    h->n_docs_w = nsel[0];
    h->n_docs_b = nsel[1];
    EZ_ALLOC(h, h->docs_b, uint32_t, std::max<uint32_t>(nsel[1], 1));
    if (nsel[1]) {
      EZ_ALLOC(h, b_key, uint32_t, nsel[1]);
      EZ_ALLOC(h, b_key_sorted, uint32_t, nsel[1]);
      k_gather_u32<<<blocks(nsel[1]), 256, 0, s>>>(d_L, b_unsorted, nsel[1], b_key);
      st1 = cub_call(h, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairsDescending(t, b, b_key, b_key_sorted, b_unsorted, h->docs_b,
                                                         (int)nsel[1], 0, 16, s);
      });
      if (st1) return st1;
      h->release(b_key);
      h->release(b_key_sorted);
    }
    h->release(fw);
    h->release(fb);
    h->release(d_iota);
    h->release(d_nsel);
    h->release(b_unsorted);
  }
  mark("before: remaining state");
  // ---- remaining state
  uint32_t *d_tofs, *d_wtok;
  EZ_ALLOC(h, d_tofs, uint32_t, h->Vt + 1);
  EZ_ALLOC(h, d_wtok, uint32_t, h->V + 1);
  EZ_CUDA(h, cudaMemcpyAsync(d_tofs, tofs.data(), 4ull * (h->Vt + 1), cudaMemcpyHostToDevice, s));
  EZ_CUDA(h, cudaMemcpyAsync(d_wtok, wtok.data(), 4ull * (h->V + 1), cudaMemcpyHostToDevice, s));
  Dev& d = h->dev;
  fill_dev(h);
  d.dofs = d_dofs;
  d.ddb = d_ddb;
  d.tw = tw;
  d.twr = twr;
  d.run_j0 = run_j0;
  d.run_dbase = run_dbase;
  d.run_len = run_len;
  d.tofs = d_tofs;
  d.wtok = d_wtok;
  d.item_word = item_word;
  d.item_r0 = item_r0;
  d.item_r1 = item_r1;
  d.item_ntok = item_ntok;
  if (h->schedule == 0 && h->branches == 3 && NI) {  // H4: per-iteration list of the live items
    EZ_ALLOC(h, h->item_iota, uint32_t, NI);
    EZ_ALLOC(h, h->item_act, uint32_t, NI);
    EZ_ALLOC(h, h->n_act, uint32_t, 1);
    EZ_ALLOC(h, d.item_live, uint8_t, NI);
    k_iota<<<blocks(NI), 256, 0, s>>>(h->item_iota, NI);
    h->sel_tmp_bytes = 0;
    EZ_CUDA(h, cub::DeviceSelect::Flagged(nullptr, h->sel_tmp_bytes, h->item_iota, d.item_live, h->item_act, h->n_act,
                                          (int)NI, s));
    EZ_ALLOC(h, h->sel_tmp, unsigned char, std::max<size_t>(h->sel_tmp_bytes, 1));
    d.item_act = h->item_act;
    d.n_act = h->n_act;
  }
  EZ_ALLOC(h, d.D, uint32_t, h->Dwords);
  EZ_ALLOC(h, d.flags, uint32_t, (R + 31) / 32);
  EZ_ALLOC(h, d.rec, ezl::WordRec, h->V);
  EZ_ALLOC(h, d.recm, ezl::WordRecM, h->V);
  EZ_ALLOC(h, d.reck, uint32_t, h->V);
  EZ_ALLOC(h, d.qexact, double, (size_t)h->V * d.nch);
  // sampler heads (8 Kpad + 32 + ce bytes per word) for every word when they fit in the free
  // device memory less a reserve (a quarter of it, at least 8 GiB, for the per-iteration
  // scratch), else for the dense words only (the other items are staged by a sampler warp, which
  // costs O(K) on the sampler's critical path per item)
  d.rs_bytes = ezl::head_bytes(h->K);
  if (h->branches == 3) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) fr = 0;
    const uint64_t reserve = std::max<uint64_t>(8ull << 30, fr / 4);
    const uint64_t budget = fr > reserve ? fr - reserve : 0;
    d.Vw = ((uint64_t)h->V * d.rs_bytes <= budget) ? h->V : h->Vd;
    if (o.debug_flags & EZLDA_DEBUG_NO_TAIL_ROWS) d.Vw = h->Vd;  // tail rows staged by a sampler warp
  }
  EZ_ALLOC(h, d.wrow, unsigned char, (size_t)d.Vw * d.rs_bytes);
  if (h->item_act) EZ_ALLOC(h, d.word_live, uint8_t, h->V);
  if (h->branches == 2 && !ezl::two_branch_word_major(h->K)) {
    EZ_ALLOC(h, d.tbw, double, (size_t)h->V * d.Kpad);
    EZ_ALLOC(h, d.tbq, double, (size_t)h->V * d.Kpad);
  }
  EZ_ALLOC(h, d.den, double, h->K);
  EZ_ALLOC(h, d.what0, double, h->K);
  EZ_ALLOC(h, d.inv_den, double, h->K);
  if (h->K > 4096u && h->Vt && h->branches == 3) {  // absent-pair order of the tail records
    EZ_ALLOC(h, d.w0ord, uint32_t, h->K);
    EZ_ALLOC(h, d.twv, double, std::max<uint64_t>(h->tail_cap, 1));  // What of the tail nonzeros
    EZ_ALLOC(h, h->w0_key_in, unsigned long long, h->K);
    EZ_ALLOC(h, h->w0_key_out, unsigned long long, h->K);
    EZ_ALLOC(h, h->w0_top_in, uint32_t, h->K);
    h->w0_tmp_bytes = 0;
    EZ_CUDA(h, cub::DeviceRadixSort::SortPairsDescending(nullptr, h->w0_tmp_bytes, h->w0_key_in, h->w0_key_out,
                                                         h->w0_top_in, d.w0ord, (int)h->K, 0, 64, s));
    EZ_ALLOC(h, h->w0_tmp, unsigned char, std::max<size_t>(h->w0_tmp_bytes, 1));
  }
  EZ_ALLOC(h, d.ctr, ezl::Counters, 1);
  for (int b = 0; b < 2; ++b) {
    Buf& B = h->buf[b];
    EZ_ALLOC(h, B.z, uint16_t, N);
    EZ_ALLOC(h, B.Wd, int32_t, (size_t)h->Vd * h->K);
    EZ_ALLOC(h, B.Wt, uint32_t, h->tail_cap);
    // (ezlda_counts copies the whole capacity; entries past tnnz are never read but stay defined)
    if (h->tail_cap) EZ_CUDA(h, cudaMemsetAsync(B.Wt, 0, sizeof(uint32_t) * h->tail_cap, s));
    EZ_ALLOC(h, B.tnnz, uint32_t, std::max<uint32_t>(h->Vt, 1));
    EZ_ALLOC(h, B.nk, int32_t, h->K);
  }
  EZ_CUDA(h, cudaMemsetAsync(d.rec, 0, sizeof(ezl::WordRec) * h->V, s));
  EZ_CUDA(h, cudaMemsetAsync(d.recm, 0, sizeof(ezl::WordRecM) * h->V, s));
  EZ_CUDA(h, cudaMemsetAsync(d.reck, 0, sizeof(uint32_t) * h->V, s));
  EZ_ALLOC(h, h->llpt_partial, double, std::max<uint32_t>(NI, 1));
  EZ_ALLOC(h, h->llpt_out, double, 1);
  EZ_CUDA(h, cudaMallocHost(&h->ctr_host, sizeof(ezl::Counters) * ezlda::kSlots));
  memset(h->ctr_host, 0, sizeof(ezl::Counters) * ezlda::kSlots);
  h->slots.resize(ezlda::kSlots);
  for (auto& sl : h->slots)
    for (auto& e : sl.ev) EZ_CUDA(h, cudaEventCreate(&e));
  h->release(d_newword);
  h->release(d_L);
  h->release(d_cnt);
  h->release(d_max);
  EZ_CUDA(h, ezl::configure_kernels(h->K, &d.sampler_grid));
  {  // per-(sampler block, slot) scratch: HBM histograms and fixed-point Q' tables (large K)
    const size_t nh = (size_t)d.sampler_grid * d.nslots * (d.Kpad + d.Kpad / 32);  // counts + bitmap
    EZ_ALLOC(h, d.hist_scratch, uint32_t, nh);
    EZ_CUDA(h, cudaMemsetAsync(d.hist_scratch, 0, nh * sizeof(uint32_t), s));
    if (d.qfx_global) EZ_ALLOC(h, d.qfx_scratch, uint32_t, (size_t)d.sampler_grid * d.nslots * d.Kpad);
  }
  mark("before: iteration 0");
  // ---- iteration 0
  h->cur = 0;
  ezl::launch_init_topics(d, h->buf[0].z, s);
  EZ_CUDA(h, cudaGetLastError());
  if ((st = rebuild_counts(h))) return st;
  EZ_CUDA(h, cudaStreamSynchronize(s));
  mark("end (iteration 0)");
  h->iteration = 0;
  return EZLDA_OK;
}

// Fold the oldest pending iteration record into `last` and `sum`.
ezlda_status fold_one(ezlda* h) {
  const int si = h->pending.front();
  h->pending.erase(h->pending.begin());
  ezlda::Slot& sl = h->slots[si];
  EZ_CUDA(h, cudaEventSynchronize(sl.ev[4]));
  ezlda_iter_stats st{};
  const ezl::Counters& c = h->ctr_host[si];
  st.iteration = sl.iteration;
  st.n_tokens = h->N;
  st.skip_S = c.skip_S;
  st.skip_final = c.skip_S + c.skip_M;
  st.sampled = c.sampled;
  st.active_runs = c.active_runs;
  st.drow_words = c.drow_words;
  st.d_nnz = c.d_nnz;
  st.kernel_launches = sl.launches;
  st.exact_redraws = c.exact;
  st.exchange_bytes = h->exchange_bytes;
  if (h->timing) {
    float a = 0, b = 0, cc = 0, dd = 0;
    float e25 = 0, e56 = 0, e63 = 0;
    EZ_CUDA(h, cudaEventElapsedTime(&a, sl.ev[0], sl.ev[1]));
    EZ_CUDA(h, cudaEventElapsedTime(&b, sl.ev[1], sl.ev[2]));
    EZ_CUDA(h, cudaEventElapsedTime(&e25, sl.ev[2], sl.ev[5]));
    EZ_CUDA(h, cudaEventElapsedTime(&e56, sl.ev[5], sl.ev[6]));
    EZ_CUDA(h, cudaEventElapsedTime(&e63, sl.ev[6], sl.ev[3]));
    EZ_CUDA(h, cudaEventElapsedTime(&dd, sl.ev[3], sl.ev[4]));
    a += e56;           // word-prep = word records + the sampler heads of the live words
    cc = e25 + e63;     // sampling = schedule + sampler + n_k
    st.ms_sampler_kernel = e63;
    st.ms_wordprep = a;
    st.ms_docpass = b;
    st.ms_sample = cc;
    st.ms_allreduce = dd;
    st.ms_total = (double)a + b + cc + dd;
  }
  // DESIGN.md byte model (algorithmic bytes at payload granularity):
  //   doc pass: per token z read 2 + tw 4 ; skipped token z write 2 ; failing token trid 4 ;
  //             D rows written 4 (nnz + 4) per doc
  //   sampler:  per active run 10 B of run table + D row 4 (nnz + 1) ; sampled token z write 2 ;
  //             per armed (live) item its word's W row (4 B x K)
  //   word-prep: W rows read 4 B x Vd K (+ tail), W rebuilt 4 B x Vd K
  const double N = (double)h->N;
  const double tok_fail = N - (double)c.skip_S;
  st.model_bytes_docpass = N * (2.0 + 4.0) + (double)c.skip_S * 2.0 + tok_fail * 4.0 +
                           4.0 * ((double)c.d_nnz + 4.0 * h->Dn);
  st.model_bytes_sample = (double)c.active_runs * 10.0 + 4.0 * (double)c.drow_words + (double)c.sampled * 2.0 +
                          (double)(h->branches == 2 ? (unsigned long long)h->n_items : c.items) * 4.0 * h->K;
  st.model_bytes = st.model_bytes_docpass + st.model_bytes_sample + 2.0 * 4.0 * (double)h->Vd * h->K;
  h->last = st;
  ezlda_iter_stats& S = h->sum;
  S.ms_total += st.ms_total;
  S.ms_wordprep += st.ms_wordprep;
  S.ms_docpass += st.ms_docpass;
  S.ms_sample += st.ms_sample;
  S.ms_sampler_kernel += st.ms_sampler_kernel;
  S.ms_allreduce += st.ms_allreduce;
  S.n_tokens += st.n_tokens;
  S.skip_S += st.skip_S;
  S.skip_final += st.skip_final;
  S.sampled += st.sampled;
  S.active_runs += st.active_runs;
  S.drow_words += st.drow_words;
  S.d_nnz += st.d_nnz;
  S.model_bytes += st.model_bytes;
  S.model_bytes_sample += st.model_bytes_sample;
  S.model_bytes_docpass += st.model_bytes_docpass;
  S.kernel_launches += st.kernel_launches;
  S.exact_redraws += st.exact_redraws;
  S.exchange_bytes += st.exchange_bytes;
  h->sum_n += 1;
  return EZLDA_OK;
}

ezlda_status fold_all(ezlda* h) {
  while (!h->pending.empty()) {
    ezlda_status st = fold_one(h);
    if (st) return st;
  }
  return EZLDA_OK;
}

}  // namespace

// ----------------------------------------------------------------------------
// C ABI
// ----------------------------------------------------------------------------
extern "C" {

ezlda_status ezlda_create(const uint32_t* word_ids, const uint32_t* doc_ids, uint64_t n_tokens, uint32_t n_docs,
                          uint32_t V, uint32_t K, double alpha, double beta, uint64_t seed,
                          const ezlda_options* opts, ezlda** out) {
  g_create_error.clear();
  if (out) *out = nullptr;
  auto bad = [&](ezlda_status s, const char* m) {
    g_create_error = m;
    return s;
  };
  if (!out || !word_ids || !doc_ids) return bad(EZLDA_E_INVALID, "NULL argument");
  if (n_tokens == 0 || K == 0 || V == 0 || n_docs == 0) return bad(EZLDA_E_INVALID, "n_tokens, K, V and n_docs must be > 0");
  if (!(alpha > 0.0) || !(beta > 0.0)) return bad(EZLDA_E_INVALID, "alpha and beta must be > 0");
  if (K > 65535) return bad(EZLDA_E_RANGE, "K > 65535 (16-bit topic packing, P:753)");
  if (ezl::sampler_slots(K) == 0)
    return bad(EZLDA_E_RANGE, "K too large for the sampler's shared-memory slot (fixed-point What' row of 4 K bytes)");
  // the setup sorts and scans (CUB) index the shard's tokens with int
  if (n_tokens >= (1ull << 31)) return bad(EZLDA_E_RANGE, "n_tokens >= 2^31 per shard");
  ezlda_options o{};
  if (opts) {  // struct_size versioning: a smaller (older) struct leaves the new fields zero
    const size_t n = opts->struct_size ? std::min<size_t>(opts->struct_size, sizeof(o)) : sizeof(o);
    std::memcpy(&o, opts, n);
  }
  if (o.g > 3) return bad(EZLDA_E_INVALID, "g must be in {1,2,3} (0 = default 2)");
  if (o.w_mode > 2) return bad(EZLDA_E_INVALID, "unknown w_mode");
  if (o.sampler != 0 && o.sampler != 2 && o.sampler != 3)
    return bad(EZLDA_E_INVALID, "sampler must be 0/3 (three-branch) or 2 (two-branch)");
  if (o.schedule > 2) return bad(EZLDA_E_INVALID, "schedule must be 0, 1 or 2");
  ezlda* h = new (std::nothrow) ezlda();
  if (!h) return bad(EZLDA_E_NOMEM, "host allocation failed");
  h->N = n_tokens;
  h->Dn = n_docs;
  h->V = V;
  h->K = K;
  h->alpha = alpha;
  h->beta = beta;
  h->seed = seed;
  h->g = o.g ? o.g : 2;
  h->rank = o.rank;
  h->world = o.world > 1 ? o.world : 1;
  h->multi = o.world > 1 || (o.world == 1 && o.nccl_unique_id != nullptr);
  h->timing = !o.no_phase_timing;
  h->exact_all = o.exact_draws ? 1u : 0u;
  h->branches = o.sampler ? o.sampler : 3u;
  h->debug_flags = o.debug_flags;
  h->schedule = o.schedule;
  h->dev.token_base = o.token_base;
  ezlda_status st = EZLDA_OK;
  if (o.stream) {
    h->stream = (cudaStream_t)o.stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
      g_create_error = "cudaStreamCreate failed (no CUDA device?)";
      delete h;
      return EZLDA_E_CUDA;
    }
    h->own_stream = true;
  }
#if EZLDA_POOL
  {
    int dev = 0;
    cudaMemPoolProps pp{};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.location.type = cudaMemLocationTypeDevice;
    if (cudaGetDevice(&dev) == cudaSuccess) pp.location.id = dev;
    if (cudaMemPoolCreate(&h->pool, &pp) == cudaSuccess) {
      uint64_t keep = ~0ull;  // freed blocks stay in the pool (reused by later allocations of create)
      cudaMemPoolSetAttribute(h->pool, cudaMemPoolAttrReleaseThreshold, &keep);
    } else {
      h->pool = nullptr;
      cudaGetLastError();
    }
  }
#endif
  if (h->multi && o.local_group) {
    if (o.rank < 0 || o.rank >= h->world) st = h->fail(EZLDA_E_INVALID, "local_group needs 0 <= rank < world");
    else if (!(h->lgroup = local_group_join(o.local_group, h->world)))
      st = h->fail(EZLDA_E_INVALID, "local_group key %llu is in use with a different world",
                   (unsigned long long)o.local_group);
    else h->lgroup_key = o.local_group;
  } else if (h->multi) {
    if (!o.nccl_unique_id || o.rank < 0 || o.rank >= h->world) {
      st = h->fail(EZLDA_E_INVALID, "world >= 1 with NCCL needs nccl_unique_id and 0 <= rank < world");
    } else if (!nccl().ok) {
      st = h->fail(EZLDA_E_NCCL, "libnccl.so.2 could not be loaded");
    } else {
      ncclUniqueId id;
      memcpy(&id, o.nccl_unique_id, sizeof(id));
      ncclResult_t r = nccl().CommInitRank(&h->comm, h->world, id, h->rank);
      if (r != ncclSuccess) st = h->fail(EZLDA_E_NCCL, "ncclCommInitRank: %s", nccl().GetErrorString(r));
    }
  }
  if (!st) st = do_create(h, word_ids, doc_ids, o);
  if (!st && h->pool) {  // give the transients' memory back (the steady state keeps its own buffers)
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) st = h->fail(EZLDA_E_CUDA, "create: stream sync failed");
    else cudaMemPoolTrimTo(h->pool, 0);
  }
  if (st) {
    g_create_error = h->err;
    ezlda_destroy(h);
    return st;
  }
  *out = h;
  return EZLDA_OK;
}

ezlda_status ezlda_iterate(ezlda* h, uint32_t n_iters) {
  if (!h) return EZLDA_E_INVALID;
  if (h->sticky) return EZLDA_E_STATE;
  cudaStream_t s = h->stream;
  for (uint32_t it = 0; it < n_iters; ++it) {
    const uint32_t i = h->iteration + 1;
    Buf& cur = h->buf[h->cur];
    Buf& nxt = h->buf[1 - h->cur];
    if ((int)h->pending.size() == ezlda::kSlots) {
      ezlda_status st = fold_one(h);
      if (st) return st;
    }
    const int si = (int)(h->slot_counter++ % ezlda::kSlots);
    ezlda::Slot& sl = h->slots[si];
    cudaEvent_t* ev = sl.ev;
    if (h->timing) EZ_CUDA(h, cudaEventRecord(ev[0], s));
    EZ_CUDA(h, cudaMemsetAsync(h->dev.ctr, 0, sizeof(ezl::Counters), s));
    EZ_CUDA(h, cudaMemsetAsync(h->dev.flags, 0, sizeof(uint32_t) * ((h->R + 31) / 32), s));
    EZ_CUDA(h, cudaMemsetAsync(nxt.Wd, 0, sizeof(int32_t) * (size_t)h->Vd * h->K, s));
    EZ_CUDA(h, cudaMemsetAsync(nxt.nk, 0, sizeof(int32_t) * h->K, s));
    EZ_CUDA(h, cudaMemsetAsync(nxt.tnnz, 0, sizeof(uint32_t) * std::max<uint32_t>(h->Vt, 1), s));
    ezl::launch_den(h->dev, cur, s);
    if (h->branches == 2) {
      // two-branch (ESCA) mode: D rebuild without the skip test, What / Q tables, one draw
      // per token, then W / n_k of the new topics from the item histograms
      if (h->timing) EZ_CUDA(h, cudaEventRecord(ev[1], s));
      ezl::launch_doc_pass(h->dev, cur, cur, h->docs_w, h->n_docs_w, h->docs_b, h->n_docs_b, i, false, s);
      if (h->timing) EZ_CUDA(h, cudaEventRecord(ev[2], s));
      if (h->timing) EZ_CUDA(h, cudaEventRecord(ev[5], s));
      if (h->timing) EZ_CUDA(h, cudaEventRecord(ev[6], s));
      ezl::launch_two_branch(h->dev, cur, nxt, h->n_items, i, s);
      if (!h->multi) ezl::launch_nk(h->dev, nxt, s);
      if (h->timing) EZ_CUDA(h, cudaEventRecord(ev[3], s));
    } else {
      if (h->dev.w0ord) {  // the iteration's absent-pair order (stable radix sort: ties by topic asc)
        k_w0_keys<<<blocks(h->K), 256, 0, s>>>(h->dev.what0, h->K, h->w0_key_in, h->w0_top_in);
        EZ_CUDA(h, cub::DeviceRadixSort::SortPairsDescending(h->w0_tmp, h->w0_tmp_bytes, h->w0_key_in, h->w0_key_out,
                                                             h->w0_top_in, h->dev.w0ord, (int)h->K, 0, 64, s));
      }
      ezl::launch_word_prep(h->dev, cur, s);
      if (h->timing) EZ_CUDA(h, cudaEventRecord(ev[1], s));
      ezl::launch_doc_pass(h->dev, cur, nxt, h->docs_w, h->n_docs_w, h->docs_b, h->n_docs_b, i, true, s);
      if (h->timing) EZ_CUDA(h, cudaEventRecord(ev[2], s));
      if (h->item_act) {  // H4: this iteration's live items (static heavy-first order kept)
        EZ_CUDA(h, cudaMemsetAsync(h->dev.word_live, 0, h->V, s));
        ezl::launch_item_schedule(h->dev, nxt, h->n_items, s);
        EZ_CUDA(h, cub::DeviceSelect::Flagged(h->sel_tmp, h->sel_tmp_bytes, h->item_iota, h->dev.item_live,
                                              h->item_act, h->n_act, (int)h->n_items, s));
      }
      if (h->timing) EZ_CUDA(h, cudaEventRecord(ev[5], s));
      ezl::launch_word_heads(h->dev, cur, s);  // heads of the live items' words (H1, second half)
      if (h->timing) EZ_CUDA(h, cudaEventRecord(ev[6], s));
      ezl::launch_sampler(h->dev, cur, nxt, h->n_items, i, false, s);
      if (!h->multi) ezl::launch_nk(h->dev, nxt, s);  // H6: n_k column sums of the new W
      if (h->timing) EZ_CUDA(h, cudaEventRecord(ev[3], s));
    }
    EZ_CUDA(h, cudaGetLastError());
    ezlda_status st;
    // H7 (world > 1): all-reduce of the dense block + all-gather of the tail
    // topics (one NCCL group) + tail-row rebuild; n_k from the merged W
    if ((st = exchange_w(h, nxt, &cur))) return st;
    if (h->multi) ezl::launch_nk(h->dev, nxt, s);  // n_k of the global W (identical on every rank)
    EZ_CUDA(h, cudaGetLastError());
    EZ_CUDA(h, cudaMemcpyAsync(h->ctr_host + si, h->dev.ctr, sizeof(ezl::Counters), cudaMemcpyDeviceToHost, s));
    EZ_CUDA(h, cudaEventRecord(ev[4], s));
    sl.iteration = i;
    // den, word-prep, doc pass tiers, sampler; two-branch: den, doc pass tiers, then one
    // word-major kernel, or What/Q tables + doc-major draw + W count
    sl.launches = 3u + (h->n_docs_w ? 1u : 0u) + (h->n_docs_b ? 1u : 0u) - (h->n_items ? 0u : 1u);
    if (h->branches == 2) sl.launches = ezl::two_branch_word_major(h->K) ? sl.launches - 1u : sl.launches + 1u;
    if (h->multi && h->Vt) sl.launches += (h->R > h->rt0 ? 1u : 0u) + 1u;  // tail gather + tail rebuild
    if (h->item_act && h->branches == 3) sl.launches += 2u;               // item schedule + CUB select
    sl.launches += 1u;                                                     // n_k column sums (k_nk)
    if (h->branches == 3 && h->dev.Vw) sl.launches += 1u;                  // word heads
    h->pending.push_back(si);
    h->cur = 1 - h->cur;
    h->iteration = i;
    h->D_fresh = false;  // D rows describe z^{i-1}
  }
  return EZLDA_OK;
}

ezlda_status ezlda_counts(ezlda* h, uint16_t* topics, int32_t* n_k, ezlda_csr* W, ezlda_csr* D) {
  if (!h) return EZLDA_E_INVALID;
  if (h->sticky) return EZLDA_E_STATE;
  cudaStream_t s = h->stream;
  Buf& b = h->buf[h->cur];
  if (topics) {
    uint16_t* tmp = h->alloc<uint16_t>(h->N);
    if (!tmp) return h->fail(EZLDA_E_NOMEM, "topics staging");
    ezl::launch_topics_to_input(b.z, h->perm, (uint32_t)h->N, tmp, s);
    EZ_CUDA(h, cudaGetLastError());
    EZ_CUDA(h, cudaMemcpyAsync(topics, tmp, sizeof(uint16_t) * h->N, cudaMemcpyDefault, s));
    EZ_CUDA(h, cudaStreamSynchronize(s));
    h->release(tmp);
  }
  if (n_k) {
    EZ_CUDA(h, cudaMemcpyAsync(n_k, b.nk, sizeof(int32_t) * h->K, cudaMemcpyDefault, s));
    EZ_CUDA(h, cudaStreamSynchronize(s));
  }
  if (W) {
    std::vector<int32_t> Wd((size_t)h->Vd * h->K);
    std::vector<uint32_t> Wt(h->tail_cap), tnnz(h->Vt), tofs(h->Vt + 1);
    if (!Wd.empty()) EZ_CUDA(h, cudaMemcpyAsync(Wd.data(), b.Wd, 4 * Wd.size(), cudaMemcpyDeviceToHost, s));
    if (!Wt.empty()) EZ_CUDA(h, cudaMemcpyAsync(Wt.data(), b.Wt, 4 * Wt.size(), cudaMemcpyDeviceToHost, s));
    if (h->Vt) {
      EZ_CUDA(h, cudaMemcpyAsync(tnnz.data(), b.tnnz, 4ull * h->Vt, cudaMemcpyDeviceToHost, s));
      EZ_CUDA(h, cudaMemcpyAsync(tofs.data(), h->dev.tofs, 4ull * (h->Vt + 1), cudaMemcpyDeviceToHost, s));
    }
    EZ_CUDA(h, cudaStreamSynchronize(s));
    const bool fill = W->col && W->val;
    uint64_t nnz = 0;
    W->rows = h->V;
    for (uint32_t ov = 0; ov < h->V; ++ov) {
      if (W->row_ptr) W->row_ptr[ov] = nnz;
      const uint32_t v = h->newword[ov];
      if (v < h->Vd) {
        const int32_t* r = &Wd[(size_t)v * h->K];
        for (uint32_t k = 0; k < h->K; ++k)
          if (r[k]) {
            if (fill) {
              if (nnz >= W->nnz) return h->fail(EZLDA_E_INVALID, "W csr capacity too small");
              W->col[nnz] = (uint16_t)k;
              W->val[nnz] = r[k];
            }
            ++nnz;
          }
      } else {
        const uint32_t t = v - h->Vd;
        for (uint32_t e = 0; e < tnnz[t]; ++e) {
          const uint32_t p = Wt[tofs[t] + e];
          if (fill) {
            if (nnz >= W->nnz) return h->fail(EZLDA_E_INVALID, "W csr capacity too small");
            W->col[nnz] = (uint16_t)(p >> 16);
            W->val[nnz] = (int32_t)(p & 0xFFFFu);
          }
          ++nnz;
        }
      }
    }
    if (W->row_ptr) W->row_ptr[h->V] = nnz;
    W->nnz = nnz;
  }
  if (D) {
    ezlda_status st = ensure_D(h);
    if (st) return st;
    std::vector<uint32_t> Dh(h->Dwords), dofs(h->Dn + 1), ddb(h->Dn);
    EZ_CUDA(h, cudaMemcpyAsync(Dh.data(), h->dev.D, 4 * Dh.size(), cudaMemcpyDeviceToHost, s));
    EZ_CUDA(h, cudaMemcpyAsync(dofs.data(), h->dev.dofs, 4ull * (h->Dn + 1), cudaMemcpyDeviceToHost, s));
    EZ_CUDA(h, cudaMemcpyAsync(ddb.data(), h->dev.ddb, 4ull * h->Dn, cudaMemcpyDeviceToHost, s));
    EZ_CUDA(h, cudaStreamSynchronize(s));
    const bool fill = D->col && D->val;
    uint64_t nnz = 0;
    D->rows = h->Dn;
    for (uint32_t d = 0; d < h->Dn; ++d) {
      if (D->row_ptr) D->row_ptr[d] = nnz;
      const uint32_t base = ddb[d];
      const uint32_t n = (dofs[d + 1] > dofs[d]) ? (Dh[base] & 0xFFFFu) : 0u;
      for (uint32_t e = 0; e < n; ++e) {
        const uint32_t p = Dh[base + ezl::kDHdr + ezl::d_at(h->dev.dperm, e)];
        if (fill) {
          if (nnz >= D->nnz) return h->fail(EZLDA_E_INVALID, "D csr capacity too small");
          D->col[nnz] = (uint16_t)ezl::d_topic(p, h->dev.dt);
          D->val[nnz] = (int32_t)(p & 0xFFFFu);
        }
        ++nnz;
      }
    }
    if (D->row_ptr) D->row_ptr[h->Dn] = nnz;
    D->nnz = nnz;
  }
  return EZLDA_OK;
}

ezlda_status ezlda_set_topics(ezlda* h, const uint16_t* topics, uint32_t iterations_done) {
  if (!h || !topics) return EZLDA_E_INVALID;
  if (h->sticky) return EZLDA_E_STATE;
  uint16_t* tmp = h->alloc<uint16_t>(h->N);
  uint32_t* d_max = h->alloc<uint32_t>(1);
  if (!tmp || !d_max) return h->fail(EZLDA_E_NOMEM, "topics staging");
  EZ_CUDA(h, cudaMemcpyAsync(tmp, topics, sizeof(uint16_t) * h->N, cudaMemcpyDefault, h->stream));
  // validate on the device (host or device input alike) before anything is replaced
  EZ_CUDA(h, cudaMemsetAsync(d_max, 0, 4, h->stream));
  k_max_u16<<<1184, 256, 0, h->stream>>>(tmp, h->N, d_max);
  uint32_t mx = 0;
  EZ_CUDA(h, cudaMemcpyAsync(&mx, d_max, 4, cudaMemcpyDeviceToHost, h->stream));
  EZ_CUDA(h, cudaStreamSynchronize(h->stream));
  h->release(d_max);
  if (mx >= h->K) {
    h->release(tmp);
    return h->fail(EZLDA_E_INVALID, "topic %u >= K = %u", mx, h->K);
  }
  ezl::launch_topics_from_input(tmp, h->perm, (uint32_t)h->N, h->buf[h->cur].z, h->stream);
  EZ_CUDA(h, cudaGetLastError());
  ezlda_status st = rebuild_counts(h);
  if (st) return st;
  EZ_CUDA(h, cudaStreamSynchronize(h->stream));
  h->release(tmp);
  h->iteration = iterations_done;
  return EZLDA_OK;
}

ezlda_status ezlda_loglik(ezlda* h, double* llpt) {
  if (!h || !llpt) return EZLDA_E_INVALID;
  if (h->sticky) return EZLDA_E_STATE;
  ezlda_status st = ensure_D(h);
  if (st) return st;
  Buf& b = h->buf[h->cur];
  ezl::launch_den(h->dev, b, h->stream);
  if (!h->llpt_scratch && ezl::llpt_smem_bytes(h->K) > 96u * 1024u) {
    h->llpt_scratch = h->alloc<double>(ezl::llpt_scratch_doubles(h->K));
    if (!h->llpt_scratch) return h->fail(EZLDA_E_NOMEM, "LLPT row scratch");
  }
  ezl::launch_llpt(h->dev, b, h->n_items, h->llpt_partial, h->llpt_out, h->llpt_scratch, h->stream);
  EZ_CUDA(h, cudaGetLastError());
  if ((st = allreduce(h, h->llpt_out, 1, ncclFloat64))) return st;
  double sum = 0;
  EZ_CUDA(h, cudaMemcpyAsync(&sum, h->llpt_out, 8, cudaMemcpyDeviceToHost, h->stream));
  EZ_CUDA(h, cudaStreamSynchronize(h->stream));
  *llpt = sum / (double)h->N_global;
  return EZLDA_OK;
}

ezlda_status ezlda_stats(const ezlda* hc, ezlda_iter_stats* last) {
  ezlda* h = const_cast<ezlda*>(hc);
  if (!h || !last) return EZLDA_E_INVALID;
  if (h->sticky) return EZLDA_E_STATE;
  ezlda_status st = fold_all(h);
  if (st) return st;
  *last = h->last;
  return EZLDA_OK;
}

ezlda_status ezlda_stats_sum(ezlda* h, ezlda_iter_stats* sum, int reset) {
  if (!h || !sum) return EZLDA_E_INVALID;
  if (h->sticky) return EZLDA_E_STATE;
  ezlda_status st = fold_all(h);
  if (st) return st;
  *sum = h->sum;
  sum->iteration = h->sum_n;
  if (reset) {
    h->sum = ezlda_iter_stats{};
    h->sum_n = 0;
  }
  return EZLDA_OK;
}

const char* ezlda_last_error(const ezlda* h) { return h ? h->err.c_str() : g_create_error.c_str(); }

void ezlda_destroy(ezlda* h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : h->allocs) {
    if (h->pool) cudaFreeAsync(p, h->stream); else cudaFree(p);
  }
  h->allocs.clear();
  if (h->pool) {
    cudaStreamSynchronize(h->stream);
    cudaMemPoolDestroy(h->pool);
    h->pool = nullptr;
  }
  if (h->ctr_host) cudaFreeHost(h->ctr_host);
  for (auto& sl : h->slots)
    for (auto& e : sl.ev)
      if (e) cudaEventDestroy(e);
  if (h->comm && nccl().ok) nccl().CommDestroy(h->comm);
  if (h->lgroup) local_group_leave(h->lgroup_key);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

size_t ezlda_nccl_id_size(void) { return sizeof(ncclUniqueId); }

ezlda_status ezlda_nccl_get_unique_id(void* id_out) {
  if (!id_out) return EZLDA_E_INVALID;
  if (!nccl().ok) return EZLDA_E_NCCL;
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != ncclSuccess) return EZLDA_E_NCCL;
  memcpy(id_out, &id, sizeof(id));
  return EZLDA_OK;
}

}  // extern "C"
