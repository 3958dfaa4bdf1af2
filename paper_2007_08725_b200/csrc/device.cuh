// device.cuh -- device helpers of the ezLDA sm_100a hot path (no torch, no oracle code).
//
// Everything parity-critical is fp64 and the library is compiled with -fmad=false, so
// each expression below rounds exactly as written (SURVEY 7.2 "Bitwise parity").
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ezl {

constexpr uint32_t kFull = 0xffffffffu;

// Per-word record written by the word-prep kernel ("MPT generate", P:546 step 1,
// Alg MPTG): top-4 topics of What[v] (ties -> smaller topic) and
// Q' = alpha * sum_{k != K1} What[v][k] (Eq 6).  48 bytes, L2 resident.
struct __align__(16) WordRec {
  double a[4];
  double Qp;
  uint16_t K[4];
};

// The doc pass's view of a word record (g <= 2): a1..a3 and Q' in one 32-byte aligned record
// (one 256-bit load per token instead of three 128-bit loads) and K1 | K2 << 16 beside it.
struct __align__(32) WordRecM {
  double a0, a1, a2, Qp;
};

// ---------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11).  Counter (t_g lo, t_g hi, iteration, 0),
// key = seed (lo, hi).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void philox4x32_10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                              uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// u = ((r0 >> 5) 2^26 + (r1 >> 6)) 2^-53: 53 random bits, exact in fp64.
__device__ __forceinline__ double philox_u(uint64_t seed, uint32_t iteration, uint64_t tg) {
  uint32_t c0 = (uint32_t)tg, c1 = (uint32_t)(tg >> 32), c2 = iteration, c3 = 0u;
  philox4x32_10(c0, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint64_t bits = ((uint64_t)(c0 >> 5) << 26) | (uint64_t)(c1 >> 6);
  return (double)bits * 0x1p-53;
}

// Round keys of Philox4x32-10 for one seed: key[2 r] = seed lo + r 0x9E3779B9, key[2 r + 1] =
// seed hi + r 0xBB67AE85 (r = 0..9), precomputed on the host so that the ten rounds take them as
// constant-bank operands instead of recomputing the key schedule per draw.
struct PhiloxKeys {
  uint32_t k[20];
};
inline PhiloxKeys philox_keys(uint64_t seed) {
  PhiloxKeys p;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    p.k[2 * r] = k0;
    p.k[2 * r + 1] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return p;
}

// philox_u with precomputed round keys (identical output)
__device__ __forceinline__ double philox_u_k(const PhiloxKeys& K, uint32_t iteration, uint64_t tg) {
  uint32_t c0 = (uint32_t)tg, c1 = (uint32_t)(tg >> 32), c2 = iteration, c3 = 0u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ K.k[2 * r], n2 = hi0 ^ c3 ^ K.k[2 * r + 1];
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  const uint64_t bits = ((uint64_t)(c0 >> 5) << 26) | (uint64_t)(c1 >> 6);
  return (double)bits * 0x1p-53;
}

// Iteration 0: z = floor(r0 K / 2^32).
__device__ __forceinline__ uint32_t philox_init_topic(uint64_t seed, uint64_t tg, uint32_t K) {
  uint32_t c0 = (uint32_t)tg, c1 = (uint32_t)(tg >> 32), c2 = 0u, c3 = 0u;
  philox4x32_10(c0, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
  return (uint32_t)(((uint64_t)c0 * (uint64_t)K) >> 32);
}

// ---------------------------------------------------------------------------------
// Warp primitives.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Inclusive Hillis-Steele scan over the 32 lanes (fixed order => deterministic).
__device__ __forceinline__ double warp_incl_scan(double x) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(kFull, x, o);
    if (lane >= (uint32_t)o) x = x + y;
  }
  return x;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

// ---------------------------------------------------------------------------------
// The MPT skip threshold (P:546 step 3; Eq 8 M = a1 (C1 + alpha); Eq 10 S_est with
// depth g; Alg MPTC): skip iff u < M / (M + S_est + Q').  Shared verbatim by the
// doc pass and the sampler so both take the identical decision.
// ---------------------------------------------------------------------------------
// exact uint32 -> fp64 with the 2^52 trick (one DADD instead of an I2F.F64)
__device__ __forceinline__ double u2d(uint32_t x) { return __hiloint2double(0x43300000, (int)x) - 0x1p52; }

__device__ __forceinline__ double mpt_M(const WordRec& r, uint32_t C1, double alpha) {
  return r.a[0] * (u2d(C1) + alpha);
}

// S_est + ... denominator of the threshold: (M + S_est) + Q'
__device__ __forceinline__ double mpt_den(const WordRec& r, double M, uint32_t C1, uint32_t C2, uint32_t C3,
                                          uint32_t L, uint32_t geff) {
  double S_est;
  if (geff == 0) {
    S_est = 0.0;
  } else if (geff == 1) {
    S_est = r.a[1] * u2d(L - C1);
  } else if (geff == 2) {
    S_est = r.a[1] * u2d(C2) + r.a[2] * u2d(L - C1 - C2);
  } else {
    S_est = (r.a[1] * u2d(C2) + r.a[2] * u2d(C3)) + r.a[3] * u2d(L - C1 - C2 - C3);
  }
  return (M + S_est) + r.Qp;
}

// The MPT decision u < thr with thr = M / den rounded as the oracle rounds it.  The
// division is skipped when u den is clear of M by a relative 2^-50 (then u < M / den
// and u < fl(M / den) agree); otherwise thr is formed exactly as written.
// (the division sits in a call of its own: inlined, the compiler speculates it -- MUFU.RCP64H
// and eight DFMA per token -- ahead of the two comparisons that almost always decide)
static __device__ __noinline__ bool mpt_skip_exact(double u, double M, double den) { return u < M / den; }
__device__ __forceinline__ bool mpt_skip(double u, double M, double den) {
  const double p = u * den;
  if (p < M * (1.0 - 0x1p-50)) return true;
  if (p > M * (1.0 + 0x1p-50)) return false;
  return mpt_skip_exact(u, M, den);
}

}  // namespace ezl
