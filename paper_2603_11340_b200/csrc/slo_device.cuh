// slo_device.cuh — device-side random-number layer of the simulator.
// Written from the DESIGN.md text, independently of oracle/ (which the product never includes).
#pragma once
#include <cstdint>

#include "../../include/slo_sim.h"

namespace slo {

constexpr uint32_t FULL = 0xFFFFFFFFu;
constexpr uint64_t INF64 = 0xFFFFFFFFFFFFFFFFull;

// ---- Philox4x32-10: 10 rounds of two 32x32->64 products (IMAD.WIDE.U32) + xors.
struct u32x4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ u32x4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                        uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    // one widening multiply each (IMAD.WIDE.U32; separate IMAD.HI + IMAD measured no faster)
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0;
    const uint32_t h1 = (uint32_t)(p1 >> 32), l1 = (uint32_t)p1;
    const uint32_t n0 = h1 ^ c1 ^ k0;
    const uint32_t n2 = h0 ^ c3 ^ k1;
    c1 = l1;
    c3 = l0;
    c0 = n0;
    c2 = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}

// Philox4x32-10 with the round keys precomputed (rk0[r] = k0 + r W0, rk1[r] = k1 + r W1): the same function as
// philox(), for loops that draw many blocks under one key (K1g)
struct PhiloxKeys {
  uint32_t k0[10], k1[10];
};
__device__ __forceinline__ PhiloxKeys philox_keys(uint32_t k0, uint32_t k1) {
  PhiloxKeys K;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    K.k0[r] = k0 + (uint32_t)r * 0x9E3779B9u;
    K.k1[r] = k1 + (uint32_t)r * 0xBB67AE85u;
  }
  return K;
}
__device__ __forceinline__ u32x4 philox_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const PhiloxKeys& K) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0;
    const uint32_t h1 = (uint32_t)(p1 >> 32), l1 = (uint32_t)p1;
    const uint32_t n0 = h1 ^ c1 ^ K.k0[r];
    const uint32_t n2 = h0 ^ c3 ^ K.k1[r];
    c1 = l1;
    c3 = l0;
    c0 = n0;
    c2 = n2;
  }
  return {c0, c1, c2, c3};
}

// ---- E_q(u) ~ 2^32 * -ln((u+1)/2^32) in Q32.32.
__device__ __forceinline__ uint64_t exp_q32(uint32_t u) {
  if (u == 0xFFFFFFFFu) return 0;                   // x = 2^32
  const uint32_t x = u + 1u;                         // [1, 2^32)
  const int e = 31 - __clz(x);                       // floor(log2 x)
  const uint32_t m = x << (31 - e);                  // [2^31, 2^32)
  const int64_t t = (int64_t)(m - 0x80000000u);      // Q0.31
  int64_t acc = -7511879LL;
  acc = 49215561LL + ((acc * t) >> 31);
  acc = -151331885LL + ((acc * t) >> 31);
  acc = 300247864LL + ((acc * t) >> 31);
  acc = -455160697LL + ((acc * t) >> 31);
  acc = 601767258LL + ((acc * t) >> 31);
  acc = -771198690LL + ((acc * t) >> 31);
  acc = 1032354281LL + ((acc * t) >> 31);
  acc = -1549061789LL + ((acc * t) >> 31);
  acc = 3098163621LL + ((acc * t) >> 31);
  acc = 0LL + ((acc * t) >> 31);
  const uint64_t y = ((uint64_t)(32 - e) << 31) - (uint64_t)acc;   // < 2^37
  // floor(y * 2977044472 / 2^31): y < 2^37 so the 128-bit product is < 2^69
  const uint64_t lo = y * 2977044472ull;
  const uint64_t hi = __umul64hi(y, 2977044472ull);
  return (lo >> 31) | (hi << 33);
}

// floor(a * b / 2^s) for 0 < s < 64 with a 128-bit intermediate
__device__ __forceinline__ uint64_t mulshr(uint64_t a, uint64_t b, int s) {
  const uint64_t lo = a * b;
  const uint64_t hi = __umul64hi(a, b);
  return (lo >> s) | (hi << (64 - s));
}

// operational capacity of a bursty phase: min(2^62, floor(D * rho / 2^16))
__device__ __forceinline__ uint64_t capacity(uint64_t D, uint64_t rho) {
  const uint64_t lo = D * rho;
  const uint64_t hi = __umul64hi(D, rho);
  if (hi >= (1ull << 14)) return 1ull << 62;
  const uint64_t x = (lo >> 16) | (hi << 48);
  return x > (1ull << 62) ? (1ull << 62) : x;
}

// ---- lengths: lo + #{l : cw[l] <= u}: the bucket guide brackets the count, a binary
// search over the (usually empty) bracket finishes it
__device__ __forceinline__ uint32_t length_guided(const uint32_t* __restrict__ tables, uint32_t off, uint32_t goff,
                                                  uint32_t lo, uint32_t u) {
  const uint32_t g = __ldg(tables + goff + (u >> 24));
  uint32_t base = g & 0xFFFFu, n = (g >> 16) - base;
  const uint32_t* cw = tables + off;
  while (n > 0) {
    const uint32_t half = n >> 1;
    if (__ldg(cw + base + half) <= u) {
      base += half + 1;
      n -= half + 1;
    } else {
      n = half;
    }
  }
  return lo + base;
}

// ---- acceptance: thresholds T_a - 1 (a = 1..gp, gp = the last a with T_a > 0) and the
// 256-entry bucket guide (A at the top of bucket u >> 24, | 0x80 if a threshold falls inside the bucket).
// Used by K1/K1c's replica setup and by the exhaustive self-test (K6), so both run the same code.
__device__ __forceinline__ uint32_t accept_thresholds(uint32_t accept_q16, uint32_t width, uint32_t gamma,
                                                      uint32_t* tm1, bool write) {
  uint64_t rr = 65536;
  for (uint32_t w = 0; w < width; ++w) rr = (rr * (65536u - accept_q16)) >> 16;
  const uint64_t ae = 65536u - rr;
  uint64_t prev = 1ull << 32;
  uint32_t gp = 0;
  for (uint32_t a = 1; a <= gamma; ++a) {
    prev = (prev * ae) >> 16;
    if (prev > 0) {
      if (write) tm1[a - 1] = (uint32_t)(prev - 1);
      gp = a;
    }
  }
  return gp;
}

// guide entries kk = first, first + stride, ... (a group's lanes split the 256 buckets)
__device__ __forceinline__ void accept_guide(const uint32_t* tm1, uint32_t gp, uint8_t* guide, uint32_t first,
                                             uint32_t stride) {
  for (uint32_t kk = first; kk < 256; kk += stride) {
    const uint32_t lo = kk << 24, top = lo | 0xFFFFFFu;
    uint32_t A = 0, inside = 0;
    for (uint32_t a = 0; a < gp; ++a) {
      const uint32_t t = tm1[a];
      A += (top <= t);
      inside |= (t >= lo && t < top);
    }
    guide[kk] = (uint8_t)(A | (inside << 7));
  }
}

// A(u) = #{a in [1, gp] : u < T_a} through the bucket guide
__device__ __forceinline__ uint32_t accepted_guided(const uint8_t* guide, const uint32_t* tm1, uint32_t u,
                                                    uint32_t gp) {
  const uint32_t g = guide[u >> 24];
  uint32_t A = g & 0x7Fu;
  if (g & 0x80u) {
    while (A < gp && u <= tm1[A]) ++A;
  }
  return A;
}

// ---- fine acceptance guide (K1g, K6): 4096 byte entries by u >> 20, entry = (A_top + 1) | inside << 7 with
// A_top = #{a : T_a - 1 >= top of the bucket} and inside = a threshold T_a - 1 falls in [bottom, top).  In a
// bucket without an inside threshold A(u) = A_top for every u, so the common case is one byte load and the four
// draws of a SPEC block sum their (A + 1) bytes with two adds (an inside flag lifts the sum past 127).  Built
// by `stride` threads: each writes the A_top of its contiguous entries by a walk down the sorted thresholds,
// then (after a barrier of the caller) accept_guide_fine_mark() flags the buckets holding a threshold.
constexpr uint32_t kGuideFine = 4096;
__device__ __forceinline__ void accept_guide_fine(const uint32_t* tm1, uint32_t gp, uint8_t* guide, uint32_t first,
                                                  uint32_t stride) {
  const uint32_t per = (kGuideFine + stride - 1) / stride;
  const uint32_t k_lo = first * per, k_hi = min(kGuideFine, k_lo + per);
  // A_top(k) = #{a : tm1_a >= (k << 20) | 0xFFFFF}: non-increasing in k; tm1 is non-increasing in a
  uint32_t A = 0;
  while (A < gp && tm1[A] >= (((k_hi - 1) << 20) | 0xFFFFFu)) ++A;   // count at the last entry
  for (uint32_t k = k_hi; k-- > k_lo;) {
    while (A < gp && tm1[A] >= ((k << 20) | 0xFFFFFu)) ++A;
    guide[k] = (uint8_t)(A + 1u);
  }
}
__device__ __forceinline__ void accept_guide_fine_mark(const uint32_t* tm1, uint32_t gp, uint8_t* guide, uint32_t t) {
  if (t == 0) {
    for (uint32_t a = 0; a < gp; ++a)
      if ((tm1[a] & 0xFFFFFu) != 0xFFFFFu) guide[tm1[a] >> 20] |= 0x80u;
  }
}
// A(u) from the entry g of bucket u >> 20; an inside bucket finishes the count over the thresholds below its
// top, which are tm1[A_top ...] in order
__device__ __forceinline__ uint32_t accepted_fine(uint32_t g, const uint32_t* tm1, uint32_t u, uint32_t gp) {
  uint32_t A = (g & 0x7Fu) - 1u;
  if (g & 0x80u) {
    while (A < gp && u <= tm1[A]) ++A;
  }
  return A;
}

// ---- decode step cost d(n) = alpha0 + alpha1 n (R10 factorised by R28: W draft branches of
// gamma tokens, W gamma + 1 verified tokens per sequence)
__device__ __forceinline__ void step_coeffs(const slo_timing& t, uint32_t gamma, uint32_t width, uint64_t& alpha0,
                                            uint64_t& alpha1) {
  if (gamma == 0) {
    alpha0 = t.dec_base_us;
    alpha1 = t.dec_seq_us;
  } else {
    const uint64_t drafted = (uint64_t)gamma * width;
    alpha0 = drafted * t.dr_base_us + t.ver_base_us;
    alpha1 = drafted * t.dr_seq_us + t.ver_seq_us + (uint64_t)t.ver_tok_us * (drafted + 1);
  }
}

// ---- batch noise factor: f = 10^6 + (b0 + b1 + b2 + b3 - 510) step ppm of a word's bytes
// (step <= 1960, so f > 0); the head's w3 for a static batch or a prefill, an ITER word for a decode iteration
__device__ __forceinline__ uint32_t noise_factor(uint32_t w, uint32_t step) {
  const uint32_t bytesum = (uint32_t)__dp4a(w, 0x01010101u, 0u);   // b0 + b1 + b2 + b3 in one IDP4A
  return (uint32_t)(1000000 + ((int32_t)bytesum - 510) * (int32_t)step);
}

// ---- FNV-1a-32 of the 32 knob bytes (independent key mode)
__host__ __device__ inline uint32_t fnv1a_knobs(const slo_knobs& k) {
  uint8_t b[32];
  b[0] = k.conc; b[1] = k.max_num_seqs; b[2] = k.draft_len; b[3] = k.spec_on;
  b[4] = k.draft_width; b[5] = k.workload;
  b[6] = (uint8_t)(k.rate_scale_q8 & 0xFF); b[7] = (uint8_t)(k.rate_scale_q8 >> 8);
  for (int i = 0; i < 4; ++i) b[8 + i] = (uint8_t)(k.accept_q16 >> (8 * i));
  for (int i = 0; i < 4; ++i) b[12 + i] = (uint8_t)(k.max_wait_us >> (8 * i));
  for (int w = 0; w < 4; ++w)
    for (int i = 0; i < 4; ++i) b[16 + 4 * w + i] = (uint8_t)(k.reserved[w] >> (8 * i));
  uint32_t h = 2166136261u;
  for (int i = 0; i < 32; ++i) h = (h ^ b[i]) * 16777619u;
  return h;
}

__host__ __device__ inline bool knobs_valid(const slo_knobs& k, uint32_t n_wl) {
  return k.conc >= 1 && k.conc <= 32 && k.max_num_seqs >= 1 && k.max_num_seqs <= 32 && k.draft_len <= 16 &&
         k.spec_on <= 1 && k.draft_width >= 1 && k.draft_width <= 4 && k.workload < n_wl &&
         k.rate_scale_q8 >= 1 && k.accept_q16 <= 65536u && k.max_wait_us <= 50000u && k.reserved[0] == 0 &&
         k.reserved[1] == 0 && k.reserved[2] == 0 && k.reserved[3] == 0;
}

// ---- warp helpers
__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(FULL, (uint32_t)v, src);
  const uint32_t hi = __shfl_sync(FULL, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint64_t shfl_up64(uint64_t v, int d) {
  const uint32_t lo = __shfl_up_sync(FULL, (uint32_t)v, d);
  const uint32_t hi = __shfl_up_sync(FULL, (uint32_t)(v >> 32), d);
  return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint64_t warp_incl_scan64(uint64_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t o = shfl_up64(v, d);
    if (lane >= d) v += o;
  }
  return v;
}

__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    const uint32_t lo = __shfl_xor_sync(FULL, (uint32_t)v, d);
    const uint32_t hi = __shfl_xor_sync(FULL, (uint32_t)(v >> 32), d);
    v += ((uint64_t)hi << 32) | lo;
  }
  return v;
}

}  // namespace slo
