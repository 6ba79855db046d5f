// slo_sim_kernel.cu — K1: one simulator replica per warp.
//
// Persistent grid; each warp pulls replica indices from a device atomic queue and runs the replica's
// whole segment. Per-warp shared memory (WarpRing) holds 64-entry rings of arrival times a_j and sorted
// completion times kappa_k, packed (P, O) lengths and noise words, the acceptance thresholds, the rarely
// touched warp-uniform state and the p99 candidate buffer. The event loop is replaced by the closed forms
// of DESIGN.md §2.6 (equal to the event definition; checked bit-exactly against the oracle):
//   s_j = max(a_j, kappa_{j-C});  t_form = max(t_idle, s_h[, min(s_h + max_wait, s_{h+B-1})]);
//   b = min(B, #{j in [h, h+C) : s_j <= t_form}) via ballot + popc;
//   Cum_m = alpha0 * S_m + alpha1 * sum_{m'} min(S_m', S_m); completion order = order of S_m.
#include <cstdint>

#include "slo_device.cuh"
#include "slo_internal.h"

namespace slo {

// A(u) = #{a in [1, gp] : u < T_a}. guide[u >> 24] holds A at the top of u's bucket
// (A is non-increasing in u, so this is the bucket minimum) and bit 7 when a threshold lies strictly
// inside the bucket; only then are the remaining thresholds counted.
__device__ __forceinline__ uint32_t accepted(const WarpRing& R, uint32_t u, uint32_t gp) {
  const uint32_t g = R.guide[u >> 24];
  uint32_t A = g & 0x7Fu;
  if (g & 0x80u) {
    while (A < gp && u <= R.tm1[A]) ++A;
  }
  return A;
}

// Lane-parallel step counts of a speculative batch of b members: member m owns the L = 32 / 2^ceil(log2 b)
// lanes [m L, (m+1) L); each round every lane of an unfinished member computes one Philox SPEC block
// (4 decode steps), a segmented scan of the block token sums finds the block where the member's cumulative
// tokens reach O_m, and that lane resolves the exact step.  Blocks past the crossing are computed
// speculatively and discarded (the definition's work is ceil(S_m/4) blocks per member).  Returns S_m in
// lane m (m < b).
__device__ __forceinline__ uint32_t spec_steps(const WarpRing& R, uint32_t k0, uint32_t k1, uint32_t h,
                                               uint32_t b, uint32_t gp, int lane) {
  const int lgb = 32 - __clz(b - 1u);                  // ceil(log2 b)
  const int lg = 5 - lgb;                              // log2 L
  const uint32_t L = 1u << lg;
  const uint32_t m = (uint32_t)lane >> lg, off = (uint32_t)lane & (L - 1u);
  const uint32_t segbase = m << lg;
  const uint32_t j = h + m;
  const uint32_t O = m < b ? (R.po[j & 63] >> 16) : 0u;
  const uint32_t lowmask = (L == 32u) ? FULL : ((1u << L) - 1u);
  uint32_t cum = 0, q = off, S = 0;
  bool pending = m < b;
  while (__any_sync(FULL, pending)) {
    uint32_t e0 = 0, e1 = 0, e2 = 0, e3 = 0;
    if (pending) {
      const u32x4 w = philox(j, 1, q, 0, k0, k1);
      e0 = accepted(R, w.x, gp) + 1;
      e1 = accepted(R, w.y, gp) + 1;
      e2 = accepted(R, w.z, gp) + 1;
      e3 = accepted(R, w.w, gp) + 1;
    }
    const uint32_t T = e0 + e1 + e2 + e3;
    uint32_t P = T;                                    // segmented inclusive scan over the L lanes
    for (int d = 1; d < (int)L; d <<= 1) {
      const uint32_t v = __shfl_up_sync(FULL, P, d);
      if ((int)off >= d) P += v;
    }
    const bool cross = pending && (cum + P >= O);
    const uint32_t segbits = (__ballot_sync(FULL, cross) >> segbase) & lowmask;
    const uint32_t first = __ffs(segbits) - 1u;        // crossing lane within the segment (if any)
    uint32_t give = P;
    if (segbits && off == first) {                     // this lane resolves the exact step
      const uint32_t c = cum + P - T;
      const uint32_t base = 4u * q;
      give = c + e0 >= O ? base + 1 : (c + e0 + e1 >= O ? base + 2 : (c + e0 + e1 + e2 >= O ? base + 3 : base + 4));
    }
    const uint32_t got = __shfl_sync(FULL, give, (int)(segbits ? segbase + first : segbase + L - 1u));
    if (pending) {
      if (segbits) {
        S = got;
        pending = false;
      } else {
        cum += got;
        q += L;
      }
    }
  }
  return __shfl_sync(FULL, S, (lane << lg) & 31);
}

// K-th largest value of buf[0..n) (1 <= K <= n): exact radix select, four 8-bit digits MSB first, with a
// per-warp shared-memory histogram.
__device__ __noinline__ uint32_t kth_largest(const uint32_t* buf, uint32_t n, uint32_t K, uint32_t* hist,
                                             int lane) {
  uint32_t prefix = 0, kk = K;
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
#pragma unroll
    for (int t = 0; t < 8; ++t) hist[lane * 8 + t] = 0;
    __syncwarp();
    const uint32_t hmask = shift == 24 ? 0u : (0xFFFFFFFFu << (shift + 8));
    for (uint32_t e = lane; e < n; e += 32) {
      const uint32_t v = buf[e];
      if ((v & hmask) == prefix) atomicAdd(&hist[(v >> shift) & 255u], 1u);
    }
    __syncwarp();
    uint32_t c[8], sum = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      c[t] = hist[lane * 8 + t];
      sum += c[t];
    }
    uint32_t incl = sum;                                 // suffix sum over lanes (bins >= 8 * lane)
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_down_sync(FULL, incl, d);
      if (lane + d < 32) incl += v;
    }
    const bool here = incl >= kk && incl - sum < kk;
    const int owner = __ffs(__ballot_sync(FULL, here)) - 1;
    uint32_t digit = 0, knew = 0;
    if (lane == owner) {
      uint32_t above = incl - sum;
#pragma unroll
      for (int t = 7; t >= 0; --t) {
        if (knew == 0 && above + c[t] >= kk) {
          digit = 8u * lane + t;
          knew = kk - above;
        }
        above += c[t];
      }
    }
    digit = __shfl_sync(FULL, digit, owner);
    kk = __shfl_sync(FULL, knew, owner);
    prefix |= digit << shift;
    __syncwarp();
  }
  return prefix;
}

// keep only values > theta (in place)
__device__ __noinline__ uint32_t compact_above(uint32_t* buf, uint32_t n, uint32_t theta, int lane) {
  uint32_t out = 0;
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t e = base + lane;
    const uint32_t v = e < n ? buf[e] : 0;
    const bool keep = e < n && v > theta;
    const uint32_t m = __ballot_sync(FULL, keep);
    __syncwarp();
    if (keep) buf[out + __popc(m & ((1u << lane) - 1u))] = v;
    out += __popc(m);
    __syncwarp();
  }
  return out;
}

// (a2, a3) generate requests [gen, gen + 32): Philox REQ blocks, exponential gaps (warp scan), bursty
// time change, lengths; written to the rings.  Warp-uniform process state lives in R.
__device__ __noinline__ void generate_chunk(WarpRing& R, const DevWorkload& W, const uint32_t* __restrict__ tables,
                                            uint32_t k0, uint32_t k1, uint32_t gen, uint32_t N, uint32_t warmup,
                                            int lane) {
  const uint32_t i = gen + (uint32_t)lane;
  const bool valid = i < N;
  const u32x4 w = philox(i, 0, 0, 0, k0, k1);
  const uint64_t E = valid ? exp_q32(w.x) : 0;
  uint64_t a = 0;
  if (W.kind == 0) {
    const uint64_t gap = mulshr(E, R.g[0], 48);
    a = R.last + warp_incl_scan64(gap, lane);
    const uint64_t last = shfl64(a, 31);
    __syncwarp();
    if (lane == 0) R.last = last;
  } else {
    const uint64_t tau = R.last + warp_incl_scan64(E, lane);
    const uint64_t last = shfl64(tau, 31);
    uint64_t pLam = R.pLam, pU = R.pU, pD = R.pD, pstart = R.pstart, nph = R.nphase;
    uint32_t ph = R.ph, pstate = R.pstate;
    bool done = !valid;
    for (;;) {
      const bool here = !done && tau < pLam + pU;
      if (here) {
        uint64_t off = mulshr(tau - pLam, R.g[pstate], 48);
        if (off > pD - 1) off = pD - 1;
        a = pstart + off;
        done = true;
      }
      if (__all_sync(FULL, done)) break;
      pLam += pU;
      pstart += pD;
      ++ph;
      pstate = (W.start_state + ph) & 1u;
      if (W.kind == 1) {
        const u32x4 pw = philox(ph, 2, 0, 0, k0, k1);
        pD = mulshr(exp_q32(pw.x), W.soj[pstate], 32);
        ++nph;
      } else {
        pD = W.soj[pstate];
      }
      pU = capacity(pD, R.rho[pstate]);
    }
    __syncwarp();
    if (lane == 0) {
      R.last = last;
      R.pLam = pLam; R.pU = pU; R.pD = pD; R.pstart = pstart; R.ph = ph; R.pstate = pstate; R.nphase = nph;
    }
  }
  if (valid) {
    const uint32_t P = length_of(tables + W.p_off, W.p_ncw, W.p_lo, w.y);
    const uint32_t O = length_of(tables + W.o_off, W.o_ncw, W.o_lo, w.z);
    R.a[i & 63] = a;
    R.po[i & 63] = P | (O << 16);
    R.w3[i & 63] = w.w;
    if (i == warmup) R.a_w = a;
  }
  __syncwarp();
}

#ifndef SLO_MAXNREG
#define SLO_MAXNREG 80
#endif
__global__ void __maxnreg__(SLO_MAXNREG) slo_sim_kernel(const SimParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  WarpRing& R = *reinterpret_cast<WarpRing*>(smem + (size_t)warp * p.warp_bytes);
  uint32_t* cand = reinterpret_cast<uint32_t*>(smem + (size_t)warp * p.warp_bytes + sizeof(WarpRing));
  const uint32_t lanemask_lt = (1u << lane) - 1u;
  const uint32_t N = p.warmup + p.seg;

  for (;;) {
    uint32_t r = 0;
    if (lane == 0) r = atomicAdd(p.queue, 1u);
    r = __shfl_sync(FULL, r, 0);
    if (r >= p.n_rep) break;

    const uint32_t ci = r / p.n_seeds;
    const slo_knobs k = p.cfg[ci];
    if (!knobs_valid(k, p.n_wl)) {  // sentinel outputs
      if (lane == 0) {
        p.p99[r] = 0xFFFFFFFFu;
        p.goodput[r] = -1.0;
        if (p.detail) p.detail[r] = slo_replica_result{0xFFFFFFFFu, 0, 0, 1u, 0, 0};
        if (p.stats) atomicAdd((unsigned long long*)&p.stats->replicas, 1ull);
      }
      continue;
    }
    const DevWorkload& W = p.wl[k.workload];
    const uint64_t seed = p.seeds[r - ci * p.n_seeds];
    const uint32_t cfgkey = p.crn ? W.stream_id : fnv1a_knobs(k);
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32) ^ cfgkey;
    const uint32_t C = k.conc, B = k.max_num_seqs, mw = k.max_wait_us;
    const uint32_t gamma = k.spec_on ? k.draft_len : 0u;

    // ---- (a1) replica setup: thresholds, step costs, arrival state
    uint32_t gp = 0;
    {
      uint64_t rr = 65536;
      for (uint32_t w = 0; w < k.draft_width; ++w) rr = (rr * (65536u - k.accept_q16)) >> 16;
      const uint64_t ae = 65536u - rr;
      uint64_t prev = 1ull << 32;
      for (uint32_t a = 1; a <= gamma; ++a) {
        prev = (prev * ae) >> 16;
        if (prev > 0) {
          if (lane == 0) R.tm1[a - 1] = (uint32_t)(prev - 1);
          gp = a;
        }
      }
    }
    if (lane == 0) {
      const uint64_t g0 = W.gap_q16[0] == INF64 ? INF64 : (W.gap_q16[0] << 8) / k.rate_scale_q8;
      const uint64_t g1 = W.gap_q16[1] == INF64 ? INF64 : (W.gap_q16[1] << 8) / k.rate_scale_q8;
      R.g[0] = g0;
      R.g[1] = g1;
      R.rho[0] = g0 == INF64 ? 0 : INF64 / g0;
      R.rho[1] = g1 == INF64 ? 0 : INF64 / g1;
      R.last = 0;
      R.nphase = 0;
      R.alpha0 = gamma == 0 ? (uint64_t)W.t.dec_base_us : (uint64_t)gamma * W.t.dr_base_us + W.t.ver_base_us;
      R.alpha1 = gamma == 0 ? (uint64_t)W.t.dec_seq_us
                            : (uint64_t)gamma * W.t.dr_seq_us + W.t.ver_seq_us + (uint64_t)W.t.ver_tok_us * (gamma + 1);
      R.pre_base = W.t.pre_base_us;
      R.pre_tok = W.t.pre_tok_us;
      R.noise = W.t.noise_step_ppm;
      if (W.kind != 0) {
        const uint32_t st = W.start_state & 1u;
        uint64_t D;
        if (W.kind == 1) {
          const u32x4 w = philox(0, 2, 0, 0, k0, k1);
          D = mulshr(exp_q32(w.x), W.soj[st], 32);
          R.nphase = 1;
        } else {
          D = W.soj[st];
        }
        R.pD = D;
        R.pU = capacity(D, R.rho[st]);
        R.pLam = 0;
        R.pstart = 0;
        R.ph = 0;
        R.pstate = st;
      }
    }
    __syncwarp();
    if (gamma > 0) {  // bucket guide for A(u)
      for (uint32_t kk = lane; kk < 256; kk += 32) {
        const uint32_t lo = kk << 24, top = lo | 0xFFFFFFu;
        uint32_t A = 0, inside = 0;
        for (uint32_t a = 0; a < gp; ++a) {
          const uint32_t t = R.tm1[a];
          A += (top <= t);
          inside |= (t >= lo && t < top);
        }
        R.guide[kk] = (uint8_t)(A | (inside << 7));
      }
      __syncwarp();
    }

    // ---- replica loop state (warp-uniform) and per-lane accumulators
    uint32_t h = 0, gen = 0;
    uint64_t t_idle = 0;
    uint32_t theta = 0, n_cand = 0;
    uint32_t my_slo = 0;         // lane m: SLO-met count of the members it held; bit 31: a latency saturated
    uint64_t my_sum = 0;         // lane m: sum of latencies
    uint32_t my_steps = 0;       // lane m: sum of S over the members it held
    uint32_t my_blk = 0;         // lane m: sum of ceil(S/4) (SPEC blocks of the definition)
    uint32_t my_bd = 0;          // lane 0: batches; lane 1: sum over batches of max S (decode steps)
    const bool big = N > (1u << 19);   // only then can a u32 lane counter overflow within a replica
    const uint32_t K = p.topk;

    while (h < N) {
      while (gen < N && gen < h + 32) {
        generate_chunk(R, W, p.tables, k0, k1, gen, N, p.warmup, lane);
        gen += 32;
      }

      // ---- (a4) issue times over the window j = h + lane: s_j = max(a_j, kappa_{j-C})
      const uint32_t j = h + lane;
      uint64_t sj = INF64;
      if ((uint32_t)lane < C && j < N) {
        const uint64_t aj = R.a[j & 63];
        const uint64_t kj = j >= C ? R.kap[(j - C) & 63] : 0;
        sj = aj > kj ? aj : kj;
      }
      // ---- (a5) formation instant and batch size
      const uint64_t sh = shfl64(sj, 0);
      uint64_t t_form = t_idle > sh ? t_idle : sh;
      if (mw > 0) {
        const uint64_t sl = shfl64(sj, (int)(B - 1));   // INF if B > C or beyond N
        const uint64_t dl = sh + mw;
        const uint64_t x = dl < sl ? dl : sl;
        if (x > t_form) t_form = x;
      }
      uint32_t b = __popc(__ballot_sync(FULL, sj <= t_form));
      if (b > B) b = B;
      const bool member = (uint32_t)lane < b;
      const uint32_t po = member ? R.po[j & 63] : 0u;

      // ---- (a7) decode: per-member step counts S_m = min{s : sum_{j<s} (A(u_{m,j}) + 1) >= O_m}
      uint32_t S;
      if (gamma == 0) {
        S = po >> 16;
      } else {
        S = spec_steps(R, k0, k1, h, b, gp, lane);
      }

      // ---- (a6) prefill with the head's noise factor
      const uint32_t w3h = R.w3[h & 63];
      const uint32_t bytesum = (w3h & 0xFF) + ((w3h >> 8) & 0xFF) + ((w3h >> 16) & 0xFF) + (w3h >> 24);
      const uint64_t f = (uint64_t)(int64_t)(1000000 + ((int32_t)bytesum - 510) * (int32_t)R.noise);
      const uint32_t maxP = __reduce_max_sync(FULL, po & 0xFFFFu);
      const uint64_t t0 = t_form + f * ((uint64_t)R.pre_base + (uint64_t)R.pre_tok * maxP) / 1000000u;

      // Completion order = order of S (ties by member index): bitonic sort of (S, member) over the first
      // 2^ceil(log2 b) lanes; at sorted position k, sum_m' min(S_m', S_(k)) = sum_{i<k} S_(i) + (b-k) S_(k)
      // and Cum_(k) = alpha0 S_(k) + alpha1 * that (d(n) = alpha0 + alpha1 n).
      const int lgn = 32 - __clz(b - 1u);
      uint32_t key = member ? (S << 5) | (uint32_t)lane : 0xFFFFFFFFu;
      for (int kk = 1; kk <= lgn; ++kk) {
        for (int jj = kk - 1; jj >= 0; --jj) {
          const uint32_t other = __shfl_xor_sync(FULL, key, 1 << jj);
          const bool up = ((lane >> kk) & 1) == 0;
          const bool lower = ((lane >> jj) & 1) == 0;
          key = (lower == up) ? min(key, other) : max(key, other);
        }
      }
      const uint32_t Sk = member ? key >> 5 : 0u;       // sorted step count at position k = lane
      const uint32_t orig = key & 31u;                   // member index of position k
      uint32_t incl = Sk;
      for (int d = 1; d < (1 << lgn); d <<= 1) {
        const uint32_t v = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += v;
      }
      const uint32_t summin = incl - Sk + (b - (uint32_t)lane) * Sk;
      const uint64_t cum = R.alpha0 * Sk + R.alpha1 * summin;
      const uint64_t c = t0 + (f * cum) / 1000000u;
      if (member) R.kap[(h + lane) & 63] = c;
      t_idle = shfl64(c, (int)b - 1);
      const uint32_t maxS = __shfl_sync(FULL, Sk, (int)b - 1);

      // ---- (a8) latencies, SLO count, sums, p99 candidates (position k holds member orig)
      const uint32_t i = h + orig;
      const bool measured = member && i >= p.warmup;
      const uint64_t l = c - (member ? R.a[i & 63] : c);
      const uint32_t ls = l > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)l;
      if (measured) {
        my_slo += (l <= p.slo_us);
        my_slo |= (l > 0xFFFFFFFFull) ? 0x80000000u : 0u;
        my_sum += l;
      }
      if (p.lat != nullptr && member) p.lat[(size_t)r * N + i] = ls;
      const bool ins = measured && ls > theta;
      const uint32_t im = __ballot_sync(FULL, ins);
      if (ins) cand[n_cand + __popc(im & lanemask_lt)] = ls;
      n_cand += __popc(im);
      if (n_cand > p.cap - 32) {
        __syncwarp();
        theta = kth_largest(cand, n_cand, K, R.hist, lane);
        n_cand = compact_above(cand, n_cand, theta, lane);
      }
      // work counters, lane-local (flushed to the warp's totals before they could overflow)
      my_steps += Sk;
      my_blk += gamma > 0 ? (Sk + 3u) >> 2 : 0u;
      my_bd += lane == 0 ? 1u : maxS;
      if (big && (my_steps >= 0x80000000u || my_bd >= 0x80000000u)) {
        if (p.stats) {
          unsigned long long* st = (unsigned long long*)p.stats;
          atomicAdd(st + 3, (unsigned long long)my_steps);
          atomicAdd(st + 4, (unsigned long long)my_blk);
          if (lane < 2) atomicAdd(st + 1 + lane, (unsigned long long)my_bd);
        }
        my_steps = my_blk = my_bd = 0;
      }
      h += b;
    }

    // ---- (a9, a10) replica outputs
    __syncwarp();
    const uint32_t p99 = n_cand >= K ? kth_largest(cand, n_cand, K, R.hist, lane) : theta;
    const uint32_t slo_met = __reduce_add_sync(FULL, my_slo & 0x7FFFFFFFu);
    const uint64_t sum = warp_sum64(my_sum);
    const bool sat = __any_sync(FULL, (my_slo >> 31) != 0);
    if (lane == 0) {
      const uint64_t Tw = t_idle - R.a_w;
      const uint64_t T = Tw < 1 ? 1 : Tw;
      p.p99[r] = p99;
      p.goodput[r] = (double)((uint64_t)slo_met * 1000000ull) / (double)T;
      if (p.detail) p.detail[r] = slo_replica_result{p99, slo_met, p.seg, sat ? 2u : 0u, T, sum};
    }
    if (p.stats) {  // requests, batches, decode steps, member steps, Philox blocks, replicas
      const uint64_t msteps = warp_sum64(my_steps);
      const uint64_t blocks = warp_sum64(my_blk);
      unsigned long long* st = (unsigned long long*)p.stats;
      if (lane < 2) atomicAdd(st + 1 + lane, (unsigned long long)my_bd);
      if (lane == 2) atomicAdd(st + 3, (unsigned long long)msteps);
      if (lane == 3) atomicAdd(st + 4, (unsigned long long)(blocks + N + R.nphase));
      if (lane == 4) atomicAdd(st + 0, (unsigned long long)N);
      if (lane == 5) atomicAdd(st + 5, 1ull);
    }
    __syncwarp();
  }
}

}  // namespace slo
