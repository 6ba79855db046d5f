// slo_sim_kernel.cu — K1: one simulator replica per warp.
//
// Persistent grid; each warp pulls replica indices from a device atomic queue and runs the replica's
// whole segment. Per-warp shared memory holds 64-entry rings of arrival times a_j and sorted completion
// times kappa_k, packed (P, O) lengths and noise words, the acceptance thresholds and the p99 candidate
// buffer. The event loop is replaced by the closed forms of DESIGN.md §2.6 (proven equal to the event
// definition and checked bit-exactly against the oracle):
//   s_j = max(a_j, kappa_{j-C});  t_form = max(t_idle, s_h[, min(s_h + max_wait, s_{h+B-1})]);
//   b = min(B, #{j in [h, h+C) : s_j <= t_form}) via ballot + popc;
//   Cum_m = alpha0 * S_m + alpha1 * sum_{m'} min(S_m', S_m); completion order = order of S_m.
#include <cstdint>

#include "slo_device.cuh"
#include "slo_internal.h"

namespace slo {

// A(u) = #{a in [1, gp] : u < T_a}: start from the bucket minimum guide[u >> 24]
// (A is non-increasing in u) and count the remaining thresholds of that bucket (rarely more than 0).
__device__ __forceinline__ uint32_t accepted(const WarpRing& R, uint32_t u, uint32_t gp) {
  uint32_t A = R.guide[u >> 24];
  while (A < gp && u <= R.tm1[A]) ++A;
  return A;
}

// Lane-parallel step counts for a speculative batch: work items (member, Philox SPEC block q) are spread
// over all 32 lanes, L = 2^floor(log2(32/u)) consecutive blocks per unfinished member per round; a
// segmented scan of block token sums finds the crossing block, whose lane resolves the exact step.
// Blocks past a member's crossing are computed speculatively and discarded (they are not part of the
// definition's work count, which is ceil(S_m/4) blocks per member).
__device__ __forceinline__ uint32_t spec_steps(WarpRing& R, uint32_t k0, uint32_t k1, uint32_t j, uint32_t O,
                                               bool member, uint32_t gp, int lane, uint32_t lanemask_lt) {
  uint32_t S = 0, cum = 0, q = 0;
  bool pending = member;
  uint32_t pend = __ballot_sync(FULL, pending);
  while (pend) {
    const uint32_t u = __popc(pend);
    const int lg = 31 - __clz(32u / u);                  // L = 2^lg <= 32/u
    const uint32_t L = 1u << lg;
    const uint32_t myslot = __popc(pend & lanemask_lt);
    if (pending) R.slot[myslot] = (uint8_t)lane;
    __syncwarp();
    const uint32_t slot = (uint32_t)lane >> lg, off = (uint32_t)lane & (L - 1u);
    const bool active = slot < u;
    const int src = active ? R.slot[slot] : 0;
    const uint32_t mj = __shfl_sync(FULL, j, src);
    const uint32_t mO = __shfl_sync(FULL, O, src);
    const uint32_t mcum = __shfl_sync(FULL, cum, src);
    const uint32_t mq = __shfl_sync(FULL, q, src);
    uint32_t e0 = 0, e1 = 0, e2 = 0, e3 = 0;
    if (active) {
      const u32x4 w = philox(mj, 1, mq + off, 0, k0, k1);
      e0 = accepted(R, w.x, gp) + 1;
      e1 = accepted(R, w.y, gp) + 1;
      e2 = accepted(R, w.z, gp) + 1;
      e3 = accepted(R, w.w, gp) + 1;
    }
    const uint32_t T = e0 + e1 + e2 + e3;
    uint32_t P = T;                                      // segmented inclusive scan over the L lanes
    for (uint32_t d = 1; d < L; d <<= 1) {
      const uint32_t v = __shfl_up_sync(FULL, P, d);
      if (off >= d) P += v;
    }
    const bool cross = active && (mcum + P >= mO);
    const uint32_t cb = __ballot_sync(FULL, cross);
    const uint32_t segmask = (L == 32u) ? FULL : (((1u << L) - 1u) << (slot * L));
    uint32_t Sx = 0;
    if (cross && (uint32_t)(__ffs(cb & segmask) - 1) == (uint32_t)lane) {
      const uint32_t c = mcum + P - T;                   // tokens before this block
      const uint32_t base = 4u * (mq + off);
      Sx = c + e0 >= mO ? base + 1 : (c + e0 + e1 >= mO ? base + 2 : (c + e0 + e1 + e2 >= mO ? base + 3 : base + 4));
    }
    const uint32_t mymask = (L == 32u) ? FULL : (((1u << L) - 1u) << (myslot * L));
    const uint32_t myfirst = cb & mymask;
    const int from = myfirst ? __ffs(myfirst) - 1 : (int)(myslot * L + L - 1u);
    const uint32_t gotS = __shfl_sync(FULL, Sx, from & 31);
    const uint32_t gotP = __shfl_sync(FULL, P, from & 31);
    if (pending) {
      if (myfirst) {
        S = gotS;
        pending = false;
      } else {
        cum += gotP;
        q += L;
      }
    }
    pend = __ballot_sync(FULL, pending);
  }
  return S;
}


// K-th largest value of buf[0..n) (K >= 1, n >= K): MSB-first radix select by warp counting.
__device__ __forceinline__ uint32_t kth_largest(const uint32_t* buf, uint32_t n, uint32_t K, int lane) {
  uint32_t prefix = 0, kk = K;
#pragma unroll 1
  for (int bit = 31; bit >= 0; --bit) {
    const uint32_t want = prefix | (1u << bit);
    const uint32_t mask = ~((1u << bit) - 1u);
    uint32_t cnt = 0;
    for (uint32_t e = lane; e < n; e += 32) cnt += ((buf[e] & mask) == want);
    cnt = __reduce_add_sync(FULL, cnt);
    if (cnt >= kk) prefix = want;
    else kk -= cnt;
  }
  return prefix;
}

// keep only values > theta (in place, order not preserved beyond stability within rounds)
__device__ __forceinline__ uint32_t compact_above(uint32_t* buf, uint32_t n, uint32_t theta, int lane) {
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

__global__ void __launch_bounds__(kMaxWarpsPerBlock * 32)
    slo_sim_kernel(const SimParams p) {
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

    // ---- acceptance thresholds; gp = number of positive thresholds
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
      if (gamma > 0) {  // bucket guide for A(u)
        __syncwarp();
        for (uint32_t kk = lane; kk < 256; kk += 32) {
          const uint32_t utop = (kk << 24) | 0xFFFFFFu;
          uint32_t A = 0;
          while (A < gp && utop <= R.tm1[A]) ++A;
          R.guide[kk] = (uint8_t)A;
        }
        __syncwarp();
      }
    }
    // ---- step-cost coefficients: d(n) = alpha0 + alpha1 * n
    const uint64_t alpha0 = gamma == 0 ? (uint64_t)W.t.dec_base_us
                                       : (uint64_t)gamma * W.t.dr_base_us + W.t.ver_base_us;
    const uint64_t alpha1 = gamma == 0 ? (uint64_t)W.t.dec_seq_us
                                       : (uint64_t)gamma * W.t.dr_seq_us + W.t.ver_seq_us +
                                             (uint64_t)W.t.ver_tok_us * (gamma + 1);
    // ---- arrival state
    const uint32_t kind = W.kind;
    const uint64_t g0 = W.gap_q16[0] == INF64 ? INF64 : (W.gap_q16[0] << 8) / k.rate_scale_q8;
    const uint64_t g1 = W.gap_q16[1] == INF64 ? INF64 : (W.gap_q16[1] << 8) / k.rate_scale_q8;
    uint64_t a_last = 0, tau_last = 0;
    uint32_t ph = 0, pstate = W.start_state & 1u;
    uint64_t pstart = 0, pD = 0, pU = 0, pLam = 0;
    uint64_t n_phase_blocks = 0;
    if (kind != 0) {
      if (kind == 1) {
        const u32x4 w = philox(0, 2, 0, 0, k0, k1);
        pD = mulshr(exp_q32(w.x), W.soj[pstate], 32);
        n_phase_blocks = 1;
      } else {
        pD = W.soj[pstate];
      }
      const uint64_t g = pstate ? g1 : g0;
      pU = g == INF64 ? 0 : (uint64_t)(((unsigned __int128)pD << 48) / g);
    }

    // ---- replica loop state (warp-uniform)
    uint32_t h = 0, gen = 0;
    uint64_t t_idle = 0;
    uint32_t theta = 0, n_cand = 0;
    // per-lane accumulators (lane m accumulates batch member m)
    uint32_t my_slo = 0;
    uint64_t my_sum = 0;
    bool my_sat = false;
    uint64_t n_batches = 0, n_dsteps = 0, n_msteps = 0, n_spec_blocks = 0;
    const uint32_t K = p.topk;

    while (h < N) {
      // ---- (a2, a3) generate requests [gen, gen + 32) until the window [h, h + 32) exists
      while (gen < N && gen < h + 32) {
        const uint32_t i = gen + lane;
        const bool valid = i < N;
        const u32x4 w = philox(i, 0, 0, 0, k0, k1);
        const uint64_t E = valid ? exp_q32(w.x) : 0;
        uint64_t a;
        if (kind == 0) {
          const uint64_t gap = mulshr(E, g0, 48);
          a = a_last + warp_incl_scan64(gap, lane);
          a_last = shfl64(a, 31);
        } else {
          const uint64_t tau = tau_last + warp_incl_scan64(E, lane);
          tau_last = shfl64(tau, 31);
          bool done = !valid;
          a = 0;
          for (;;) {
            const bool here = !done && tau < pLam + pU;
            if (here) {
              const uint64_t g = pstate ? g1 : g0;
              uint64_t off = mulshr(tau - pLam, g, 48);
              if (off > pD - 1) off = pD - 1;
              a = pstart + off;
              done = true;
            }
            if (__all_sync(FULL, done)) break;
            pLam += pU;
            pstart += pD;
            ++ph;
            pstate = (W.start_state + ph) & 1u;
            if (kind == 1) {
              const u32x4 pw = philox(ph, 2, 0, 0, k0, k1);
              pD = mulshr(exp_q32(pw.x), W.soj[pstate], 32);
              ++n_phase_blocks;
            } else {
              pD = W.soj[pstate];
            }
            const uint64_t g = pstate ? g1 : g0;
            pU = g == INF64 ? 0 : (uint64_t)(((unsigned __int128)pD << 48) / g);
          }
        }
        if (valid) {
          const uint32_t P = length_of(p.tables + W.p_off, W.p_ncw, W.p_lo, w.y);
          const uint32_t O = length_of(p.tables + W.o_off, W.o_ncw, W.o_lo, w.z);
          R.a[i & 63] = a;
          R.po[i & 63] = P | (O << 16);
          R.w3[i & 63] = w.w;
          if (i == p.warmup) R.a_w = a;
        }
        gen += 32;
        __syncwarp();
      }

      // ---- (a4) issue times over the window j = h + lane: s_j = max(a_j, kappa_{j-C})
      const uint32_t j = h + lane;
      const bool inwin = (uint32_t)lane < C && j < N;
      const uint64_t aj = j < N ? R.a[j & 63] : INF64;
      uint64_t sj = INF64;
      if (inwin) {
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

      // ---- (a6) prefill with the head's noise factor
      const uint32_t w3h = R.w3[h & 63];
      const uint64_t f = (uint64_t)(1000000 + ((int64_t)((w3h & 0xFF) + ((w3h >> 8) & 0xFF) +
                                                         ((w3h >> 16) & 0xFF) + (w3h >> 24)) -
                                               510) *
                                                  (int64_t)W.t.noise_step_ppm);
      const uint32_t po = member ? R.po[j & 63] : 0u;
      const uint32_t maxP = __reduce_max_sync(FULL, po & 0xFFFFu);
      const uint64_t Dp = f * ((uint64_t)W.t.pre_base_us + (uint64_t)W.t.pre_tok_us * maxP) / 1000000u;

      // ---- (a7) decode: per-member step counts S_m = min{s : sum_{j<s} (A(u_{m,j}) + 1) >= O_m}
      uint32_t S = 0;
      if (gamma == 0) {
        S = member ? (po >> 16) : 0u;
      } else {
        S = spec_steps(R, k0, k1, j, po >> 16, member, gp, lane, lanemask_lt);
      }
      // Cum_m = alpha0 * S_m + alpha1 * sum_m' min(S_m', S_m); rank_m = position in completion order
      uint32_t summin = 0, rank = 0, maxS = 0;
      for (uint32_t m = 0; m < b; ++m) {
        const uint32_t Sm = __shfl_sync(FULL, S, (int)m);
        summin += Sm < S ? Sm : S;
        rank += (Sm < S) || (Sm == S && m < (uint32_t)lane);
        maxS = Sm > maxS ? Sm : maxS;
      }
      const uint64_t cum = alpha0 * S + alpha1 * summin;
      const uint64_t c = t_form + Dp + (f * cum) / 1000000u;
      if (member) R.kap[(h + rank) & 63] = c;
      const uint32_t lastm = __ballot_sync(FULL, member && rank == b - 1);
      t_idle = shfl64(c, __ffs(lastm) - 1);

      // ---- (a8) latencies, SLO count, sums, p99 candidates
      const bool measured = member && j >= p.warmup;
      const uint64_t l = c - aj;
      const uint32_t ls = l > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)l;
      if (measured) {
        my_slo += (l <= p.slo_us);
        my_sum += l;
        my_sat |= (l > 0xFFFFFFFFull);
      }
      if (p.lat != nullptr && member) p.lat[(size_t)r * N + j] = ls;
      const bool ins = measured && ls > theta;
      const uint32_t im = __ballot_sync(FULL, ins);
      if (ins) cand[n_cand + __popc(im & lanemask_lt)] = ls;
      n_cand += __popc(im);
      __syncwarp();
      if (n_cand > p.cap - 32) {
        theta = kth_largest(cand, n_cand, K, lane);
        n_cand = compact_above(cand, n_cand, theta, lane);
      }
      // counters
      ++n_batches;
      n_dsteps += maxS;
      const uint32_t bsteps = __reduce_add_sync(FULL, S);
      n_msteps += bsteps;
      if (gamma > 0) n_spec_blocks += __reduce_add_sync(FULL, (S + 3u) >> 2);
      h += b;
    }

    // ---- (a9, a10) replica outputs
    __syncwarp();
    const uint32_t p99 = n_cand >= K ? kth_largest(cand, n_cand, K, lane) : theta;
    const uint32_t slo_met = __reduce_add_sync(FULL, my_slo);
    const uint64_t sum = warp_sum64(my_sum);
    const bool sat = __any_sync(FULL, my_sat);
    if (lane == 0) {
      const uint64_t Tw = t_idle - R.a_w;
      const uint64_t T = Tw < 1 ? 1 : Tw;
      p.p99[r] = p99;
      p.goodput[r] = (double)((uint64_t)slo_met * 1000000ull) / (double)T;
      if (p.detail) p.detail[r] = slo_replica_result{p99, slo_met, p.seg, sat ? 2u : 0u, T, sum};
      if (p.stats) {
        atomicAdd((unsigned long long*)&p.stats->requests, (unsigned long long)N);
        atomicAdd((unsigned long long*)&p.stats->batches, (unsigned long long)n_batches);
        atomicAdd((unsigned long long*)&p.stats->decode_steps, (unsigned long long)n_dsteps);
        atomicAdd((unsigned long long*)&p.stats->member_steps, (unsigned long long)n_msteps);
        atomicAdd((unsigned long long*)&p.stats->philox_blocks,
                  (unsigned long long)(N + n_phase_blocks + n_spec_blocks));
        atomicAdd((unsigned long long*)&p.stats->replicas, 1ull);
      }
    }
    __syncwarp();
  }
}

}  // namespace slo
