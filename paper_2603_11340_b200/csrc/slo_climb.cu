// slo_climb.cu — K2 (per-config aggregation over seeds) and K3 (device-resident Alg. 1 step).
// Eq. (2)-(3), Alg. 1, neighbour rule PAPER.md:142; the exact
// integer definitions are DESIGN.md §2.9.
#include <cstdint>

#include "slo_device.cuh"
#include "slo_internal.h"

namespace slo {

// ------------------------------------------------------------------------------------------------
// K2: d_agg[c] = sum_s detail[c * n_seeds + s]   (one warp per config)
// ------------------------------------------------------------------------------------------------
__global__ void slo_aggregate_kernel(const slo_replica_result* __restrict__ detail, uint32_t n_cfg,
                                     uint32_t n_seeds, slo_config_agg* __restrict__ agg) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_cfg) return;
  uint64_t sp = 0, sm = 0, sw = 0;
  uint32_t fl = 0;
  const slo_replica_result* d = detail + (size_t)warp * n_seeds;
  for (uint32_t s = lane; s < n_seeds; s += 32) {
    const slo_replica_result x = d[s];
    sp += x.p99_us;
    sm += x.slo_met;
    sw += x.window_us;
    fl |= x.flags;
  }
  sp = warp_sum64(sp);
  sm = warp_sum64(sm);
  sw = warp_sum64(sw);
  fl = __reduce_or_sync(FULL, fl);
  if (lane == 0) agg[warp] = slo_config_agg{sp, sm, sw, n_seeds, fl};
}

__global__ void slo_aggregate_reduce_kernel(const slo_config_agg* __restrict__ parts, uint32_t n_parts,
                                            uint32_t n_cfg, slo_config_agg* __restrict__ out) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cfg) return;
  slo_config_agg a{0, 0, 0, 0, 0};
  for (uint32_t p = 0; p < n_parts; ++p) {
    const slo_config_agg x = parts[(size_t)p * n_cfg + c];
    a.sum_p99_us += x.sum_p99_us;
    a.sum_slo_met += x.sum_slo_met;
    a.sum_window_us += x.sum_window_us;
    a.n_seeds += x.n_seeds;
    a.flags |= x.flags;
  }
  out[c] = a;
}

// ------------------------------------------------------------------------------------------------
// NEXT-4 peer exchange: K2x aggregates and pushes into every rank's window, K2w waits and sums
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ slo_config_agg* inbox(char* base, uint32_t par, uint32_t world, uint32_t src,
                                                 uint32_t n_cfg) {
  return reinterpret_cast<slo_config_agg*>(base + kXHeader) + ((size_t)par * world + src) * n_cfg;
}
__device__ __forceinline__ unsigned long long* xflag(char* base, uint32_t par, uint32_t src) {
  return reinterpret_cast<unsigned long long*>(base) + par * kXMaxRanks + src;
}

// one warp per config: the K2 sums, stored into slot [parity][rank] of every rank's window (P2P stores over
// NVLink for the peers); the last block to finish publishes flag[parity][rank] = epoch in every window
__global__ void slo_aggregate_push_kernel(const slo_replica_result* __restrict__ detail, uint32_t n_cfg,
                                          uint32_t n_seeds, char* const* __restrict__ peers, uint32_t world,
                                          uint32_t rank, XState* st) {
  const unsigned long long e = *(volatile unsigned long long*)&st->epoch + 1ull;
  const uint32_t par = (uint32_t)(e & 1ull);
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp < n_cfg) {
    uint64_t sp = 0, sm = 0, sw = 0;
    uint32_t fl = 0;
    const slo_replica_result* d = detail + (size_t)warp * n_seeds;
    for (uint32_t s = lane; s < n_seeds; s += 32) {
      const slo_replica_result x = d[s];
      sp += x.p99_us;
      sm += x.slo_met;
      sw += x.window_us;
      fl |= x.flags;
    }
    sp = warp_sum64(sp);
    sm = warp_sum64(sm);
    sw = warp_sum64(sw);
    fl = __reduce_or_sync(FULL, fl);
    const slo_config_agg a{sp, sm, sw, n_seeds, fl};
    if ((uint32_t)lane < world) inbox(peers[lane], par, world, rank, n_cfg)[warp] = a;   // lane r -> rank r
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(&st->arrive_push, 1u) == gridDim.x - 1) {       // every block's stores are fenced
      st->arrive_push = 0;
      __threadfence_system();
      for (uint32_t r = 0; r < world; ++r) {
        unsigned long long* f = xflag(peers[r], par, rank);
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
      }
    }
  }
}

// every block waits for all ranks' flags of this epoch (acquire), then sums its configs over ranks in rank
// order; the last block to finish advances the local epoch
__global__ void slo_exchange_wait_kernel(const char* window, uint32_t n_cfg, uint32_t world, XState* st,
                                         slo_config_agg* __restrict__ out) {
  const unsigned long long e = *(volatile unsigned long long*)&st->epoch + 1ull;
  const uint32_t par = (uint32_t)(e & 1ull);
  char* base = const_cast<char*>(window);
  if (threadIdx.x < world) {
    const unsigned long long* f = xflag(base, par, threadIdx.x);
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      unsigned long long v, now;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v == e) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > 30000000000ull) {                           // 30 s: a peer never arrived
        atomicOr(&st->error, 1u);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cfg; c += gridDim.x * blockDim.x) {
    slo_config_agg a{0, 0, 0, 0, 0};
    for (uint32_t r = 0; r < world; ++r) {
      const slo_config_agg x = inbox(base, par, world, r, n_cfg)[c];
      a.sum_p99_us += x.sum_p99_us;
      a.sum_slo_met += x.sum_slo_met;
      a.sum_window_us += x.sum_window_us;
      a.n_seeds += x.n_seeds;
      a.flags |= x.flags;
    }
    out[c] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&st->arrive_wait, 1u) == gridDim.x - 1) {       // every block has read the epoch
      st->arrive_wait = 0;
      *(volatile unsigned long long*)&st->epoch = e;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// K4: Philox4x32-10 throughput at full occupancy (the RNG roofline of DESIGN.md §7), keyed per thread,
// counters (iteration, 1, thread, 0) like the SPEC stream; the XOR fold keeps every block live
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) slo_philox_peak_kernel(uint32_t iters, uint32_t* __restrict__ sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t k0 = 0x5EED0000u ^ tid, k1 = 0x9E3779B9u * (tid + 1u);
  uint32_t acc = 0;
#pragma unroll 1
  for (uint32_t q = 0; q < iters; ++q) {
    const u32x4 w = philox(q, 1, tid, 0, k0, k1);
    acc ^= w.x ^ w.y ^ w.z ^ w.w;
  }
  sink[tid] = acc;
}

// ------------------------------------------------------------------------------------------------
// neighbours (host + device)
// ------------------------------------------------------------------------------------------------
__host__ __device__ static inline int32_t dim_get(const slo_knobs& k, int d) {
  switch (d) {
    case 0: return k.conc;
    case 1: return k.max_num_seqs;
    case 2: return k.draft_len;
    case 3: return k.draft_width;
    default: return (int32_t)k.max_wait_us;
  }
}

__host__ __device__ static inline void dim_set(slo_knobs& k, int d, int32_t v) {
  switch (d) {
    case 0: k.conc = (uint8_t)v; break;
    case 1: k.max_num_seqs = (uint8_t)v; break;
    case 2: k.draft_len = (uint8_t)v; break;
    case 3: k.draft_width = (uint8_t)v; break;
    default: k.max_wait_us = (uint32_t)v; break;
  }
}

__host__ __device__ static inline bool knobs_equal(const slo_knobs& a, const slo_knobs& b) {
  const uint32_t* x = reinterpret_cast<const uint32_t*>(&a);
  const uint32_t* y = reinterpret_cast<const uint32_t*>(&b);
  for (int i = 0; i < 8; ++i)
    if (x[i] != y[i]) return false;
  return true;
}

__host__ __device__ static inline int32_t clampi(int32_t v, int32_t lo, int32_t hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

__host__ __device__ static inline void push_unique(const slo_knobs& K, const slo_knobs& c, slo_knobs* out,
                                                   uint32_t& n, uint32_t cap) {
  if (knobs_equal(c, K)) return;
  for (uint32_t i = 0; i < n; ++i)
    if (knobs_equal(out[i], c)) return;
  if (n < cap) out[n++] = c;
}

__host__ __device__ static inline slo_knobs moved(const slo_space& sp, const slo_knobs& K, int d, int sign) {
  slo_knobs c = K;
  dim_set(c, d, clampi(dim_get(K, d) + sign * sp.step[d], sp.lo[d], sp.hi[d]));
  return c;
}

__host__ __device__ uint32_t neighbors_of(const slo_space& sp, const slo_knobs& K, slo_knobs* out, uint32_t cap) {
  uint32_t n = 0;
  slo_knobs toggle = K;
  toggle.spec_on = K.spec_on ? 0 : 1;
  if (sp.stencil == 0) {  // conc, max_num_seqs, draft_len (minus before plus), then the toggle
    for (int d = 0; d < 3; ++d) {
      push_unique(K, moved(sp, K, d, -1), out, n, cap);
      push_unique(K, moved(sp, K, d, +1), out, n, cap);
    }
    push_unique(K, toggle, out, n, cap);
  } else if (sp.stencil == 1) {  // W, k, B, max_wait
    const int order[4] = {3, 2, 1, 4};
    for (int i = 0; i < 4; ++i) {
      push_unique(K, moved(sp, K, order[i], -1), out, n, cap);
      push_unique(K, moved(sp, K, order[i], +1), out, n, cap);
    }
  } else {  // wide-32: 26 non-zero moves of (conc, B, gamma) in lexicographic order, W-/+, wait-/+, toggle
    for (int dc = -1; dc <= 1; ++dc)
      for (int db = -1; db <= 1; ++db)
        for (int dg = -1; dg <= 1; ++dg) {
          if (dc == 0 && db == 0 && dg == 0) continue;
          slo_knobs c = K;
          dim_set(c, 0, clampi(dim_get(K, 0) + dc * sp.step[0], sp.lo[0], sp.hi[0]));
          dim_set(c, 1, clampi(dim_get(K, 1) + db * sp.step[1], sp.lo[1], sp.hi[1]));
          dim_set(c, 2, clampi(dim_get(K, 2) + dg * sp.step[2], sp.lo[2], sp.hi[2]));
          push_unique(K, c, out, n, cap);
        }
    push_unique(K, moved(sp, K, 3, -1), out, n, cap);
    push_unique(K, moved(sp, K, 3, +1), out, n, cap);
    push_unique(K, moved(sp, K, 4, -1), out, n, cap);
    push_unique(K, moved(sp, K, 4, +1), out, n, cap);
    push_unique(K, toggle, out, n, cap);
  }
  return n;
}

// the i-th raw move of neighbors_of's stencil order (i < raw_moves(sp)); a raw move equal to K or to an earlier
// raw move is dropped there
__device__ static inline uint32_t raw_moves(const slo_space& sp) { return sp.stencil == 0 ? 7u : (sp.stencil == 1 ? 8u : 31u); }
__device__ static inline slo_knobs raw_move(const slo_space& sp, const slo_knobs& K, uint32_t i) {
  if (sp.stencil == 0) {                 // conc -, +, max_num_seqs -, +, draft_len -, +, toggle
    if (i == 6) {
      slo_knobs t = K;
      t.spec_on = K.spec_on ? 0 : 1;
      return t;
    }
    return moved(sp, K, (int)(i >> 1), (i & 1) ? +1 : -1);
  }
  if (sp.stencil == 1) {                 // W, k, B, max_wait
    const int order[4] = {3, 2, 1, 4};
    return moved(sp, K, order[i >> 1], (i & 1) ? +1 : -1);
  }
  if (i < 26) {                          // (dc, db, dg) in {-1, 0, 1}^3 \ 0, lexicographic
    const uint32_t v = i < 13 ? i : i + 1;
    const int dc = (int)(v / 9) - 1, db = (int)((v / 3) % 3) - 1, dg = (int)(v % 3) - 1;
    slo_knobs c = K;
    dim_set(c, 0, clampi(dim_get(K, 0) + dc * sp.step[0], sp.lo[0], sp.hi[0]));
    dim_set(c, 1, clampi(dim_get(K, 1) + db * sp.step[1], sp.lo[1], sp.hi[1]));
    dim_set(c, 2, clampi(dim_get(K, 2) + dg * sp.step[2], sp.lo[2], sp.hi[2]));
    return c;
  }
  if (i < 30) return moved(sp, K, i < 28 ? 3 : 4, (i & 1) ? +1 : -1);   // W -, +, max_wait -, +
  slo_knobs t = K;
  t.spec_on = K.spec_on ? 0 : 1;
  return t;
}

// neighbors_of on one warp (every lane calls it; out in shared memory): lane i builds raw move i, keeps it when
// it differs from K and from every raw move before it, and the kept moves are compacted in order (the first cap)
__device__ static uint32_t neighbors_warp(const slo_space& sp, const slo_knobs& K, slo_knobs* out, uint32_t cap) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nraw = raw_moves(sp);
  const bool have = lane < nraw;
  const slo_knobs c = have ? raw_move(sp, K, lane) : K;
  // raw moves differ from K only in words 0 (C, B, gamma, spec_on), 1 (W) and 3 (max_wait)
  const uint32_t* cw = reinterpret_cast<const uint32_t*>(&c);
  const uint32_t* kw = reinterpret_cast<const uint32_t*>(&K);
  bool keep = have && !(cw[0] == kw[0] && cw[1] == kw[1] && cw[3] == kw[3]);
  for (uint32_t j = 0; j + 1 < nraw; ++j) {
    const uint32_t w0 = __shfl_sync(FULL, cw[0], (int)j), w1 = __shfl_sync(FULL, cw[1], (int)j),
                   w3 = __shfl_sync(FULL, cw[3], (int)j);
    if (j < lane && w0 == cw[0] && w1 == cw[1] && w3 == cw[3]) keep = false;
  }
  const uint32_t km = __ballot_sync(FULL, keep);
  const uint32_t pos = __popc(km & ((1u << lane) - 1u));
  __syncwarp();
  if (keep && pos < cap) out[pos] = c;
  __syncwarp();
  const uint32_t n = __popc(km);
  return n < cap ? n : cap;
}

// ------------------------------------------------------------------------------------------------
// K3: one warp; lane k scores candidate k (Eq. 3), warp argmax, Alg. 1 move + best, next stencil.
// ------------------------------------------------------------------------------------------------
__device__ static inline int64_t hw_cost_micro(const slo_knobs& k, const slo_score_params& sp) {
  const int64_t gamma = k.spec_on ? k.draft_len : 0;
  int64_t hw = sp.w_conc_micro * k.conc + sp.w_max_micro * k.max_num_seqs + sp.w_spec_micro * gamma;
  if (gamma > 0) hw += sp.w_W_micro * k.draft_width + sp.w_k_micro * ((int64_t)sp.k_max - gamma);
  return hw;
}

// Eq. (3) in micro-rps; `ema` >= 0 replaces the seed-mean p99 of the violation term (current point of the
// simulator controller); the violation term is multiplied by viol_mult (10 lambda).
__device__ static inline int64_t score_micro(const slo_config_agg& a, const slo_knobs& k, const slo_score_params& sp,
                                             int64_t ema) {
  if (a.n_seeds == 0 || (a.flags & 1u) || a.sum_window_us == 0) return INT64_MIN;
  const unsigned __int128 gp = ((unsigned __int128)a.sum_slo_met * 1000000000000ull) / a.sum_window_us;
  unsigned __int128 pen = 0;
  const unsigned __int128 lam = (unsigned __int128)sp.lambda_milli * sp.viol_mult;
  if (ema >= 0) {
    if ((uint64_t)ema > sp.slo_us) pen = (lam * ((uint64_t)ema - sp.slo_us)) / 1000u;
  } else {
    const unsigned __int128 bound = (unsigned __int128)a.n_seeds * sp.slo_us;
    if ((unsigned __int128)a.sum_p99_us > bound)
      pen = (lam * ((unsigned __int128)a.sum_p99_us - bound)) / ((unsigned __int128)1000u * a.n_seeds);
  }
  return (int64_t)gp - (int64_t)pen - hw_cost_micro(k, sp);
}

// one Alg. 1 step on one warp: lane k < n_cand holds candidate k's pooled aggregate `a` (cands[0] = state.K);
// scores (Eq. 3), argmax over k >= 1 (lowest index on ties), move rule, best-so-far; lane 0 writes the state
// and next[0..n_cand) = [K', neighbours(K'), padding]
__device__ static void climb_core(const slo_space& space, const slo_score_params& sp, const slo_knobs* cands,
                                  uint32_t n_cand, const slo_config_agg& a, slo_climb_state* state, slo_knobs* next,
                                  int64_t* scores) {
  const int lane = threadIdx.x & 31;
  int64_t s = INT64_MIN;
  int64_t ema_new = -1;
  if ((uint32_t)lane < n_cand) {
    const slo_knobs mine = cands[lane];
    int64_t ema = -1;
    if (lane == 0 && sp.ema_beta_q16 > 0 && a.n_seeds > 0 && !(a.flags & 1u)) {  // EMA of p99
      const uint64_t sample = a.sum_p99_us / a.n_seeds;
      const slo_climb_state& st0 = *state;
      ema = st0.has_ema ? (int64_t)((sp.ema_beta_q16 * (unsigned __int128)sample +
                                     (65536u - sp.ema_beta_q16) * (unsigned __int128)st0.ema_p99_us) >> 16)
                        : (int64_t)sample;
    }
    s = score_micro(a, mine, sp, ema);
    if (scores) scores[lane] = s;
    if (lane == 0) ema_new = ema;
  }
  // argmax over k >= 1, lowest index on ties
  int64_t bs = (lane >= 1 && (uint32_t)lane < n_cand) ? s : INT64_MIN;
  int32_t bi = (lane >= 1 && (uint32_t)lane < n_cand) ? lane : 1000;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    const int64_t os = (int64_t)(((uint64_t)__shfl_xor_sync(FULL, (uint32_t)((uint64_t)bs >> 32), d) << 32) |
                                 __shfl_xor_sync(FULL, (uint32_t)(uint64_t)bs, d));
    const int32_t oi = __shfl_xor_sync(FULL, bi, d);
    if (os > bs || (os == bs && oi < bi)) {
      bs = os;
      bi = oi;
    }
  }
  const int64_t s0 = (int64_t)(((uint64_t)__shfl_sync(FULL, (uint32_t)((uint64_t)s >> 32), 0) << 32) |
                               __shfl_sync(FULL, (uint32_t)(uint64_t)s, 0));
  const uint64_t p99sum0 = shfl64(a.sum_p99_us, 0);
  const uint32_t n0 = __shfl_sync(FULL, a.n_seeds, 0);
  __syncwarp();
  if (lane == 0) {
    slo_climb_state st = *state;
    if (!st.has_best || s0 > st.S_best_micro) {
      st.S_best_micro = s0;
      st.K_best = cands[0];
      st.has_best = 1;
    }
    int moved_ = 0;
    uint32_t idx = 0;
    if (ema_new >= 0) {
      st.ema_p99_us = (uint64_t)ema_new;
      st.has_ema = 1;
    }
    if (n_cand > 1) {
      idx = (uint32_t)bi;
      const __int128 diff = (__int128)bs - (__int128)s0;
      const bool violated = ema_new >= 0 ? (uint64_t)ema_new > sp.slo_us
                                         : n0 > 0 && (unsigned __int128)p99sum0 > (unsigned __int128)n0 * sp.slo_us;
      moved_ = (diff >= (__int128)sp.delta_micro) || (violated && bs > s0);
      if (!sp.strict_alg1 && bs > st.S_best_micro) {
        st.S_best_micro = bs;
        st.K_best = cands[idx];
      }
    }
    const slo_knobs K = moved_ ? cands[idx] : cands[0];
    st.K = K;
    st.step += 1;
    st.moved = moved_;
    st.argmax = idx;
    next[0] = K;
    *state = st;
  }
  __syncwarp();
  const slo_knobs K = next[0];                          // [K', neighbours(K'), padding] on the whole warp
  const uint32_t nn = 1 + neighbors_warp(space, K, next + 1, n_cand > 0 ? n_cand - 1 : 0);
  for (uint32_t i = nn + (uint32_t)lane; i < n_cand; i += 32) next[i] = slo_knobs{};   // conc = 0: invalid
  if (lane == 0) state->n_next = nn;
  __syncwarp();
}

__global__ void slo_climb_kernel(slo_space space, slo_score_params sp, slo_knobs* cands, uint32_t n_cand,
                                 const slo_config_agg* aggs, uint32_t n_parts, slo_climb_state* state,
                                 int64_t* scores) {
  const int lane = threadIdx.x & 31;
  __shared__ slo_knobs next[32];
  slo_config_agg a{0, 0, 0, 0, 0};
  if ((uint32_t)lane < n_cand) {
    for (uint32_t p = 0; p < n_parts; ++p) {
      const slo_config_agg x = aggs[(size_t)p * n_cand + lane];
      a.sum_p99_us += x.sum_p99_us;
      a.sum_slo_met += x.sum_slo_met;
      a.sum_window_us += x.sum_window_us;
      a.n_seeds += x.n_seeds;
      a.flags |= x.flags;
    }
  }
  climb_core(space, sp, cands, n_cand, a, state, next, scores);
  if ((uint32_t)lane < n_cand) cands[lane] = next[lane];
}

// ------------------------------------------------------------------------------------------------
// Lookahead climb (SV §8(f) NEXT-4): one round evaluates U(K) = {K} u N(K) u (union of N(c), c in N(K)) — every
// candidate the next two Alg. 1 steps can look at, whatever the first step decides — minus what the previous
// round's U already measured (a candidate's aggregate is a function of its knob record and the seeds only:
// its Philox key is (seed, config key)), then takes two steps from the table.  The trajectory equals the plain
// climb's step for step.
// ------------------------------------------------------------------------------------------------
__device__ static inline uint32_t knob_hash(const slo_knobs& k) {
  const uint32_t* x = reinterpret_cast<const uint32_t*>(&k);
  uint32_t h = 0x811C9DC5u;
  for (int i = 0; i < 8; ++i) h = (h ^ x[i]) * 0x01000193u;
  return h ? h : 1u;                                     // 0 marks an empty slot
}

constexpr int kLookRaw = 1024;   // [K], N(K) (<= 31), N(c) for each c (31 x 31): 993 slots

// block-wide exclusive prefix sum of a 0/1 flag (blockDim.x = 1024); returns the total via *tot
__device__ static inline uint32_t block_excl(bool f, uint32_t* warp_tot, uint32_t* tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t m = __ballot_sync(FULL, f);
  if (lane == 0) warp_tot[w] = __popc(m);
  __syncthreads();
  if (w == 0) {
    const uint32_t v = warp_tot[lane];
    uint32_t incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(FULL, incl, d);
      if (lane >= d) incl += o;
    }
    warp_tot[lane] = incl - v;
    if (lane == 31) *tot = incl;
  }
  __syncthreads();
  const uint32_t r = warp_tot[w] + __popc(m & ((1u << lane) - 1u));
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024) slo_lookahead_prepare_kernel(slo_space space, const slo_climb_state* state,
                                                                      LookTable* T, slo_knobs* sim) {
  __shared__ slo_knobs raw[kLookRaw];
  __shared__ __align__(16) uint32_t rh[kLookRaw];        // slot hashes, 0 = empty slot (valid hashes are != 0)
  __shared__ uint32_t oh[kLookCap];                      // the cache's hashes
  __shared__ uint32_t cnt[32];
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t s_tot;
  const uint32_t t = threadIdx.x;
  const uint32_t wid = t >> 5;
  if (wid == 0) {
    if (t == 0) raw[0] = state->K;
    __syncwarp();
    const uint32_t n1 = neighbors_warp(space, raw[0], raw + 1, 31);
    if (t == 0) cnt[0] = n1;
  }
  __syncthreads();
  const uint32_t nb = cnt[0];
  if (wid >= 1 && wid <= nb) {                           // warp w: the neighbours of raw[w]
    const uint32_t nw = neighbors_warp(space, raw[wid], raw + 32 + (wid - 1) * 31, 31);
    if ((t & 31) == 0) cnt[wid] = nw;
  }
  __syncthreads();
  // slot t holds a candidate: 0 = K, 1..nb = N(K), 32 + 31 (i - 1) + j = the j-th neighbour of raw[i]
  bool valid = t <= nb;
  if (t >= 32) {
    const uint32_t i = 1 + (t - 32) / 31, j = (t - 32) % 31;
    valid = i <= nb && j < cnt[i];
  }
  const uint32_t h = valid ? knob_hash(raw[t]) : 0u;
  rh[t] = h;
  const uint32_t n_old = T->n_old;
  for (uint32_t j = t; j < n_old; j += blockDim.x) oh[j] = T->old_h[j];
  __syncthreads();
  bool first = valid;
  for (uint32_t u0 = 0; first && u0 < t; u0 += 4) {      // an equal record in an earlier slot? (4 hashes a load)
    const uint4 q = *reinterpret_cast<const uint4*>(rh + u0);
    const uint32_t hq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t u = u0 + (uint32_t)k;
      if (u < t && hq[k] == h && knobs_equal(raw[u], raw[t])) first = false;
    }
  }
  const uint32_t pos = block_excl(first, warp_tot, &s_tot);
  const uint32_t n_new = s_tot < kLookCap ? s_tot : kLookCap;
  if (first && pos < kLookCap) {
    T->new_k[pos] = raw[t];
    T->new_h[pos] = h;
  }
  if (t == 0) {
    T->n_new = n_new;
    if (s_tot > kLookCap) T->overflow = s_tot;
  }
  __syncthreads();
  // measured last round?  map[i] >= 0: the old table's entry; < 0: simulation list entry -map - 1
  int32_t m = -1;
  if (t < n_new) {
    const slo_knobs k = T->new_k[t];
    const uint32_t hk = T->new_h[t];
    for (uint32_t j = 0; j < n_old; ++j)
      if (oh[j] == hk && knobs_equal(T->old_k[j], k)) {
        m = (int32_t)j;
        break;
      }
  }
  const bool miss = t < n_new && m < 0;
  const uint32_t sp_ = block_excl(miss, warp_tot, &s_tot);
  if (t < n_new) T->map[t] = miss ? -(int32_t)sp_ - 1 : m;
  if (miss) sim[sp_] = T->new_k[t];
  if (t >= s_tot && t < kLookCap) sim[t] = slo_knobs{};   // padding: conc = 0, invalid, no simulation work
  if (t == 0) T->n_sim = s_tot;
}

__global__ void slo_lookahead_step_kernel(slo_space space, slo_score_params sp, LookTable* T,
                                          const slo_config_agg* aggs, uint32_t n_parts, uint32_t n_cand,
                                          slo_climb_state* state, slo_climb_state* traj) {
  const int lane = threadIdx.x & 31;
  __shared__ slo_knobs cands[32], next[32];
  __shared__ slo_config_agg tab[kLookCap];
  __shared__ uint32_t nh[kLookCap];
  const uint32_t n_new = T->n_new;
  for (uint32_t i = lane; i < n_new; i += 32) nh[i] = T->new_h[i];
  for (uint32_t i = lane; i < n_new; i += 32) {          // the round's table: last round's or just simulated
    const int32_t m = T->map[i];
    slo_config_agg a{0, 0, 0, 0, 0};
    if (m >= 0) {
      a = T->old_a[m];
    } else {
      const uint32_t c = (uint32_t)(-m - 1);
      for (uint32_t p = 0; p < n_parts; ++p) {
        const slo_config_agg x = aggs[(size_t)p * kLookCap + c];
        a.sum_p99_us += x.sum_p99_us;
        a.sum_slo_met += x.sum_slo_met;
        a.sum_window_us += x.sum_window_us;
        a.n_seeds += x.n_seeds;
        a.flags |= x.flags;
      }
    }
    tab[i] = a;
  }
  if (lane == 0) cands[0] = state->K;                   // [K, neighbours(K), padding]: the plain climb's list
  __syncwarp();
  {
    const uint32_t nn = 1 + neighbors_warp(space, cands[0], cands + 1, n_cand - 1);
    for (uint32_t i = nn + (uint32_t)lane; i < n_cand; i += 32) cands[i] = slo_knobs{};
  }
  __syncwarp();
  for (int st = 0; st < 2; ++st) {
    slo_config_agg a{0, 0, 0, 0, 1u};                    // not in U: a padding record (invalid, INT64_MIN)
    if ((uint32_t)lane < n_cand) {
      const slo_knobs k = cands[lane];
      const uint32_t hk = knob_hash(k);
      if (k.conc != 0)
        for (uint32_t j = 0; j < n_new; ++j)
          if (nh[j] == hk && knobs_equal(T->new_k[j], k)) {
            a = tab[j];
            break;
          }
    }
    climb_core(space, sp, cands, n_cand, a, state, next, nullptr);
    if (lane == 0) traj[st] = *state;
    if ((uint32_t)lane < n_cand) cands[lane] = next[lane];
    __syncwarp();
  }
  for (uint32_t i = lane; i < n_new; i += 32) {          // this round's table is the next round's cache
    T->old_k[i] = T->new_k[i];
    T->old_h[i] = T->new_h[i];
    T->old_a[i] = tab[i];
  }
  if (lane == 0) T->n_old = n_new;
}

}  // namespace slo
