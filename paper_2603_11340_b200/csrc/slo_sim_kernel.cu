// slo_sim_kernel.cu — the simulation kernels of libslosim.
//
//  K0 slo_classify_kernel : sorts replicas into work lists by lane-group size and chain kind, each list in 16
//                           cost buckets (longest expected chains first).
//  The split path (default; slo_sim_opts.gen_policy):
//  K1g slo_gen_kernel     : per-request generation at full width — Philox REQ block (arrival increment, P, O,
//                           noise word) and the SPEC blocks that resolve the step count S_i — written as one
//                           16-B record per request.
//  K1s slo_serve_kernel   : the static-batching chain over the records; 32/G replicas per warp (G = 4 .. 32),
//                           completion order and costs by rank counting, own-lane latencies; min(C, B) = 1 by
//                           a 32-request max-plus scan (scan_mode).
//  K1c slo_sim_cont_kernel: continuous (iteration-level) batching, decode iterations fast-forwarded to the next
//                           event (SPLIT: over K1g's records; its warps first run K1e, the min(C, B) = 1 scans).
//  The inline path (gen_policy = 1) and the think-time loops:
//  K1 slo_sim_kernel      : persistent; a warp runs 32/G replicas at once, one per G-lane group, generation
//                           inline, the batch order by a bitonic network.  K1t: its think-time instantiation.
//  K1b slo_select_kernel  : per replica, the exact nearest-rank p99 (p50, p95) of the measured latencies: a
//                           log-scale histogram pass over the row, the selected bucket copied into shared
//                           memory by a second pass and ranked there; writes p99 and goodput.
//
// The event loop is replaced by the closed forms of DESIGN.md §2.6 (equal to the event definition;
// checked bit-exactly against the oracle):
//   s_j = max(a_j, kappa_{j-C});  t_form = max(t_idle, s_h[, min(s_h + max_wait, s_{h+B-1})]);
//   b = min(B, #{j in [h, h+C) : s_j <= t_form});
//   Cum_m = alpha0 S_m + alpha1 sum_{m'} min(S_m', S_m); completion order = order of (S_m, m);
//   S_m depends on request m's own SPEC stream only, so it is resolved at generation;
//   min(C, B) = 1: t_j = max(t_{j-1} + w, a_j + w) + D_j, a max-plus scan.
#include <cstdint>

#include "slo_device.cuh"
#include "slo_internal.h"

#ifdef SLO_K1C_PROF   // profiling builds only (tools/k1c_prof.py): K1c pass statistics
__device__ unsigned long long g_k1c_prof[16];
#define KPROF(i, v) do { if (v) atomicAdd(&g_k1c_prof[i], (unsigned long long)(v)); } while (0)
extern "C" int slo_debug_k1c_prof(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_k1c_prof, sizeof(g_k1c_prof)) != cudaSuccess) return -1;
  if (reset) { unsigned long long z[16] = {}; cudaMemcpyToSymbol(g_k1c_prof, z, sizeof(z)); }
  return 0;
}
#else
#define KPROF(i, v) do { } while (0)
#endif

namespace slo {

// ------------------------------------------------------------------------------------------------
// group-scoped collectives (all 32 lanes execute them; each G-lane group is independent)
// ------------------------------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ uint32_t gballot(bool pred, int lane) {
  const uint32_t m = __ballot_sync(FULL, pred);
  if constexpr (G == 32) {
    return m;
  } else {
    return (m >> (lane & ~(G - 1))) & ((1u << G) - 1u);
  }
}
template <int G>
__device__ __forceinline__ uint32_t gshfl(uint32_t v, int src) {
  return __shfl_sync(FULL, v, src, G);
}
template <int G>
__device__ __forceinline__ uint64_t gshfl64(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(FULL, (uint32_t)v, src, G);
  const uint32_t hi = __shfl_sync(FULL, (uint32_t)(v >> 32), src, G);
  return ((uint64_t)hi << 32) | lo;
}
template <int G>
__device__ __forceinline__ uint64_t gscan64(uint64_t v, int li) {  // inclusive prefix sum
#pragma unroll
  for (int d = 1; d < G; d <<= 1) {
    const uint32_t lo = __shfl_up_sync(FULL, (uint32_t)v, d, G);
    const uint32_t hi = __shfl_up_sync(FULL, (uint32_t)(v >> 32), d, G);
    if (li >= d) v += ((uint64_t)hi << 32) | lo;
  }
  return v;
}
template <int G>
__device__ __forceinline__ uint32_t gmax(uint32_t v) {
#pragma unroll
  for (int m = G / 2; m >= 1; m >>= 1) v = max(v, __shfl_xor_sync(FULL, v, m, G));
  return v;
}
template <int G>
__device__ __forceinline__ uint64_t gmax64(uint64_t v) {
#pragma unroll
  for (int m = G / 2; m >= 1; m >>= 1) {
    const uint32_t lo = __shfl_xor_sync(FULL, (uint32_t)v, m, G);
    const uint32_t hi = __shfl_xor_sync(FULL, (uint32_t)(v >> 32), m, G);
    const uint64_t o = ((uint64_t)hi << 32) | lo;
    v = o > v ? o : v;
  }
  return v;
}
template <int G>
__device__ __forceinline__ uint32_t gmin(uint32_t v) {
#pragma unroll
  for (int m = G / 2; m >= 1; m >>= 1) v = min(v, __shfl_xor_sync(FULL, v, m, G));
  return v;
}
template <int G>
__device__ __forceinline__ uint32_t gsum(uint32_t v) {
#pragma unroll
  for (int m = G / 2; m >= 1; m >>= 1) v += __shfl_xor_sync(FULL, v, m, G);
  return v;
}
template <int G>
__device__ __forceinline__ uint64_t gsum64(uint64_t v) {
#pragma unroll
  for (int m = G / 2; m >= 1; m >>= 1) {
    const uint32_t lo = __shfl_xor_sync(FULL, (uint32_t)v, m, G);
    const uint32_t hi = __shfl_xor_sync(FULL, (uint32_t)(v >> 32), m, G);
    v += ((uint64_t)hi << 32) | lo;
  }
  return v;
}

// ------------------------------------------------------------------------------------------------
// per-replica shared-memory state of one G-lane group
// ------------------------------------------------------------------------------------------------
template <int G>
struct alignas(16) Group {
  static constexpr int RING = 4 * G;  // a, po, w3 for [h, gen) with gen <= h + 3G
  static constexpr int KRING = 4 * G > 64 ? 4 * G : 64;   // kappa for [h - C, h + b): C + b <= 64
  uint64_t a[RING];                   // arrival time of request j at a[j % RING]
  uint64_t kap[KRING];                // kappa_k (k-th completion, ascending) at kap[k % KRING]
  uint32_t po[RING];                  // P | (O << 16)
  uint32_t w3[RING];                  // noise word
  uint16_t ss[RING];                  // S_j: decode steps request j needs (its own draws only, §2.6)
  uint32_t tm1[16];                   // T_a - 1, a = 1..gp
  uint8_t guide[256];                 // A at the top of bucket u >> 24, | 0x80 if a threshold is inside
  uint64_t g[2], rho[2];              // scaled mean gaps, floor((2^64-1)/g)
  uint64_t last;                      // last generated a (kind 0) or tau (kinds 1, 2)
  uint64_t pstart, pD, pU, pLam, nphase, a_w, alpha0, alpha1;
  uint32_t ph, pstate, pre_base, pre_tok, noise, kind, start_state, gp;
  uint32_t k0, k1, wl, pad;
  uint4 knob;                         // C, B, max_wait_us, gamma_eff (kept here, not in registers)
  uint32_t cnt_meas, cnt_incl, stopped, pad3;   // stop rule (§2.14): measured completions, counted ones, done
};

// (a1) set up a newly acquired replica (group-convergent; other groups do not enter)
// (ACCEPT = false: K1s, whose chain never draws acceptance words — K1g resolved every S_i)
template <int G, bool ACCEPT = true, class GR>
__device__ __forceinline__ void setup_replica(GR& R, const DevWorkload& W, const slo_knobs& k, uint32_t k0,
                                              uint32_t k1, uint32_t gamma, uint32_t& gp, int li, uint32_t gmask) {
  gp = 0;
  if constexpr (ACCEPT) gp = accept_thresholds(k.accept_q16, k.draft_width, gamma, R.tm1, li == 0);
  if (li == 0) {
    const uint64_t g0 = W.gap_q16[0] == INF64 ? INF64 : (W.gap_q16[0] << 8) / k.rate_scale_q8;
    const uint64_t g1 = W.gap_q16[1] == INF64 ? INF64 : (W.gap_q16[1] << 8) / k.rate_scale_q8;
    R.g[0] = g0;
    R.g[1] = g1;
    R.rho[0] = g0 == INF64 || g0 == 0 ? 0 : INF64 / g0;   // (g0 = 0: a zero mean think time, kind 4)
    R.rho[1] = g1 == INF64 || g1 == 0 ? 0 : INF64 / g1;
    R.last = 0;
    R.nphase = 0;
    R.kind = W.kind;
    R.start_state = W.start_state;
    uint64_t a0, a1;
    step_coeffs(W.t, gamma, k.draft_width, a0, a1);     // d(n) = alpha0 + alpha1 n (R10, R28)
    R.alpha0 = a0;
    R.alpha1 = a1;
    R.pre_base = W.t.pre_base_us;
    R.pre_tok = W.t.pre_tok_us;
    R.noise = W.t.noise_step_ppm;
    if (W.kind == 1 || W.kind == 2) {
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
  if (li == 0) {
    R.gp = gp;
    R.k0 = k0;
    R.k1 = k1;
    R.cnt_meas = 0;
    R.stopped = 0;
  }
  __syncwarp(gmask);
  if constexpr (ACCEPT) {
    if (gamma > 0) accept_guide(R.tm1, gp, R.guide, (uint32_t)li, G);   // bucket guide for A(u)
  }
  __syncwarp(gmask);
}

// (a3, a7) request i's lengths and decode step count from its REQ block w: P and O through
// the length tables' bucket guides, and S_i = min{s : sum_{j<s} (A(u_{i,j}) + 1) >= O_i}.  With static batches a
// member's j counts its steps within its batch and with continuous batching its own decode iterations, so in
// both models S_i depends on request i's own SPEC stream only and is resolved here, one SPEC block (4 steps)
// per loop trip.  gp = 0 (no speculation, or alpha_eff = 0): A = 0 and S = O.  Shared by the inline
// generation of K1 / K1c and by K1g, so both paths run the same arithmetic.
__device__ __forceinline__ void request_attrs(const DevWorkload& W, const uint32_t* __restrict__ tables,
                                              const uint8_t* guide, const uint32_t* tm1, uint32_t gp, uint32_t i,
                                              uint32_t k0, uint32_t k1, const u32x4& w, uint32_t& P, uint32_t& S) {
  P = length_guided(tables, W.p_off, W.p_goff, W.p_lo, w.y);
  const uint32_t O = length_guided(tables, W.o_off, W.o_goff, W.o_lo, w.z);
  S = O;
  if (gp > 0) {
    uint32_t tok = 0;
    for (uint32_t q = 0;; ++q) {
      const u32x4 b = philox(i, 1, q, 0, k0, k1);
      uint32_t g0 = guide[b.x >> 24], g1 = guide[b.y >> 24];
      uint32_t g2 = guide[b.z >> 24], g3 = guide[b.w >> 24];
      if ((g0 | g1 | g2 | g3) & 0x80u) {           // a threshold inside one of the buckets (rare)
        g0 = accepted_guided(guide, tm1, b.x, gp);
        g1 = accepted_guided(guide, tm1, b.y, gp);
        g2 = accepted_guided(guide, tm1, b.z, gp);
        g3 = accepted_guided(guide, tm1, b.w, gp);
      }
      const uint32_t c1 = tok + (g0 & 0x7Fu) + 1u, c2 = c1 + (g1 & 0x7Fu) + 1u;
      const uint32_t c3 = c2 + (g2 & 0x7Fu) + 1u, c4 = c3 + (g3 & 0x7Fu) + 1u;
      if (c4 >= O) {
        S = 4u * q + 1u + (c1 < O) + (c2 < O) + (c3 < O);
        break;
      }
      tok = c4;
    }
  }
}

// (a2) arrival instants of requests [gen, gen + G) from their increments x: a group scan with
// the carry R.last gives a_i (kind 0) or the operational epoch tau_i (kinds 1, 2), then the bursty Cox time
// change walks the phases in order (kind 1 draws a PHASE block per new phase).  All lanes execute.
template <int G, class GR>
__device__ __forceinline__ uint64_t arrivals(GR& R, const DevWorkload* __restrict__ wls, uint32_t wl, uint32_t k0,
                                             uint32_t k1, uint64_t x, uint32_t i, uint32_t N, bool go, int lane,
                                             int li) {
  __syncwarp();     // the previous call's R.last / phase-state writes are visible to every lane
  const uint32_t kind = go ? R.kind : 0u;
  const uint64_t last = go ? R.last : 0ull;
  const uint64_t sc = last + gscan64<G>(x, li);     // kind 0: a_i; kinds 1, 2: tau_i; kind 3: 0
  const uint64_t newlast = gshfl64<G>(sc, G - 1);
  uint64_t a = sc;
  const bool bursty = go && (kind == 1 || kind == 2);
  if (__any_sync(FULL, bursty)) {                   // bursty: Cox time change, phases advance in order
    uint64_t pLam = 0, pU = 0, pD = 0, pstart = 0, nph = 0;
    uint32_t ph = 0, pstate = 0;
    if (bursty) {
      pLam = R.pLam; pU = R.pU; pD = R.pD; pstart = R.pstart; nph = R.nphase; ph = R.ph; pstate = R.pstate;
    }
    bool done = !(bursty && i < N);
    for (;;) {
      if (!done && sc < pLam + pU) {
        uint64_t off = mulshr(sc - pLam, R.g[pstate], 48);
        if (off > pD - 1) off = pD - 1;
        a = pstart + off;
        done = true;
      }
      const bool grp_open = gballot<G>(!done, lane) != 0;
      if (!__any_sync(FULL, grp_open)) break;
      if (grp_open) {
        pLam += pU;
        pstart += pD;
        ++ph;
        pstate = (R.start_state + ph) & 1u;
        if (R.kind == 1) {
          const u32x4 pw = philox(ph, 2, 0, 0, k0, k1);
          pD = mulshr(exp_q32(pw.x), wls[wl].soj[pstate], 32);
          ++nph;
        } else {
          pD = wls[wl].soj[pstate];
        }
        pU = capacity(pD, R.rho[pstate]);
      }
    }
    __syncwarp();   // every lane has read the phase state above
    if (bursty && li == 0) {
      R.pLam = pLam; R.pU = pU; R.pD = pD; R.pstart = pstart; R.ph = ph; R.pstate = pstate; R.nphase = nph;
    }
  }
  __syncwarp();     // every lane has read R.last
  if (go && li == 0) R.last = newlast;
  return a;
}

// (a2, a3) generate requests [gen, gen + G) for every group with `go` (all lanes execute)
template <int G, class GR>
__device__ __forceinline__ void generate(GR& R, const DevWorkload* __restrict__ wls, uint32_t wl,
                                         const uint32_t* __restrict__ tables, uint32_t k0, uint32_t k1, uint32_t gen,
                                         uint32_t N, uint32_t warmup, bool go, int lane, int li) {
  const uint32_t i = gen + (uint32_t)li;
  const bool valid = go && i < N;
  const uint32_t kind = go ? R.kind : 0u;
  const u32x4 w = philox(i, 0, 0, 0, k0, k1);
  const uint64_t E = valid ? exp_q32(w.x) : 0;
  // kind 0: gaps; kinds 1, 2: operational-time increments; kinds 3, 4 (closed loop): every a_i = 0
  const uint64_t x = kind == 0 ? mulshr(E, go ? R.g[0] : 0ull, 48) : (kind >= 3 ? 0ull : E);
  const uint64_t a = arrivals<G>(R, wls, wl, k0, k1, x, i, N, go, lane, li);
  if (valid) {
    uint32_t P, S;
    request_attrs(wls[wl], tables, R.guide, R.tm1, R.gp, i, k0, k1, w, P, S);
    R.a[i % GR::RING] = a;
    R.po[i % GR::RING] = P;             // (the chain reads P only; O is folded into S)
    R.w3[i % GR::RING] = w.w;
    if (i == warmup) R.a_w = a;
    R.ss[i % GR::RING] = (uint16_t)S;
  }
  __syncwarp();
}

// ------------------------------------------------------------------------------------------------
// K1g: the per-request attributes of the static-batching replicas (split path).  Everything a
// request draws from its own streams — REQ block (arrival increment, P, O, noise word) and the SPEC blocks
// that resolve S_i — is independent of the batch chain, so it is computed here at full width (one thread per
// request, 4 requests per thread, one block per 1,024-request tile of a replica) and handed to K1s as one
// 16-B record per request: {x lo, x hi, P | S << 16, w3} with x = the scaled Poisson gap (kind 0), the
// operational increment E_q (kinds 1, 2) or 0 (closed loop).  K1s keeps only the scan of x, the bursty phase
// walk and the batch chain.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ bool split_static(const slo_knobs& k, const DevWorkload* __restrict__ wl, uint32_t n_wl) {
  return knobs_valid(k, n_wl) && wl[k.workload].kind != 4;   // (K0 put it in one of K1g's lists)
}

// K1g's lists in K1s / K1e / K1c order: static scan, G = 4, 8, 16, 32; continuous scan, G = 4, 8, 16, 32
__device__ __forceinline__ int gen_list(int q) {
  return q == 0 ? kScanList : q == 1 ? kG4List : q <= 4 ? q - 2 : q == 5 ? kCScanList : q == 6 ? kCG4List : q - 4;
}

#ifndef SLO_GEN_MINB
#define SLO_GEN_MINB 3
// K1c refills its 2G-word noise window once more than SLO_CONT_REFILL / 8 of it is used (pooled over the
// warp's groups); with both ITER blocks of a lane drawn together (SLO_CONT_PAIRDRAW) 5 (1.25G) measured best
// on C2-cont (4: +0.8 %, 6: +0.3 %, 7: +1 %); must stay < 8 (an exhausted window would leave K = 0)
#ifndef SLO_CONT_REFILL
#define SLO_CONT_REFILL 5
#endif
static_assert(SLO_CONT_REFILL >= 1 && SLO_CONT_REFILL < 8, "SLO_CONT_REFILL in [1, 7]");
#ifndef SLO_CONT_PAIRDRAW
#define SLO_CONT_PAIRDRAW 1
#endif
#endif
__global__ void __launch_bounds__(kGenThreads, SLO_GEN_MINB) slo_gen_kernel(const SimParams p, uint4* __restrict__ rec) {
  __shared__ uint32_t s_tm1[16];
  __shared__ __align__(16) uint8_t s_guide[kGuideFine];
  // tile = rpt rounds of 256 requests: whole replicas per block in a large launch; a launch with fewer tiles of
  // 2,048 requests than blocks takes one request per thread (C1: eight blocks instead of one)
  const uint32_t tid = threadIdx.x;
  const uint32_t N = p.warmup + p.seg;
  // a block takes whole replicas when the launch has enough of them to fill the grid (the guide is then rebuilt
  // at most once per replica, and no block barrier falls between its tiles); a small launch splits replicas
  // into 2,048-request tiles so every block has work
  // the replicas: this slice of the static split lists (K0's order: longest expected chains first, so the
  // records K1s needs first are written first)
  uint32_t lo[kGenLists + 1];
  lo[0] = 0;
  for (int q = 0; q < kGenLists; ++q) lo[q + 1] = lo[q] + p.counts[gen_list(q)];
  const uint32_t n_rep = lo[kGenLists];
  const uint32_t big = kGenThreads * kGenPerThread;
  const uint32_t rpt = (uint64_t)n_rep * ((N + big - 1) / big) >= gridDim.x ? (uint32_t)kGenPerThread : 1u;
  const uint32_t TILE = kGenThreads * rpt;
  const uint32_t tpr0 = (N + TILE - 1) / TILE;
  const uint32_t tpr = (uint64_t)n_rep >= 2ull * gridDim.x ? 1u : tpr0;   // tiles per replica
  const uint32_t rounds = tpr == 1 ? tpr0 * rpt : rpt;                     // 256-request rounds per tile
  const uint64_t total = (uint64_t)n_rep * tpr;
  uint32_t cur = 0xFFFFFFFFu, gp = 0, kind = 0, wl = 0, gkey = 0xFFFFFFFFu, rl = 0;
  bool spec = false;                                   // gamma_eff > 0: a SPEC stream is consumed (S_i blocks)
  PhiloxKeys K = philox_keys(0, 0);
  const bool count = p.stats && !(p.stop_n | p.stop_t);  // (under a stop rule K1s counts what it simulates)
  unsigned long long steps = 0, blocks = 0;               // member steps (sum of S) and SPEC blocks consumed
  uint64_t g0 = 0;
  bool skip = true;
  for (uint64_t tt = blockIdx.x; tt < total; tt += gridDim.x) {
    const uint32_t en = (uint32_t)(tt / tpr), tile = (uint32_t)(tt - (uint64_t)en * tpr);
    if (en != cur) {                                   // block-uniform: a new replica
      cur = en;
      int q = 0;
      while (en >= lo[q + 1]) ++q;
      const uint32_t r = p.lists[(size_t)gen_list(q) * p.n_chunk + (en - lo[q])];
      rl = r - p.r_base;
      const uint32_t ci = r / p.n_seeds;
      const slo_knobs k = p.cfg[ci];
      skip = !split_static(k, p.wl, p.n_wl);
      if (!skip) {
        wl = k.workload;
        const DevWorkload& W = p.wl[wl];
        const uint64_t seed = p.seeds[r - ci * p.n_seeds];
        const uint32_t cfgkey = p.crn ? W.stream_id : fnv1a_knobs(k);
        K = philox_keys((uint32_t)seed, (uint32_t)(seed >> 32) ^ cfgkey);
        kind = W.kind;
        g0 = kind == 0 ? (W.gap_q16[0] << 8) / k.rate_scale_q8 : 0ull;   // (kind 0: finite, validated)
        const uint32_t gamma = k.spec_on ? k.draft_len : 0u;
        spec = gamma > 0;
        // the guide depends on (alpha, W, gamma) only: rebuilt when they change
        const uint32_t key = gamma == 0 ? 0u : (k.accept_q16 << 7) ^ (k.draft_width << 5) ^ gamma;
        if (key != gkey) {
          gkey = key;
          __syncthreads();                             // the previous guide's reads are done
          gp = accept_thresholds(k.accept_q16, k.draft_width, gamma, s_tm1, tid == 0);
          __syncthreads();
          if (gamma > 0) accept_guide_fine(s_tm1, gp, s_guide, tid, kGenThreads);
          __syncthreads();
          if (gamma > 0) accept_guide_fine_mark(s_tm1, gp, s_guide, tid);
          __syncthreads();
        }
      }
    }
    if (skip) continue;
    const DevWorkload& W = p.wl[wl];
    uint4* out = rec + (size_t)rl * N;
#pragma unroll 1
    for (uint32_t e = 0; e < rounds; ++e) {
      const uint32_t i = tile * TILE + e * kGenThreads + tid;
      if (i >= N) break;
      // REQ block: arrival increment, lengths, noise word
      const u32x4 w = philox_rk(i, 0, 0, 0, K);
      const uint64_t E = exp_q32(w.x);
      const uint64_t x = kind == 0 ? mulshr(E, g0, 48) : (kind >= 3 ? 0ull : E);
      const uint32_t P = length_guided(p.tables, W.p_off, W.p_goff, W.p_lo, w.y);
      const uint32_t O = length_guided(p.tables, W.o_off, W.o_goff, W.o_lo, w.z);
      // S_i = min{s : sum_{j<s} (A(u_{i,j}) + 1) >= O_i}, one SPEC block (4 steps) per trip
      uint32_t S = O;
      if (gp > 0) {
        uint32_t tok = 0;
        // two SPEC blocks per trip (q, q + 1): two independent Philox chains per trip (measured 2 % faster than
        // one); the second block of the last trip is drawn but not consumed when the crossing falls in the first
        // (it is not counted as consumed work)
        for (uint32_t q = 0;; q += 2) {
          const u32x4 ba = philox_rk(i, 1, q, 0, K);
          const u32x4 bb = philox_rk(i, 1, q + 1u, 0, K);
          uint32_t a0 = s_guide[ba.x >> 20], a1 = s_guide[ba.y >> 20], a2 = s_guide[ba.z >> 20], a3 = s_guide[ba.w >> 20];
          uint32_t b0 = s_guide[bb.x >> 20], b1 = s_guide[bb.y >> 20], b2 = s_guide[bb.z >> 20], b3 = s_guide[bb.w >> 20];
          uint32_t sa = a0 + a1 + a2 + a3, sb = b0 + b1 + b2 + b3;   // sums of (A + 1) unless a flag lifts one >= 128
          if ((sa | sb) >= 128u) {                      // a threshold inside one of the buckets (rare)
            a0 = accepted_fine(a0, s_tm1, ba.x, gp) + 1u;
            a1 = accepted_fine(a1, s_tm1, ba.y, gp) + 1u;
            a2 = accepted_fine(a2, s_tm1, ba.z, gp) + 1u;
            a3 = accepted_fine(a3, s_tm1, ba.w, gp) + 1u;
            b0 = accepted_fine(b0, s_tm1, bb.x, gp) + 1u;
            b1 = accepted_fine(b1, s_tm1, bb.y, gp) + 1u;
            b2 = accepted_fine(b2, s_tm1, bb.z, gp) + 1u;
            b3 = accepted_fine(b3, s_tm1, bb.w, gp) + 1u;
            sa = a0 + a1 + a2 + a3;
            sb = b0 + b1 + b2 + b3;
          }
          if (tok + sa >= O) {
            const uint32_t c1 = tok + a0, c2 = c1 + a1, c3 = c2 + a2;
            S = 4u * q + 1u + (c1 < O) + (c2 < O) + (c3 < O);
            break;
          }
          tok += sa;
          if (tok + sb >= O) {
            const uint32_t c1 = tok + b0, c2 = c1 + b1, c3 = c2 + b2;
            S = 4u * q + 5u + (c1 < O) + (c2 < O) + (c3 < O);
            break;
          }
          tok += sb;
        }
      }
      out[i] = make_uint4((uint32_t)x, (uint32_t)(x >> 32), P | (S << 16), w.w);
      steps += S;
      blocks += spec ? (S + 3u) >> 2 : 0u;
    }
  }
  if (count) {
    steps = warp_sum64(steps);
    blocks = warp_sum64(blocks);
    if ((tid & 31) == 0) {
      atomicAdd((unsigned long long*)&p.stats->member_steps, steps);
      atomicAdd((unsigned long long*)&p.stats->philox_blocks, blocks);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// group-scoped sorting networks and scans (K1, K1t, K1c)
// ------------------------------------------------------------------------------------------------
// bitonic sort of u32 keys over the first 2^LG lanes of each G-lane group (ascending)
template <int G, int LG>
__device__ __forceinline__ uint32_t gsort_n(uint32_t key, int li) {
  constexpr int n = (1 << LG) < G ? (1 << LG) : G;
#pragma unroll
  for (int kk = 2; kk <= n; kk <<= 1) {
#pragma unroll
    for (int jj = kk >> 1; jj >= 1; jj >>= 1) {
      const uint32_t other = __shfl_xor_sync(FULL, key, jj, G);
      const bool up = (li & kk) == 0;
      const bool lower = (li & jj) == 0;
      key = (lower == up) ? min(key, other) : max(key, other);
    }
  }
  return key;
}

// inclusive prefix sum over the first 2^LG lanes of each G-lane group
template <int G, int LG>
__device__ __forceinline__ uint32_t gscan_n(uint32_t v, int li) {
  constexpr int n = (1 << LG) < G ? (1 << LG) : G;
#pragma unroll
  for (int d = 1; d < n; d <<= 1) {
    const uint32_t o = __shfl_up_sync(FULL, v, d, G);
    if (li >= d) v += o;
  }
  return v;
}

// bitonic sort of (t, q) pairs over each G-lane group, ascending by t then q (kind 4's pending issues)
template <int G>
__device__ __forceinline__ void gsort_pair(uint64_t& t, uint32_t& q, int li) {
#pragma unroll
  for (int kk = 2; kk <= G; kk <<= 1) {
#pragma unroll
    for (int jj = kk >> 1; jj >= 1; jj >>= 1) {
      const uint32_t olo = __shfl_xor_sync(FULL, (uint32_t)t, jj, G);
      const uint32_t ohi = __shfl_xor_sync(FULL, (uint32_t)(t >> 32), jj, G);
      const uint32_t oq = __shfl_xor_sync(FULL, q, jj, G);
      const uint64_t ot = ((uint64_t)ohi << 32) | olo;
      const bool other_less = ot < t || (ot == t && oq < q);
      const bool keep_min = ((li & kk) == 0) == ((li & jj) == 0);
      if (keep_min ? other_less : !other_less) {   // equal pairs are identical: either choice is the same
        t = ot;
        q = oq;
      }
    }
  }
}

struct Counters {   // lane-local work counters (flushed to slo_stats)
  uint32_t steps, blocks, batches, dsteps;
};

__device__ __forceinline__ void flush_counters(const SimParams& p, Counters& ct) {
  if (p.stats) {
    unsigned long long* st = (unsigned long long*)p.stats;   // requests, batches, dsteps, msteps, blocks
    if (ct.batches) atomicAdd(st + 1, (unsigned long long)ct.batches);
    if (ct.dsteps) atomicAdd(st + 2, (unsigned long long)ct.dsteps);
    if (ct.steps) atomicAdd(st + 3, (unsigned long long)ct.steps);
    if (ct.blocks) atomicAdd(st + 4, (unsigned long long)ct.blocks);
  }
  ct = Counters{0, 0, 0, 0};
}

// ------------------------------------------------------------------------------------------------
// one lane-group mode of K1: groups pull replicas from work list `cls` until it is exhausted
// ------------------------------------------------------------------------------------------------
// THINK (kind 4): issue instants come from the group's C pending user chains, kept sorted in
// the lanes (lane l = the l-th earliest ready instant, with its chain id) instead of s_j = max(a_j, kappa_{j-C})
template <int G, bool STOP, bool THINK>
__device__ __forceinline__ void run_mode(const SimParams& p, int cls, uint8_t* wsmem, int lane, Counters& ct) {
  constexpr int RING = Group<G>::RING;
  const int g = lane / G, li = lane % G;
  Group<G>& R = reinterpret_cast<Group<G>*>(wsmem)[g];
  const uint32_t gmask = (G == 32) ? FULL : (((1u << G) - 1u) << (g * G));
  const uint32_t N = p.warmup + p.seg;
  const uint32_t count = p.counts[cls];
  const uint32_t* list = p.lists + (size_t)cls * p.n_chunk;

  uint32_t r = 0, h = 0, gen = 0, rowoff = 0;   // rowoff = (r - r_base) * N: this replica's latency row
  uint64_t t_idle = 0;
  uint32_t my_slo = 0;
  uint64_t my_sum = 0;
  bool active = false, exhausted = count == 0;      // (an empty list: no cursor atomics)
  uint64_t pq = INF64;        // THINK: this lane's pending ready instant
  uint32_t pid = 0xFFFFFFFFu; // THINK: its user chain id

  bool acq = true;
  for (;;) {
    __syncwarp();   // every lane is past the previous iteration's reads of its group's record
    // ---- acquire replicas for idle groups
    if (acq) {   // acquisition and the exit test only after a replica finished (warp-uniform)
      bool want = !active && !exhausted;
      while (__any_sync(FULL, want)) {
        uint32_t idx = 0;
        if (want && li == 0) idx = atomicAdd(p.cursor + cls, 1u);
        idx = gshfl<G>(idx, 0);
        if (want) {
          if (idx >= count) {
            exhausted = true;
          } else {
            r = list[idx];
            const uint32_t ci = r / p.n_seeds;
            const slo_knobs k = p.cfg[ci];
            if (!knobs_valid(k, p.n_wl)) {  // sentinel outputs
              if (li == 0) {
                p.part[r] = slo_replica_result{0xFFFFFFFFu, 0, 0, 1u, 0, 0};
                if (p.stats) atomicAdd((unsigned long long*)&p.stats->replicas, 1ull);
              }
            } else {
              const DevWorkload& W = p.wl[k.workload];
              const uint64_t seed = p.seeds[r - ci * p.n_seeds];
              const uint32_t cfgkey = p.crn ? W.stream_id : fnv1a_knobs(k);
              const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32) ^ cfgkey;
              const uint32_t gamma = k.spec_on ? k.draft_len : 0u;
              uint32_t gp;
              if (li == 0) {
                R.knob = make_uint4(k.conc, k.max_num_seqs, k.max_wait_us, gamma);
                R.wl = k.workload;
                R.cnt_incl = 0;
              }
              setup_replica<G>(R, W, k, k0, k1, gamma, gp, li, gmask);
              rowoff = (r - p.r_base) * N;           // < 2^32: a chunk's rows are capped by the scratch budget
              h = 0;
              gen = 0;
              t_idle = 0;
              my_slo = 0;
              my_sum = 0;
              if constexpr (THINK) {                 // the first C chains are ready at t = 0
                pq = ((uint32_t)li < k.conc && (uint32_t)li < N) ? 0ull : INF64;
                pid = (uint32_t)li;
              }
              active = true;
            }
          }
        }
        want = !active && !exhausted;
      }
      if (!__any_sync(FULL, active)) break;
      acq = false;
    }
    __syncwarp();   // orders this iteration's ring reads/writes after the previous iteration's (ring reuse)

    // ---- (a2, a3) keep [h, h + G) generated (groups with room generate ahead to share the pass)
    bool need = active && gen < N && gen < h + G;
    while (__any_sync(FULL, need)) {
      const bool go = active && gen < N && gen < h + 3 * G;
      generate<G>(R, p.wl, R.wl, p.tables, R.k0, R.k1, gen, N, p.warmup, go, lane, li);
      if (go) gen += G;
      need = active && gen < N && gen < h + G;
    }

    // ---- (a4) issue times over the window j = h + li: s_j = max(a_j, kappa_{j-C})
    const uint4 kn = R.knob;
    const uint32_t C = kn.x, B = kn.y, mw = kn.z;
    const uint32_t j = h + li;
    uint64_t sj = INF64;
    if constexpr (THINK) {
      if (active) sj = pq;                      // issue order = ready order; INF past the pending chains
    } else if (active && (uint32_t)li < C && j < N) {
      const uint64_t aj = R.a[j % RING];
      const uint64_t kj = j >= C ? R.kap[(j - C) % Group<G>::KRING] : 0;
      sj = aj > kj ? aj : kj;
    }
    // ---- (a5) formation instant and batch size
    const uint64_t sh = gshfl64<G>(sj, 0);
    uint64_t t_form = t_idle > sh ? t_idle : sh;
    // s_{h+B-1}: INF if B > C (the queue never holds B) or beyond N; B <= C implies B <= G (K0: G >= min(C, B))
    const uint64_t slB = gshfl64<G>(sj, (int)(B - 1) & (G - 1));
    const uint64_t sl = B > C ? INF64 : slB;
    if (mw > 0) {                                                 // (mw is group-uniform, not warp-uniform)
      const uint64_t dl = sh + mw;
      const uint64_t x = dl < sl ? dl : sl;
      if (x > t_form) t_form = x;
    }
    uint32_t b = __popc(gballot<G>(sj <= t_form, lane));
    if (b > B) b = B;
    if (!active) b = 0;                     // an idle group has s_j = t_form = INF: no batch
    const bool member = (uint32_t)li < b;
    const uint32_t po = member ? R.po[j % RING] : 0u;

    // ---- (a7) decode: S_m = min{s : sum_{j<s} (A(u_{m,j}) + 1) >= O_m}
    const uint32_t S = member ? (uint32_t)R.ss[j % RING] : 0u;      // resolved at generation
    const bool spec = kn.w > 0;

    // ---- (a6) prefill with the head's noise factor
    const uint64_t f = noise_factor(R.w3[h % RING], R.noise);
    const uint32_t maxP = gmax<G>(po & 0xFFFFu);
    const uint64_t t0 = t_form + f * ((uint64_t)R.pre_base + (uint64_t)R.pre_tok * maxP) / 1000000u;

    // completion order = order of (S, member): at sorted position k,
    // sum_m' min(S_m', S_(k)) = sum_{i<k} S_(i) + (b - k) S_(k)
    // only the first n = 2^ceil(log2 max b) lanes of each group hold members: a bitonic network on n
    // lanes (the first stages of the G-lane network) sorts them, and the prefix sum needs log2 n steps
    const uint32_t bmax = __reduce_max_sync(FULL, b);
    const int lgn = bmax > 1 ? 32 - __clz(bmax - 1u) : 0;
    uint32_t key = member ? (S << 5) | (uint32_t)li : 0xFFFFFFFFu;
    uint32_t incl;
    switch (lgn) {
      case 0: incl = member ? key >> 5 : 0u; break;
      case 1: key = gsort_n<G, 1>(key, li); incl = gscan_n<G, 1>(member ? key >> 5 : 0u, li); break;
      case 2: key = gsort_n<G, 2>(key, li); incl = gscan_n<G, 2>(member ? key >> 5 : 0u, li); break;
      case 3: key = gsort_n<G, 3>(key, li); incl = gscan_n<G, 3>(member ? key >> 5 : 0u, li); break;
      case 4: key = gsort_n<G, 4>(key, li); incl = gscan_n<G, 4>(member ? key >> 5 : 0u, li); break;
      default: key = gsort_n<G, 5>(key, li); incl = gscan_n<G, 5>(member ? key >> 5 : 0u, li); break;
    }
    const uint32_t Sk = member ? key >> 5 : 0u;
    const uint32_t orig = key & 31u;
    const uint32_t summin = incl - Sk + (b - (uint32_t)li) * Sk;
    const uint64_t cum = R.alpha0 * Sk + R.alpha1 * summin;
    const uint64_t c = t0 + (f * cum) / 1000000u;
    if (member) R.kap[(h + li) % Group<G>::KRING] = c;
    if constexpr (THINK) {
      // completion h + li (sorted position li) starts chain h + li + C, ready Z later (THINK block h + li);
      // it takes the place of the pending entry lane li just batched, then the pending list is re-sorted
      const uint32_t kord = h + (uint32_t)li;
      const bool spawn = member && kord + C < N;
      uint64_t z = 0;
      if (spawn) z = mulshr(exp_q32(philox(kord, 4, 0, 0, R.k0, R.k1).x), R.g[0], 48);
      if (member) {
        pq = spawn ? c + z : INF64;
        pid = spawn ? kord + C : 0xFFFFFFFFu;
      }
      gsort_pair<G>(pq, pid, li);
      ct.blocks += spawn ? 1u : 0u;
    }
    const int lastm = (int)(b > 0 ? b - 1 : 0);
    const uint64_t tend = gshfl64<G>(c, lastm);
    const uint32_t maxS = gshfl<G>(Sk, lastm);

    // ---- (a8) latency of the member at sorted position k; SLO count, sum, HBM row for the p99
    const uint32_t i = h + orig;
    const bool measured = member && i >= p.warmup;
    // latency origin: arrival (open loop, R2) or issue (closed loop, §2.11: s_i sits in window lane orig)
    const uint64_t s_orig = gshfl64<G>(sj, (int)orig);
    const bool from_issue = R.kind >= 3;
    if (from_issue && member && i == p.warmup) R.a_w = s_orig;     // the goodput window starts at that issue
    const uint64_t l = c - (member ? (from_issue ? s_orig : R.a[i % RING]) : c);
    // stop rule (§2.14): this batch's measured completions in sorted (= time) order continue the count;
    // the first one that is the k-th with k >= n_min and ends >= t0 + t_min is t*, and only c <= t* counts
    bool inc = true;
    if constexpr (STOP) {                           // compiled into the stop-rule kernels only
      __syncwarp();                                 // R.a_w of a closed-loop warmup issue written above
      const uint32_t mm = gballot<G>(measured, lane);
      const uint32_t before = active ? R.cnt_meas : 0u;
      const uint32_t kpos = before + __popc(mm & ((1u << li) - 1u)) + 1u;
      const uint32_t need = p.stop_n ? p.stop_n : 1u;
      const bool cand = active && !R.stopped && measured && kpos >= need && c >= R.a_w + p.stop_t;
      const uint32_t cmk = gballot<G>(cand, lane);
      const uint64_t tstar = gshfl64<G>(c, (int)((cmk ? __ffs(cmk) - 1 : 0) & (G - 1)));
      inc = cmk == 0 || c <= tstar;
      const uint32_t ninc = __popc(gballot<G>(measured && inc, lane));
      __syncwarp();
      if (active && li == 0) {
        R.cnt_meas = before + __popc(mm);
        R.cnt_incl += ninc;
        if (cmk) R.stopped = 1;
      }
    }
    if (measured && inc) {
      my_slo += (l <= p.slo_us);
      my_slo |= (l > 0xFFFFFFFFull) ? 0x80000000u : 0u;
      my_sum += l;
    }
    if (member) p.lat[rowoff + i] = !inc ? 0xFFFFFFFFu : (l > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)l);

    // work counters, lane-local
    ct.steps += Sk;
    ct.blocks += spec ? (Sk + 3u) >> 2 : 0u;
    if (active && li == 0) {
      ct.batches += 1;
      ct.dsteps += maxS;
    }
    if (active) {
      t_idle = tend;
      h += b;
    }
    if constexpr (STOP) {                           // stopped: the rest of the segment is never simulated
      __syncwarp();
      if (active && R.stopped) {
        for (uint32_t j = h + (uint32_t)li; j < N; j += G) p.lat[rowoff + j] = 0xFFFFFFFFu;
        h = N;
      }
    }

    // ---- groups that finished their replica: outputs (p99 and goodput follow in K1b)
    const bool fin = active && h >= N;
    if (__any_sync(FULL, fin)) {
      const uint32_t slo_met = gsum<G>(my_slo & 0x7FFFFFFFu);
      const uint64_t sum = gsum64<G>(my_sum);
      const bool sat = gballot<G>((my_slo >> 31) != 0, lane) != 0;
      // the window ends at the last MEASURED completion (§2.8): all earlier batches ended before this one
      // formed, so it is the largest c among this last batch's measured members (not t_idle, which may be
      // a warmup member's completion when the segment is shorter than the batch)
      const uint64_t cm = gmax64<G>(measured && inc ? c : 0ull);
      if (fin && li == 0) {
        const uint64_t Tw = cm - R.a_w;
        const uint32_t fl = (sat ? 2u : 0u) | (STOP && !R.stopped ? 4u : 0u);
        p.part[r] = slo_replica_result{0, slo_met, STOP ? R.cnt_incl : p.seg, fl, Tw < 1 ? 1 : Tw, sum};
        if (p.stats) {
          unsigned long long* st = (unsigned long long*)p.stats;
          atomicAdd(st + 0, (unsigned long long)N);
          atomicAdd(st + 4, (unsigned long long)(N + R.nphase));
          atomicAdd(st + 5, 1ull);
        }
      }
      if (fin) active = false;
      acq = true;                                       // (the only way a group goes idle)
    }
    if (ct.steps >= 0x40000000u || ct.dsteps >= 0x40000000u) flush_counters(p, ct);  // rare
  }
}

// ------------------------------------------------------------------------------------------------
// K1s: the static-batching batch chain over K1g's request records (split path).
//
// Generation (Philox, E_q, lengths, S_i) already happened in K1g, so a batch iteration is only the chain of
// §2.6's closed forms.  Per batch, lane li of a group holds request j = h + li of the issue window:
//   s_j = max(a_j, kappa_{j-C}); t_form and b from two shuffles and a ballot (as K1);
//   completion order and cumulative cost by RANK COUNTING instead of a sorting network: every member shuffles in
//   the packed words w_m = S_m << 18 | m << 13 | P_m of the members (distinct, ordered by (S, m)), and
//     rank_li = #{m < b : w_m < w_li}            (its completion index: kappa_{h + rank} = c_li),
//     sum_m min(S_m, S_li) = sum_m (min(w_m, w_li) >> 18),  max P, max S, sum S  (prefill, batch end);
//   so every lane computes its OWN completion c_li = t0 + f (alpha0 S + alpha1 sum min) / 10^6 and latency,
//   stored in request order (no permutation shuffles), and the batch end t_end = c of the largest S.
// Records are register-staged one refill ahead (a refill falls at least one batch after its load was issued).
// A launch with few replicas spreads them over more warps (p.gpw groups per warp): the chain is latency-bound,
// so one replica per warp on an otherwise idle scheduler runs fastest.
// ------------------------------------------------------------------------------------------------
template <int G>
struct alignas(16) SGroup {
  static constexpr int RING = 4 * G;                  // a, w, f for [h, gen), gen <= h + 2G
  static constexpr int KRING = 4 * G > 64 ? 4 * G : 64;   // kappa for [h - C, h + b): C + b <= 64
  uint64_t a[RING];                                   // arrival time a_j at a[j % RING]
  uint64_t kap[KRING];                                // kappa_k (k-th completion) at kap[k % KRING]
  uint32_t w[RING];                                   // S_j << 18 | P_j (the lane index is or-ed in at use)
  uint32_t f[RING];                                   // noise factor of request j as a batch head (ppm, §2.4)
  uint64_t g[2], rho[2];                              // arrival-process state (arrivals(), setup_replica())
  uint64_t last, pstart, pD, pU, pLam, nphase, a_w, alpha0, alpha1;
  uint32_t ph, pstate, pre_base, pre_tok, noise, kind, start_state, gp;
  uint32_t k0, k1, wl, cnt_meas, cnt_incl, stopped;
};

template <int G, bool STOP>
__device__ __forceinline__ void serve_mode(const SimParams& p, int cls, uint8_t* wsmem, int lane, Counters& ct) {
  using SG = SGroup<G>;
  constexpr int RING = SG::RING, KRING = SG::KRING;
  const int g = lane / G, li = lane % G;
  SG& R = reinterpret_cast<SG*>(wsmem)[g];
  const uint32_t gmask = (G == 32) ? FULL : (((1u << G) - 1u) << (g * G));
  const uint32_t N = p.warmup + p.seg;
  const uint32_t count = p.counts[cls];
  const uint32_t* list = p.lists + (size_t)cls * p.n_chunk;

  uint32_t r = 0, h = 0, gen = 0, rowoff = 0;          // rowoff = (r - r_base) * N: the replica's row
  uint32_t C = 0, B = 0, mw = 0, pre_base = 0, pre_tok = 0, noise = 0;
  uint64_t alpha0 = 0, alpha1 = 0, t_idle = 0, my_sum = 0;
  uint32_t my_slo = 0;
  unsigned long long dsteps = 0;                       // decode steps (sum over batches of max S), lane 0
  bool active = false, exhausted = (uint32_t)g >= p.gpw || count == 0, closed = false, spec = false;
  uint4 stg{0, 0, 0, 0};                               // K1g record of request gen + li, loaded ahead

  bool acq = true;
  for (;;) {
    __syncwarp();
    // ---- acquire replicas for idle groups
    if (acq) {   // acquisition and the exit test only after a replica finished (warp-uniform)
      bool want = !active && !exhausted;
      while (__any_sync(FULL, want)) {
        uint32_t idx = 0;
        if (want && li == 0) idx = atomicAdd(p.cursor + cls, 1u);
        idx = gshfl<G>(idx, 0);
        if (want) {
          if (idx >= count) {
            exhausted = true;
          } else {
            r = list[idx];
            const uint32_t ci = r / p.n_seeds;
            const slo_knobs k = p.cfg[ci];
            if (!knobs_valid(k, p.n_wl)) {  // sentinel outputs
              if (li == 0) {
                p.part[r] = slo_replica_result{0xFFFFFFFFu, 0, 0, 1u, 0, 0};
                if (p.stats) atomicAdd((unsigned long long*)&p.stats->replicas, 1ull);
              }
            } else {
              const DevWorkload& W = p.wl[k.workload];
              const uint64_t seed = p.seeds[r - ci * p.n_seeds];
              const uint32_t cfgkey = p.crn ? W.stream_id : fnv1a_knobs(k);
              const uint32_t gamma = k.spec_on ? k.draft_len : 0u;
              uint32_t gp;
              if (li == 0) {
                R.wl = k.workload;
                R.cnt_incl = 0;
              }
              setup_replica<G, false>(R, W, k, (uint32_t)seed, (uint32_t)(seed >> 32) ^ cfgkey, gamma, gp, li, gmask);
              C = k.conc;
              B = k.max_num_seqs;
              mw = k.max_wait_us;
              spec = gamma > 0;
              closed = W.kind >= 3;
              pre_base = W.t.pre_base_us;
              pre_tok = W.t.pre_tok_us;
              noise = W.t.noise_step_ppm;
              step_coeffs(W.t, gamma, k.draft_width, alpha0, alpha1);   // d(n) = alpha0 + alpha1 n (R10, R28)
              rowoff = (r - p.r_base) * N;
              stg = (uint32_t)li < N ? __ldcs(p.rec + rowoff + li) : uint4{0, 0, 0, 0};
              h = 0;
              gen = 0;
              t_idle = 0;
              my_slo = 0;
              my_sum = 0;
              active = true;
            }
          }
        }
        want = !active && !exhausted;
      }
      if (!__any_sync(FULL, active)) break;
      acq = false;
    }
    __syncwarp();

    // ---- (a2) keep [h, h + G) in the ring, up to 2G ahead: scan of the increments, bursty time change
    bool need = active && gen < N && gen < h + G;
    while (__any_sync(FULL, need)) {
      const bool go = active && gen < N && gen < h + 2 * G;
      const uint32_t i = gen + (uint32_t)li;
      const bool valid = go && i < N;
      const uint64_t x = valid ? (((uint64_t)stg.y << 32) | stg.x) : 0ull;
      const uint64_t a = arrivals<G>(R, p.wl, R.wl, R.k0, R.k1, x, i, N, go, lane, li);
      if (valid) {
        R.a[i % RING] = a;
        R.w[i % RING] = ((stg.z >> 16) << 18) | (stg.z & 0xFFFFu);
        R.f[i % RING] = noise_factor(stg.w, noise);
        if (i == p.warmup) R.a_w = a;
      }
      if (go) {
        gen += G;
        if (gen + (uint32_t)li < N) stg = __ldcs(p.rec + rowoff + gen + li);
      }
      need = active && gen < N && gen < h + G;
    }
    __syncwarp();

    // ---- (a4) issue window j = h + li: s_j = max(a_j, kappa_{j-C})
    const uint32_t j = h + (uint32_t)li;
    uint64_t sj = INF64, aj = 0;
    uint32_t wj = 0xFFFFE000u;                         // not a member: above every real word, P = 0
    if (active && j < N) {
      aj = R.a[j % RING];
      wj = R.w[j % RING] | ((uint32_t)li << 13);
      if ((uint32_t)li < C) {
        const uint64_t kj = j >= C ? R.kap[(j - C) % KRING] : 0;
        sj = aj > kj ? aj : kj;
      }
    }
    // ---- (a5) formation instant and batch size (DESIGN.md §2.6 closed form 2)
    const uint64_t sh = gshfl64<G>(sj, 0);
    const uint64_t slB = gshfl64<G>(sj, (int)(B - 1) & (G - 1));
    uint64_t t_form = t_idle > sh ? t_idle : sh;
    if (mw > 0) {
      const uint64_t sl = B > C ? INF64 : slB;
      const uint64_t dl = sh + mw;
      const uint64_t x = dl < sl ? dl : sl;
      if (x > t_form) t_form = x;
    }
    uint32_t b = __popc(gballot<G>(sj <= t_form, lane));
    if (b > B) b = B;
    if (!active) b = 0;
    const bool member = (uint32_t)li < b;

    // ---- (a6, a7) rank counting over the members' words: rank = #{m < b : w_m < w_li}, lts = the S of those
    // m; then sum_m min(S_m, S_li) = lts + S_li (b - rank) and the batch ends with the largest key (rank b - 1)
    const uint32_t S = wj >> 18;
    uint32_t rank = 0, lts = 0, mrank = 0;
    uint32_t maxP = 0;
    auto rank_step = [&](uint32_t m) {
      const uint32_t wm = __shfl_sync(FULL, wj, (int)(m & (G - 1)), G);
      const bool in = m < b, lt = in && wm < wj;
      rank += lt ? 1u : 0u;
      lts += lt ? wm >> 18 : 0u;
      if (G <= 8) maxP = max(maxP, in ? wm & 0x1FFFu : 0u);     // (wider groups: one reduction below)
      if (STOP) mrank += lt && h + m >= p.warmup;   // measured completions before this one
    };
    if constexpr (G <= 8) {                            // straight-line (the shuffles do not wait for b)
#pragma unroll
      for (int m = 0; m < G; ++m) rank_step((uint32_t)m);
    } else {                                           // four members per trip up to the warp's largest batch
      const uint32_t bmax = __reduce_max_sync(FULL, b);
      for (uint32_t m0 = 0; m0 < bmax; m0 += 4) {
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u) rank_step(m0 + u);
      }
      maxP = gmax<G>(member ? wj & 0x1FFFu : 0u);
    }
    const uint64_t f = R.f[h % RING];                  // the head's noise factor
    // f times the cost coefficients (known at the batch head, off the rank -> completion chain); the sums are
    // the same integers as f (pre_base + pre_tok maxP) and f (alpha0 S + alpha1 summin)
    const uint64_t fpb = f * pre_base, fpt = f * pre_tok, fa0 = f * alpha0, fa1 = f * alpha1;
    const uint64_t t0 = t_form + (fpb + fpt * maxP) / 1000000u;
    const uint32_t summin = lts + S * (b - rank);
    const uint64_t c = t0 + (fa0 * S + fa1 * summin) / 1000000u;
    if (member) R.kap[(h + rank) % KRING] = c;
    const uint32_t lastm = gballot<G>(member && rank + 1u == b, lane);
    const int ll = lastm ? __ffs(lastm) - 1 : 0;
    const uint64_t tend = gshfl64<G>(c, ll);           // the largest completion: the batch end
    const uint32_t Smax = gshfl<G>(S, ll);

    // ---- (a8) this lane's own latency: from arrival (open loop, R2) or issue (closed loop, §2.11)
    const bool measured = member && j >= p.warmup;
    if (closed && member && j == p.warmup) R.a_w = sj;   // the goodput window starts at that issue
    const uint64_t l = c - (closed ? sj : aj);
    bool inc = true;
    if constexpr (STOP) {                              // stop rule (§2.14), completion order = rank order
      __syncwarp();                                    // R.a_w of a closed-loop warmup issue written above
      const uint32_t mm = gballot<G>(measured, lane);
      const uint32_t before = active ? R.cnt_meas : 0u;
      const uint32_t kpos = before + mrank + 1u;
      const uint32_t need_n = p.stop_n ? p.stop_n : 1u;
      const bool cand = active && !R.stopped && measured && kpos >= need_n && c >= R.a_w + p.stop_t;
      const uint32_t rmin = gmin<G>(cand ? rank : 0xFFFFFFFFu);
      const uint32_t cmk = gballot<G>(cand && rank == rmin, lane);
      const uint64_t tstar = gshfl64<G>(c, (int)((cmk ? __ffs(cmk) - 1 : 0) & (G - 1)));
      inc = cmk == 0 || c <= tstar;
      const uint32_t ninc = __popc(gballot<G>(measured && inc, lane));
      __syncwarp();
      if (active && li == 0) {
        R.cnt_meas = before + __popc(mm);
        R.cnt_incl += ninc;
        if (cmk) R.stopped = 1;
      }
    }
    if (measured && inc) {
      my_slo += (l <= p.slo_us);
      my_slo |= (l > 0xFFFFFFFFull) ? 0x80000000u : 0u;
      my_sum += l;
    }
    if (member) p.lat[rowoff + j] = !inc ? 0xFFFFFFFFu : (l > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)l);

    // work counters, lane-local (member steps and SPEC blocks are counted by K1g, except under a stop rule,
    // where only what was simulated counts)
    if constexpr (STOP) {
      if (member) {
        ct.steps += S;
        ct.blocks += spec ? (S + 3u) >> 2 : 0u;
      }
    }
    if (active && li == 0) {
      ct.batches += 1;
      dsteps += Smax;
    }
    if (active) {
      t_idle = tend;
      h += b;
    }
    if constexpr (STOP) {                              // stopped: the rest of the segment is never simulated
      __syncwarp();
      if (active && R.stopped) {
        for (uint32_t jj = h + (uint32_t)li; jj < N; jj += G) p.lat[rowoff + jj] = 0xFFFFFFFFu;
        h = N;
      }
    }

    // ---- groups that finished their replica: outputs (p99 and goodput follow in K1b)
    const bool fin = active && h >= N;
    if (__any_sync(FULL, fin)) {
      const uint32_t slo_met = gsum<G>(my_slo & 0x7FFFFFFFu);
      const uint64_t sum = gsum64<G>(my_sum);
      const bool sat = gballot<G>((my_slo >> 31) != 0, lane) != 0;
      // the window ends at the last MEASURED completion (§2.8): the largest c among this last batch's measured
      // members (every earlier batch ended before this one formed)
      const uint64_t cm = gmax64<G>(measured && inc ? c : 0ull);
      if (fin && li == 0) {
        const uint64_t Tw = cm - R.a_w;
        const uint32_t fl = (sat ? 2u : 0u) | (STOP && !R.stopped ? 4u : 0u);
        p.part[r] = slo_replica_result{0, slo_met, STOP ? R.cnt_incl : p.seg, fl, Tw < 1 ? 1 : Tw, sum};
        if (p.stats) {
          unsigned long long* st = (unsigned long long*)p.stats;
          atomicAdd(st + 0, (unsigned long long)N);
          atomicAdd(st + 4, (unsigned long long)(N + R.nphase));
          atomicAdd(st + 5, 1ull);
        }
      }
      if (fin) active = false;
      acq = true;                                       // (the only way a group goes idle)
    }
    if (STOP && ct.steps >= 0x40000000u) flush_counters(p, ct);  // rare
  }
  if (p.stats && dsteps) atomicAdd((unsigned long long*)&p.stats->decode_steps, dsteps);
}

// ------------------------------------------------------------------------------------------------
// K1s scan mode (list 12): static batching with min(C, B) = 1.  Every batch is the single request at the head,
// batch j is request j and completions come in index order, so with t_j = c_j:
//   s_j = max(a_j, t_{j-C}) and t_form_j = max(t_{j-1}, s_j + w), w = max_wait if B > C (= 1) else 0, hence
//   t_j = max(t_{j-1} + w, a_j + w) + D_j,  D_j = floor(f_j (pre_base + pre_tok P_j) / 10^6)
//                                                + floor(f_j (alpha0 + alpha1) S_j / 10^6)
// (t_{j-C} <= t_{j-1}; for B = 1 the max_wait term vanishes because s_{h+B-1} = s_h; for C = 1 < B the queue
// never reaches B and the batch forms at s_h + max_wait).  x -> max(x + A, Bv) maps compose associatively,
// (A1, B1) then (A2, B2) = (A1 + A2, max(B1 + A2, B2)), so a warp resolves 32 requests per step with a
// 5-stage max-plus scan instead of 32 dependent batch iterations.  One replica per warp (G = 32).
// CONT (list 14, continuous batching §2.12 with min(C, B) = 1): the running set never holds more than one
// request, so request j runs alone — a prefill, then its S_j decode iterations it_j .. it_j + S_j - 1 of the
// replica's decode counter (it_j = S_0 + .. + S_{j-1}, an exclusive scan) — and the same recursion holds with
// w = 0 and D_j = floor(f_j (pre_base + pre_tok P_j) / 10^6) + sum_k floor(f_ITER(it_j + k) d(1) / 10^6): each
// lane sums its request's iterations (one ITER Philox block each, the §2.12 draws).
// ------------------------------------------------------------------------------------------------
template <bool STOP, bool CONT = false>
__device__ __forceinline__ void scan_mode(const SimParams& p, int cls, uint8_t* wsmem, int lane, Counters& ct) {
  SGroup<32>& R = *reinterpret_cast<SGroup<32>*>(wsmem);  // arrival-process state (arrivals(), setup_replica())
  const uint32_t N = p.warmup + p.seg;
  const uint32_t count = p.counts[cls];
  const uint32_t* list = p.lists + (size_t)cls * p.n_chunk;
  if (count == 0) return;                             // (an empty list: no cursor atomics)
  for (;;) {
    uint32_t idx = 0;
    if (lane == 0) idx = atomicAdd(p.cursor + cls, 1u);
    idx = __shfl_sync(FULL, idx, 0);
    if (idx >= count) break;
    const uint32_t r = list[idx];
    const uint32_t ci = r / p.n_seeds;
    const slo_knobs k = p.cfg[ci];                     // (K0 lists valid records only here)
    const DevWorkload& W = p.wl[k.workload];
    const uint64_t seed = p.seeds[r - ci * p.n_seeds];
    const uint32_t cfgkey = p.crn ? W.stream_id : fnv1a_knobs(k);
    const uint32_t gamma = k.spec_on ? k.draft_len : 0u;
    uint32_t gp;
    __syncwarp();
    if (lane == 0) R.wl = k.workload;
    setup_replica<32, false>(R, W, k, (uint32_t)seed, (uint32_t)(seed >> 32) ^ cfgkey, gamma, gp, lane, FULL);
    const uint32_t C = k.conc;
    const uint64_t w = (!CONT && k.max_num_seqs > k.conc) ? (uint64_t)k.max_wait_us : 0ull;
    const bool closed = W.kind >= 3, spec = gamma > 0;
    const uint32_t pre_base = W.t.pre_base_us, pre_tok = W.t.pre_tok_us, noise = W.t.noise_step_ppm;
    uint64_t alpha0, alpha1;
    step_coeffs(W.t, gamma, k.draft_width, alpha0, alpha1);
    const uint64_t alpha = alpha0 + alpha1;           // d(1): one active sequence
    const uint32_t rowoff = (r - p.r_base) * N;
    const uint4* rec = p.rec + rowoff;
    uint4 stg = (uint32_t)lane < N ? __ldcs(rec + lane) : uint4{0, 0, 0, 0};
    uint64_t carry = 0;                                // t_{base - 1} (t_{-1} = 0: the idle server at t = 0)
    uint32_t itc = 0;                                  // CONT: decode iterations before this step's requests
    uint64_t tprev = 0;                                // t of request (base - 32 + lane)
    uint64_t a_w = 0, my_sum = 0, tlast = 0, tstar = 0;
    uint32_t my_slo = 0, nmeas = 0, jstar = 0xFFFFFFFFu;
    unsigned long long steps = 0, blocks = 0, dsteps = 0, batches = 0;
    bool stopped = false;
    for (uint32_t base = 0; base < N && !stopped; base += 32) {
      const uint32_t i = base + (uint32_t)lane;
      const bool valid = i < N;
      const uint4 rc = stg;
      if (base + 32u + (uint32_t)lane < N) stg = __ldcs(rec + base + 32u + lane);   // next step's records
      const uint64_t x = valid ? (((uint64_t)rc.y << 32) | rc.x) : 0ull;
      const uint64_t a = arrivals<32>(R, p.wl, R.wl, R.k0, R.k1, x, i, N, true, lane, lane);
      const uint32_t P = rc.z & 0xFFFFu, S = rc.z >> 16;
      const uint64_t f = noise_factor(rc.w, noise);
      uint64_t D = f * ((uint64_t)pre_base + (uint64_t)pre_tok * P) / 1000000u;
      if constexpr (CONT) {                             // S_j decode iterations alone, each with its ITER noise
        uint32_t Sv = valid ? S : 0u, ex = Sv;          // exclusive scan of S over the lanes
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t o = __shfl_up_sync(FULL, ex, d);
          if (lane >= d) ex += o;
        }
        const uint32_t it0 = itc + ex - Sv;
        itc += __shfl_sync(FULL, ex, 31);
        const uint32_t d1 = (uint32_t)alpha;            // d(1) < 2^31 (create-time check)
        if (noise == 0) {
          D += (uint64_t)d1 * Sv;
        } else {
          for (uint32_t q = 0; q < Sv; ++q)
            D += (uint64_t)noise_factor(philox(it0 + q, 3, 0, 0, R.k0, R.k1).x, noise) * d1 / 1000000u;
        }
      } else {
        D += f * (alpha * S) / 1000000u;
      }
      // inclusive max-plus scan of (A, Bv) = (w + D, a + w + D); invalid lanes carry the identity (0, 0)
      uint64_t A = valid ? w + D : 0ull, Bv = valid ? a + w + D : 0ull;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t Ao = shfl_up64(A, d), Bo = shfl_up64(Bv, d);
        if (lane >= d) {
          const uint64_t nb = Bo + A;
          Bv = nb > Bv ? nb : Bv;
          A += Ao;
        }
      }
      const uint64_t ca = carry + A;
      const uint64_t t = ca > Bv ? ca : Bv;             // t_i = c_i
      carry = shfl64(t, 31);                            // (invalid lanes keep the last valid t)
      // issue instant s_i = max(a_i, t_{i-C}) (closed loops measure latency from it, §2.11)
      const int src = lane - (int)C;
      const uint64_t tc_in = shfl64(t, src & 31), tc_prev = shfl64(tprev, src & 31);
      const uint64_t tC = i < C ? 0ull : (src >= 0 ? tc_in : tc_prev);
      const uint64_t si = a > tC ? a : tC;
      if (p.warmup >= base && p.warmup < base + 32u) a_w = shfl64(closed ? si : a, (int)(p.warmup - base));
      const bool measured = valid && i >= p.warmup;
      const uint64_t l = t - (closed ? si : a);
      bool inc = true;
      if constexpr (STOP) {                            // stop rule (§2.14): completion order = index order
        const uint32_t need = p.stop_n ? p.stop_n : 1u;
        const bool cand = measured && i - p.warmup + 1u >= need && t >= a_w + p.stop_t;
        const uint32_t cm = __ballot_sync(FULL, cand);
        if (cm) {
          const int fl = __ffs(cm) - 1;
          jstar = base + (uint32_t)fl;
          tstar = shfl64(t, fl);
          stopped = true;
        }
        inc = i <= jstar;
      }
      if (measured && inc) {
        my_slo += (l <= p.slo_us);
        my_slo |= (l > 0xFFFFFFFFull) ? 0x80000000u : 0u;
        my_sum += l;
        ++nmeas;
      }
      if (valid) p.lat[rowoff + i] = !inc ? 0xFFFFFFFFu : (l > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)l);
      if (valid && inc) {                               // work counters: one batch (prefill) per request
        ++batches;
        dsteps += S;
        if (CONT && noise) blocks += S;                 // its ITER blocks
        if (STOP) {
          steps += S;
          blocks += spec ? (S + 3u) >> 2 : 0u;
        }
      }
      tprev = t;
      tlast = carry;
    }
    if constexpr (STOP) {                              // never simulated past t*: sentinels for the rest
      if (stopped) {
        for (uint32_t j = (jstar & ~31u) + 32u + (uint32_t)lane; j < N; j += 32) p.lat[rowoff + j] = 0xFFFFFFFFu;
      }
    }
    const uint32_t slo_met = __reduce_add_sync(FULL, my_slo & 0x7FFFFFFFu);
    const uint64_t sum = warp_sum64(my_sum);
    const bool sat = __any_sync(FULL, (my_slo >> 31) != 0);
    const uint32_t n_meas = __reduce_add_sync(FULL, nmeas);
    ct.batches += (uint32_t)batches;
    ct.dsteps += (uint32_t)dsteps;
    ct.steps += (uint32_t)steps;
    ct.blocks += (uint32_t)blocks;
    if (lane == 0) {
      // the window ends at the last measured completion (t*, or t_{N-1}: completions are in index order)
      const uint64_t Tw = (STOP && stopped ? tstar : tlast) - a_w;
      const uint32_t fl = (sat ? 2u : 0u) | (STOP && !stopped ? 4u : 0u);
      p.part[r] = slo_replica_result{0, slo_met, STOP ? n_meas : p.seg, fl, Tw < 1 ? 1 : Tw, sum};
      if (p.stats) {
        unsigned long long* st = (unsigned long long*)p.stats;
        atomicAdd(st + 0, (unsigned long long)N);
        atomicAdd(st + 4, (unsigned long long)(N + R.nphase));
        atomicAdd(st + 5, 1ull);
      }
    }
    if (ct.steps >= 0x40000000u || ct.dsteps >= 0x40000000u || ct.batches >= 0x40000000u) flush_counters(p, ct);
  }
}

// ------------------------------------------------------------------------------------------------
// K1c: continuous (iteration-level, vLLM-style) batching, DESIGN.md §2.12.
//
// A warp runs 32/G replicas at once, one per G-lane group with G >= min(C, B) (lane = one slot of the
// running set R, |R| <= min(C, B)).  The server's free instants are iteration ends and, when it idles, the next issue.  The
// gate's closed form s_j = max(a_j, kappa_{j-C}) holds for any service order (issue is in index order and
// completions only free slots), so a group keeps s_next = s_{nq} (the next request to admit) and:
//   * prefill iteration iff |R| < B and s_next <= t: a ballot over the window j = nq + li counts the queue,
//     the first k = min(B - |R|, queue) requests take the free slots;
//   * else decode iteration iff |R| > 0: every running lane takes its next acceptance draw, completions at
//     the iteration end fill kappa;
//   * else idle until s_next.
// A request's decode-iteration count S_i depends on its own SPEC stream only (its j counts its own
// iterations), so generation resolves it and a slot just counts down; between events the decode iterations
// are fast-forwarded (K = first completion, first prefill opportunity, or the noise window).  Noise words
// come from a window of the next G decode iterations per group (ITER blocks; when any group has used half
// of its window every group shifts its window and draws the consumed part in the same pass).
// ------------------------------------------------------------------------------------------------
template <int G>
struct alignas(16) CGroup {
  static constexpr int RING = 4 * G;   // a, po, w3 for [nq, gen), gen < nq + 2G
  static constexpr int KRING = 64;     // kappa_k for k in [nq - C, ndone): span <= C + B <= 64
  uint64_t a[RING];
  uint64_t kap[KRING];
  uint32_t po[RING];
  uint32_t w3[RING];
  uint16_t ss[RING];                   // S_j: decode iterations request j needs (§2.12: its own draws only)
  uint32_t tm1[16];
  uint8_t guide[256];
  uint64_t g[2], rho[2];
  uint64_t last;
  uint64_t pstart, pD, pU, pLam, nphase, a_w, alpha0, alpha1;
  uint32_t ph, pstate, pre_base, pre_tok, noise, kind, start_state, gp;
  uint32_t k0, k1, wl, pad;
  uint32_t cnt_meas, stopped, pad3[2];          // stop rule (§2.14): measured completions so far, stopped
};

// THINK (kind 4, §2.11): the C pending user chains sit sorted in the lanes (lane l = request nq + l) and give
// s_next and the prefill window in place of s_j = max(a_j, kappa_{j-C})
// SPLIT: the requests' attributes come from K1g's records (register-staged one refill ahead) instead of inline
// generation (Philox REQ / SPEC blocks, lengths, S_i)
template <int G, bool STOP, bool THINK, bool SPLIT = false>
__device__ __forceinline__ void run_cont(const SimParams& p, int cls, uint8_t* wsmem, int lane, Counters& ct) {
  using CG = CGroup<G>;
  constexpr int RING = CG::RING, KRING = CG::KRING;
  const int g = lane / G, li = lane % G;
  CG& R = reinterpret_cast<CG*>(wsmem)[g];
  const uint32_t gmask = (G == 32) ? FULL : (((1u << G) - 1u) << (g * G));
  const uint32_t ltg = (1u << li) - 1u;                 // group-relative lanes below this one
  const uint32_t N = p.warmup + p.seg;
  const uint32_t count = p.counts[cls];
  const uint32_t* list = p.lists + (size_t)cls * p.n_chunk;

  // group-uniform state (every lane of a group holds the same value)
  uint32_t r = 0, rowoff = 0, nq = 0, ndone = 0, gen = 0, it = 0, nrun = 0, npre = 0;
  uint32_t C = 0, B = 0, gamma = 0, noise = 0, k0 = 0, k1 = 0, alpha0 = 0, alpha1 = 0;
  uint64_t t = 0, s_next = INF64, a_w = 0;
  bool active = false, exhausted = count == 0, need_s = false, closed = false;
  // slot state (lane = one slot of the running set)
  bool run = false;
  // sleft: decode iterations the slot's request still runs; stot: its S (counters); fw: noise window
  uint32_t mi = 0, sleft = 0, stot = 0, fw = 0, fw2 = 0, nzc = 0, my_slo = 0;
  uint64_t origin = 0, my_sum = 0, my_cmax = 0;
  uint64_t pq = INF64;          // THINK: this lane's pending ready instant
  uint32_t pid = 0xFFFFFFFFu;   // THINK: its user chain id
  uint4 stg{0, 0, 0, 0};        // SPLIT: K1g record of request gen + li, loaded one refill ahead
  // requests [gen, gen + G) into the rings for the groups with `go` (all lanes execute)
  auto refill = [&](bool go) {
    if constexpr (SPLIT) {
      const uint32_t i = gen + (uint32_t)li;
      const bool valid = go && i < N;
      const uint64_t x = valid ? (((uint64_t)stg.y << 32) | stg.x) : 0ull;
      const uint64_t a = arrivals<G>(R, p.wl, R.wl, k0, k1, x, i, N, go, lane, li);
      if (valid) {
        R.a[i % RING] = a;
        R.po[i % RING] = stg.z & 0xFFFFu;
        R.w3[i % RING] = stg.w;
        R.ss[i % RING] = (uint16_t)(stg.z >> 16);
        if (i == p.warmup) R.a_w = a;
      }
      __syncwarp();
      if (go) {
        gen += G;
        if (gen + (uint32_t)li < N) stg = __ldcs(p.rec + rowoff + gen + li);
      }
    } else {
      generate<G>(R, p.wl, R.wl, p.tables, k0, k1, gen, N, p.warmup, go, lane, li);
      if (go) gen += G;
    }
  };
  constexpr uint32_t LOOK = SPLIT ? 2 * G : G;   // the split path refills one window ahead (record latency)

  bool acq = true;
  for (;;) {
    __syncwarp();
    // ---- acquire replicas for idle groups
    if (acq) {   // acquisition and the exit test only after a replica finished (warp-uniform)
      bool want = !active && !exhausted;
      while (__any_sync(FULL, want)) {
        uint32_t idx = 0;
        if (want && li == 0) idx = atomicAdd(p.cursor + cls, 1u);
        idx = gshfl<G>(idx, 0);
        if (want) {
          if (idx >= count) {
            exhausted = true;
          } else {
            r = list[idx];
            const uint32_t ci = r / p.n_seeds;
            const slo_knobs k = p.cfg[ci];
            if (!knobs_valid(k, p.n_wl)) {   // (K0 puts invalid records in list 0; kept for safety)
              if (li == 0) {
                p.part[r] = slo_replica_result{0xFFFFFFFFu, 0, 0, 1u, 0, 0};
                if (p.stats) atomicAdd((unsigned long long*)&p.stats->replicas, 1ull);
              }
            } else {
              const DevWorkload& W = p.wl[k.workload];
              const uint64_t seed = p.seeds[r - ci * p.n_seeds];
              const uint32_t cfgkey = p.crn ? W.stream_id : fnv1a_knobs(k);
              k0 = (uint32_t)seed;
              k1 = (uint32_t)(seed >> 32) ^ cfgkey;
              gamma = k.spec_on ? k.draft_len : 0u;
              uint32_t gp;
              if (li == 0) R.wl = k.workload;
              setup_replica<G, !SPLIT>(R, W, k, k0, k1, gamma, gp, li, gmask);
              C = k.conc;
              B = k.max_num_seqs;
              closed = W.kind >= 3;
              if constexpr (THINK) {                       // the first C chains are ready at t = 0
                pq = ((uint32_t)li < C && (uint32_t)li < N) ? 0ull : INF64;
                pid = (uint32_t)li;
              }
              noise = W.t.noise_step_ppm;
              alpha0 = (uint32_t)R.alpha0;                 // d(n) = alpha0 + alpha1 n
              alpha1 = (uint32_t)R.alpha1;
              rowoff = (r - p.r_base) * N;
              if constexpr (SPLIT) stg = (uint32_t)li < N ? __ldcs(p.rec + rowoff + li) : uint4{0, 0, 0, 0};
              t = 0;
              s_next = INF64;
              a_w = 0;
              nq = ndone = gen = it = nrun = npre = 0;
              nzc = 2 * G;                                 // noise window empty: filled at the first decode
              run = false;
              my_slo = 0;
              my_sum = 0;
              my_cmax = 0;
              need_s = true;
              active = true;
            }
          }
        }
        want = !active && !exhausted;
      }
      if (!__any_sync(FULL, active)) break;
      acq = false;
    }
    __syncwarp();   // setup / previous iteration's ring writes before this iteration's reads
    if (lane == 0) KPROF(0, 1u);
    if (li == 0) KPROF(1, active ? 1u : 0u);
    if (li == 0) KPROF(2, need_s ? 1u : 0u);

    // ---- s_next = s_{nq} for groups whose nq or gate changed; keep [nq, nq + G) generated
    if (__any_sync(FULL, need_s)) {
      bool gn = need_s && gen < N && gen < nq + G;
      while (__any_sync(FULL, gn)) {
        refill(need_s && gen < N && gen < nq + LOOK);
        gn = need_s && gen < N && gen < nq + G;
      }
      const uint64_t pq0 = gshfl64<G>(pq, 0);
      if (need_s) {
        s_next = INF64;
        if (THINK) {
          s_next = pq0;
        } else if (nq < min(N, ndone + C)) {
          const uint64_t aj = R.a[nq % RING];
          const uint64_t kj = nq >= C ? R.kap[(nq - C) % KRING] : 0;
          s_next = aj > kj ? aj : kj;
        }
        need_s = false;
      }
    }
    if (active && nrun == 0 && s_next > t) t = s_next;   // idle until the next issue
    const bool pre = active && nrun < B && s_next <= t;

    // ---- prefill iteration: admit the first k queued requests into free slots (§2.12)
    if (__any_sync(FULL, pre)) {
      if (lane == 0) KPROF(10, 1u);
      if (li == 0) KPROF(3, pre ? 1u : 0u);
      bool gn = pre && gen < N && gen < nq + G;          // the window [nq, nq + G) must be generated
      while (__any_sync(FULL, gn)) {
        refill(pre && gen < N && gen < nq + LOOK);
        gn = pre && gen < N && gen < nq + G;
      }
      __syncwarp();
      const uint32_t j = nq + (uint32_t)li;
      uint64_t sj = INF64;
      if (THINK) {
        if (pre) sj = pq;
      } else if (pre && j < min(N, ndone + C)) {
        const uint64_t aj = R.a[j % RING];
        const uint64_t kj = j >= C ? R.kap[(j - C) % KRING] : 0;
        sj = aj > kj ? aj : kj;
      }
      const uint32_t avail = __popc(gballot<G>(sj <= t, lane));
      const uint32_t runm = gballot<G>(run, lane);
      const uint32_t kk = pre ? min(B - nrun, avail) : 0u;
      const uint32_t rank = __popc(~runm & ltg);
      const bool adm = pre && !run && rank < kk;
      const uint64_t s_r = gshfl64<G>(sj, (int)(rank & (G - 1)));
      uint32_t P = 0;
      if (adm) {
        const uint32_t i = nq + rank;
        const uint32_t po = R.po[i % RING];
        P = po & 0xFFFFu;
        mi = i;
        stot = R.ss[i % RING];                          // S_i, resolved at generation (§2.12: own draws only)
        sleft = stot;
        origin = closed ? s_r : R.a[i % RING];
        run = true;
      }
      const bool wsrc = pre && closed && p.warmup >= nq && p.warmup < nq + kk;
      if (__any_sync(FULL, wsrc)) {                      // closed loop: the window starts at s_warmup
        const uint64_t sw = gshfl64<G>(sj, (int)((p.warmup - nq) & (G - 1)));
        if (wsrc) a_w = sw;
      }
      const uint32_t maxP = gmax<G>(P);
      // s_next = s_{nq + k} straight from the window (INF if beyond the gate); k = G: recompute at the top
      const uint64_t sn = gshfl64<G>(sj, (int)(kk & (G - 1)));
      if (pre) {
        const uint64_t f = noise_factor(R.w3[nq % RING], noise);
        t += f * ((uint64_t)R.pre_base + (uint64_t)R.pre_tok * maxP) / 1000000u;
        nq += kk;
        nrun += kk;
        ++npre;
        s_next = sn;
        if (kk == (uint32_t)G) need_s = true;
      }
      if constexpr (THINK) {                             // the admitted chains leave the pending list
        const int src = li + (int)kk;
        const uint64_t sp = gshfl64<G>(pq, src & (G - 1));
        const uint32_t sq = gshfl<G>(pid, src & (G - 1));
        if (pre) {
          pq = src < G ? sp : INF64;
          pid = src < G ? sq : 0xFFFFFFFFu;
        }
      }
    }
    // a group that just prefilled decodes in the same pass unless another prefill is due at once
    const bool dec = active && !need_s && nrun > 0 && !(nrun < B && s_next <= t);

    // ---- decode iterations over the running set, fast-forwarded to the next event.  While no member
    // finishes and no prefill can start, consecutive decode iterations change nothing but t, the members'
    // token counts and the random-word cursors, so a group advances K of them at once: lane k holds the
    // durations of iterations it + 2k and it + 2k + 1 (D = floor(f d(n) / 10^6), d(n) = alpha0 + alpha1 n),
    // a group scan gives their end times (up to 2G iterations per pass), and
    //   K = min(first iteration at whose end a member finishes,
    //           first iteration at whose end a prefill can start (|R| < B and s_next <= end),
    //           the iterations whose random words are buffered).
    if (__any_sync(FULL, dec)) {
      const bool nz = dec && noise != 0;
      // noise window of 2G decode iterations: lane li holds positions li (fw) and G + li (fw2) after nzc used
      if (__any_sync(FULL, nz && nzc > (uint32_t)(SLO_CONT_REFILL * G / 4))) {   // pooled shift-refill once
                                                       // SLO_CONT_REFILL / 8 of it is used
        if (lane == 0) KPROF(8, 1u);
        const uint32_t sA = (uint32_t)li + nzc, sB = (uint32_t)(G + li) + nzc;   // old positions of the new ones
        const uint32_t a0 = __shfl_sync(FULL, fw, (int)(sA & (G - 1)), G);
        const uint32_t b0 = __shfl_sync(FULL, fw2, (int)(sA & (G - 1)), G);
        const uint32_t b1 = __shfl_sync(FULL, fw2, (int)(sB & (G - 1)), G);
        if (nz && nzc > 0) {
#if SLO_CONT_PAIRDRAW
          // both ITER blocks drawn together (two independent Philox chains interleave); kept only where new
          const uint32_t na = noise_factor(philox(it + (uint32_t)li, 3, 0, 0, k0, k1).x, noise);
          const uint32_t nb = noise_factor(philox(it + (uint32_t)(G + li), 3, 0, 0, k0, k1).x, noise);
          fw = sA < (uint32_t)(2 * G) ? (sA < (uint32_t)G ? a0 : b0) : na;
          fw2 = sB < (uint32_t)(2 * G) ? b1 : nb;
#else
          if (sA < (uint32_t)(2 * G)) {
            fw = sA < (uint32_t)G ? a0 : b0;
          } else {                                       // ITER block it + li, word 0 (§2.12)
            fw = noise_factor(philox(it + (uint32_t)li, 3, 0, 0, k0, k1).x, noise);
          }
          if (sB < (uint32_t)(2 * G)) {
            fw2 = b1;
          } else {                                       // ITER block it + G + li
            fw2 = noise_factor(philox(it + (uint32_t)(G + li), 3, 0, 0, k0, k1).x, noise);
          }
#endif
          nzc = 0;
        }
      }
      // end times of the next 2G iterations: lane k <-> iterations it + 2k and it + 2k + 1
      const uint32_t d = alpha0 + alpha1 * nrun;          // < 2^31 (timing values < 2^20, gamma <= 16)
      const uint32_t p0 = nzc + 2u * (uint32_t)li, p1 = p0 + 1u;
      const uint32_t x0 = __shfl_sync(FULL, fw, (int)(p0 & (G - 1)), G), y0 = __shfl_sync(FULL, fw2, (int)(p0 & (G - 1)), G);
      const uint32_t x1 = __shfl_sync(FULL, fw, (int)(p1 & (G - 1)), G), y1 = __shfl_sync(FULL, fw2, (int)(p1 & (G - 1)), G);
      const uint32_t f0 = p0 < (uint32_t)G ? x0 : y0, f1 = p1 < (uint32_t)G ? x1 : y1;
      const uint32_t D0 = nz ? (uint32_t)(((uint64_t)f0 * d) / 1000000u) : d;
      const uint32_t D1 = nz ? (uint32_t)(((uint64_t)f1 * d) / 1000000u) : d;
      const uint64_t end1 = gscan64<G>((uint64_t)D0 + D1, li);   // end of iteration 2k + 1
      const uint64_t end0 = end1 - D1;                            // end of iteration 2k
      // K = min(first completion, first iteration end at which a prefill can start, the noise window)
      uint32_t K = gmin<G>(dec && run ? sleft : 0xFFFFu);
      K = min(K, nz ? (uint32_t)(2 * G) - nzc : (uint32_t)(2 * G));
      const bool canpre = dec && nrun < B;                          // s_next = INF: never
      const uint32_t m0 = gballot<G>(canpre && 2u * (uint32_t)li < K && t + end0 >= s_next, lane);
      const uint32_t m1 = gballot<G>(canpre && 2u * (uint32_t)li + 1u < K && t + end1 >= s_next, lane);
      const uint32_t i0 = m0 ? 2u * (uint32_t)(__ffs(m0) - 1) : 0xFFFFu, i1 = m1 ? 2u * (uint32_t)(__ffs(m1) - 1) + 1u : 0xFFFFu;
      if (m0 | m1) K = min(i0, i1) + 1u;                  // the first such iteration end
      const uint64_t tK = gshfl64<G>(((K - 1u) & 1u) ? end1 : end0, (int)(((K - 1u) >> 1) & (G - 1)));
      if (lane == 0) KPROF(11, 1u);
      if (li == 0 && dec) {
        KPROF(4, 1u);
        KPROF(5, K);
        KPROF(7, (m0 | m1) ? 1u : 0u);
        KPROF(14, K == 2u * G ? 1u : 0u);
        KPROF(13, nrun);
      }
      bool fin = false;
      if (dec) {
        t += tK;
        it += K;
        if (nz) nzc += K;
        if (run) {
          sleft -= K;
          fin = sleft == 0;
        }
      }
#ifdef SLO_K1C_PROF
      const uint32_t pf_fin = gballot<G>(fin, lane);
      if (li == 0) KPROF(6, (dec && pf_fin) ? 1u : 0u);
#endif
      if (__any_sync(FULL, fin)) {
        const uint32_t nf = __popc(gballot<G>(fin, lane));
        if (lane == 0) KPROF(12, 1u);
        if (li == 0) KPROF(9, nf);
        if (fin) {                                       // (a8) completion at t
          const uint64_t l = t - origin;
          p.lat[rowoff + mi] = l > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)l;
          if (mi >= p.warmup) {
            my_slo += (l <= p.slo_us);
            my_slo |= (l > 0xFFFFFFFFull) ? 0x80000000u : 0u;
            my_sum += l;
            my_cmax = t;
          }
          if (!SPLIT || STOP) {                          // (split, no stop rule: K1g counted them)
            ct.steps += stot;
            ct.blocks += gamma > 0 ? (stot + 3u) >> 2 : 0u;
          }
          run = false;
        }
        if constexpr (THINK) {
          // completion ndone + (rank of mi among this iteration's finishers) starts chain + C, ready Z later
          uint32_t rk = 0;
#pragma unroll 4
          for (int o = 0; o < G; ++o) {
            const uint32_t mo = gshfl<G>(mi, o), fo = gshfl<G>(fin ? 1u : 0u, o);
            rk += (fo && mo < mi) ? 1u : 0u;
          }
          const uint32_t kord = ndone + rk;
          const bool spawn = fin && kord + C < N;
          const uint64_t z = spawn ? mulshr(exp_q32(philox(kord, 4, 0, 0, k0, k1).x), R.g[0], 48) : 0ull;
          const uint64_t st_ = spawn ? t + z : INF64;
          const uint32_t sid = spawn ? kord + C : 0xFFFFFFFFu;
          const uint32_t sm = gballot<G>(spawn, lane);
          const int np = __popc(gballot<G>(pq != INF64, lane));   // real pending entries (sorted first)
          const int idx = li - np;
          const bool take = idx >= 0 && idx < __popc(sm);
          const int src = take ? (int)__fns(sm, 0, idx + 1) : 0;
          const uint64_t v = gshfl64<G>(st_, src);
          const uint32_t vq = gshfl<G>(sid, src);
          if (take) {
            pq = v;
            pid = vq;
          }
          gsort_pair<G>(pq, pid, li);
          ct.blocks += spawn ? 1u : 0u;
        }
        if (dec && (uint32_t)li < nf) R.kap[(ndone + li) % KRING] = t;
        const uint64_t pq0 = THINK ? gshfl64<G>(pq, 0) : 0ull;   // (all lanes: the shuffle needs the warp)
        if (dec) {
          ndone += nf;
          nrun -= nf;
          if (THINK) {
            s_next = pq0;                                // the earliest pending chain after the spawns
          } else if (s_next == INF64 && nq < N) {
            need_s = true;                               // completions may have opened the gate for nq
          }
        }
        if constexpr (STOP) {                            // stop rule (§2.14): completions at t continue the count
          const uint32_t nfm = __popc(gballot<G>(fin && mi >= p.warmup, lane));
          const uint32_t before = dec ? R.cnt_meas : 0u;
          const uint64_t t0 = closed ? a_w : R.a_w;
          const uint32_t need = p.stop_n ? p.stop_n : 1u;
          const bool stop_now = dec && !R.stopped && nfm > 0 && before + nfm >= need && t >= t0 + p.stop_t;
          __syncwarp();
          if (dec && li == 0) {
            R.cnt_meas = before + nfm;
            if (stop_now) R.stopped = 1;
          }
          if (stop_now) {                                // t* = t: whatever has not completed never counts
            if (run) p.lat[rowoff + mi] = 0xFFFFFFFFu;
            for (uint32_t j = nq + (uint32_t)li; j < N; j += G) p.lat[rowoff + j] = 0xFFFFFFFFu;
            run = false;
            ndone = N;
          }
        }
      }
    }

    // ---- groups that finished their replica: outputs (p99 and goodput follow in K1b)
    const bool done = active && ndone >= N;
#ifdef SLO_K1C_PROF
    const uint32_t pf_act = __popc(__ballot_sync(FULL, active && li == 0));
    if (lane == 0) KPROF(15, pf_act);
#endif
    if (__any_sync(FULL, done)) {
      const uint32_t slo_met = gsum<G>(my_slo & 0x7FFFFFFFu);
      const uint64_t sum = gsum64<G>(my_sum);
      const uint64_t cm = gmax64<G>(my_cmax);
      const bool sat = gballot<G>((my_slo >> 31) != 0, lane) != 0;
      if (done && li == 0) {
        const uint64_t Tw = cm - (closed ? a_w : R.a_w);
        const uint32_t fl = (sat ? 2u : 0u) | (STOP && !R.stopped ? 4u : 0u);
        p.part[r] = slo_replica_result{0, slo_met, STOP ? R.cnt_meas : p.seg, fl, Tw < 1 ? 1 : Tw, sum};
        ct.batches += npre;
        ct.dsteps += it;
        ct.blocks += noise ? it : 0u;
        if (p.stats) {
          unsigned long long* st = (unsigned long long*)p.stats;
          atomicAdd(st + 0, (unsigned long long)N);
          atomicAdd(st + 4, (unsigned long long)(N + R.nphase));
          atomicAdd(st + 5, 1ull);
        }
      }
      if (done) active = false;
      acq = true;                                       // (the only way a group goes idle)
      if (ct.steps >= 0x40000000u || ct.dsteps >= 0x40000000u || ct.blocks >= 0x40000000u) flush_counters(p, ct);
    }
  }
}

#ifndef SLO_MAXNREG
#define SLO_MAXNREG 80
#endif
template <bool STOP>
__global__ void __maxnreg__(SLO_MAXNREG) slo_sim_kernel_t(const SimParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  uint8_t* wsmem = smem + (size_t)(threadIdx.x >> 5) * p.warp_bytes;
  Counters ct{0, 0, 0, 0};
  run_mode<8, STOP, false>(p, 0, wsmem, lane, ct);
  run_mode<16, STOP, false>(p, 1, wsmem, lane, ct);
  run_mode<32, STOP, false>(p, 2, wsmem, lane, ct);
  if (p.stats) {
    const uint64_t steps = warp_sum64(ct.steps), blocks = warp_sum64(ct.blocks);
    const uint64_t batches = warp_sum64(ct.batches), dsteps = warp_sum64(ct.dsteps);
    if (lane == 0) {
      unsigned long long* st = (unsigned long long*)p.stats;
      atomicAdd(st + 1, (unsigned long long)batches);
      atomicAdd(st + 2, (unsigned long long)dsteps);
      atomicAdd(st + 3, (unsigned long long)steps);
      atomicAdd(st + 4, (unsigned long long)blocks);
    }
  }
}

// K1s: the static-batching chain over K1g's request records (split path); leaner than K1, so a lower register cap
#ifndef SLO_SERVE_MAXNREG
#define SLO_SERVE_MAXNREG 80
#endif
template <bool STOP>
__global__ void __maxnreg__(SLO_SERVE_MAXNREG) slo_serve_kernel_t(const SimParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  uint8_t* wsmem = smem + (size_t)(threadIdx.x >> 5) * p.warp_bytes;
  Counters ct{0, 0, 0, 0};
  scan_mode<STOP>(p, kScanList, wsmem, lane, ct);   // min(C, B) = 1: a max-plus scan, 32 requests per step
  serve_mode<4, STOP>(p, kG4List, wsmem, lane, ct);   // min(C, B) <= 4: eight replicas per warp
  serve_mode<8, STOP>(p, 0, wsmem, lane, ct);
  serve_mode<16, STOP>(p, 1, wsmem, lane, ct);
  serve_mode<32, STOP>(p, 2, wsmem, lane, ct);
  if (p.stats) {
    const uint64_t steps = warp_sum64(ct.steps), blocks = warp_sum64(ct.blocks);
    const uint64_t batches = warp_sum64(ct.batches), dsteps = warp_sum64(ct.dsteps);
    if (lane == 0) {
      unsigned long long* st = (unsigned long long*)p.stats;
      atomicAdd(st + 1, (unsigned long long)batches);
      atomicAdd(st + 2, (unsigned long long)dsteps);
      atomicAdd(st + 3, (unsigned long long)steps);
      atomicAdd(st + 4, (unsigned long long)blocks);
    }
  }
}

// K1t: closed loops with think time (kind 4), launched only when a workload uses it
template <bool STOP>
__global__ void __maxnreg__(SLO_MAXNREG) slo_sim_think_kernel_t(const SimParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  uint8_t* wsmem = smem + (size_t)(threadIdx.x >> 5) * p.warp_bytes;
  Counters ct{0, 0, 0, 0};
  run_mode<8, STOP, true>(p, 6, wsmem, lane, ct);
  run_mode<16, STOP, true>(p, 7, wsmem, lane, ct);
  run_mode<32, STOP, true>(p, 8, wsmem, lane, ct);
  if (p.stats) {
    const uint64_t steps = warp_sum64(ct.steps), blocks = warp_sum64(ct.blocks);
    const uint64_t batches = warp_sum64(ct.batches), dsteps = warp_sum64(ct.dsteps);
    if (lane == 0) {
      unsigned long long* st = (unsigned long long*)p.stats;
      atomicAdd(st + 1, (unsigned long long)batches);
      atomicAdd(st + 2, (unsigned long long)dsteps);
      atomicAdd(st + 3, (unsigned long long)steps);
      atomicAdd(st + 4, (unsigned long long)blocks);
    }
  }
}

// K1c: the continuous-batching work list, launched only when a workload uses it
#ifndef SLO_CONT_MAXNREG
#define SLO_CONT_MAXNREG 88   // (no spills; 96 measured +0.6 %, 80 / 104 +3 % on C2-cont; still 5 blocks of 4 warps)
#endif
template <bool STOP, bool THINK, bool SPLIT>
__global__ void __maxnreg__(SLO_CONT_MAXNREG) slo_sim_cont_kernel_t(const SimParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  uint8_t* wsmem = smem + (size_t)(threadIdx.x >> 5) * p.warp_bytes;
  Counters ct{0, 0, 0, 0};
  constexpr int l0 = THINK ? 9 : 3;   // THINK: the closed loops with think time (kind 4), lists 9-11
  // split path: the min(C, B) = 1 replicas' max-plus scans first (K1e, one replica per warp; their chains are
  // the longest), then the fast-forward lists
  if constexpr (SPLIT && !THINK) {
    scan_mode<STOP, true>(p, kCScanList, wsmem, lane, ct);
    run_cont<4, STOP, THINK, SPLIT>(p, kCG4List, wsmem, lane, ct);
  }
  run_cont<8, STOP, THINK, SPLIT>(p, l0, wsmem, lane, ct);
  run_cont<16, STOP, THINK, SPLIT>(p, l0 + 1, wsmem, lane, ct);
  run_cont<32, STOP, THINK, SPLIT>(p, l0 + 2, wsmem, lane, ct);
  if (p.stats) {
    const uint64_t steps = warp_sum64(ct.steps), blocks = warp_sum64(ct.blocks);
    const uint64_t batches = warp_sum64(ct.batches), dsteps = warp_sum64(ct.dsteps);
    if (lane == 0) {
      unsigned long long* st = (unsigned long long*)p.stats;
      atomicAdd(st + 1, (unsigned long long)batches);
      atomicAdd(st + 2, (unsigned long long)dsteps);
      atomicAdd(st + 3, (unsigned long long)steps);
      atomicAdd(st + 4, (unsigned long long)blocks);
    }
  }
}

// K1 / K1c and their stop-rule variants: separate instantiations, so the default path
// carries none of the stop rule's code
template __global__ void slo_sim_kernel_t<false>(const SimParams p);
template __global__ void slo_sim_kernel_t<true>(const SimParams p);
template __global__ void slo_serve_kernel_t<false>(const SimParams p);
template __global__ void slo_serve_kernel_t<true>(const SimParams p);
template __global__ void slo_sim_think_kernel_t<false>(const SimParams p);
template __global__ void slo_sim_think_kernel_t<true>(const SimParams p);
template __global__ void slo_sim_cont_kernel_t<false, false, false>(const SimParams p);
template __global__ void slo_sim_cont_kernel_t<true, false, false>(const SimParams p);
template __global__ void slo_sim_cont_kernel_t<false, true, false>(const SimParams p);
template __global__ void slo_sim_cont_kernel_t<true, true, false>(const SimParams p);
template __global__ void slo_sim_cont_kernel_t<false, false, true>(const SimParams p);
template __global__ void slo_sim_cont_kernel_t<true, false, true>(const SimParams p);

size_t cont_warp_bytes() {
  size_t m = sizeof(SGroup<32>);              // (the split path's continuous scan, K1e)
  if (8 * sizeof(CGroup<4>) > m) m = 8 * sizeof(CGroup<4>);
  if (4 * sizeof(CGroup<8>) > m) m = 4 * sizeof(CGroup<8>);
  if (2 * sizeof(CGroup<16>) > m) m = 2 * sizeof(CGroup<16>);
  if (sizeof(CGroup<32>) > m) m = sizeof(CGroup<32>);
  return m;
}

size_t serve_warp_bytes() {
  size_t m = 8 * sizeof(SGroup<4>);
  if (4 * sizeof(SGroup<8>) > m) m = 4 * sizeof(SGroup<8>);
  if (2 * sizeof(SGroup<16>) > m) m = 2 * sizeof(SGroup<16>);
  if (sizeof(SGroup<32>) > m) m = sizeof(SGroup<32>);
  return m;
}

size_t group_warp_bytes() {
  size_t m = 4 * sizeof(Group<8>);
  if (2 * sizeof(Group<16>) > m) m = 2 * sizeof(Group<16>);
  if (sizeof(Group<32>) > m) m = sizeof(Group<32>);
  return m;
}

// ------------------------------------------------------------------------------------------------
// K0: work lists by lane-group size, longest expected replicas first (a 16-bucket counting sort)
// ------------------------------------------------------------------------------------------------
// Expected cost ~ (batches per segment) x (cost per batch); a saturated replica runs ~N / min(C, B) batches
// and a speculative batch costs ~3x a plain one.  bucket = floor(log2(beff^2)) (+3 ~ 2 log2 3 if not
// speculative), so bucket 0 = most expensive; invalid records (no work) go last.
#ifndef SLO_SCAN
#define SLO_SCAN 1
#endif
#ifndef SLO_G4
#define SLO_G4 1
#endif
#ifndef SLO_CG4
#define SLO_CG4 1
#endif
__device__ __forceinline__ uint32_t work_class(const slo_knobs& k, const DevWorkload* __restrict__ wl, uint32_t n_wl,
                                               uint32_t wide, uint32_t& bucket) {
  const bool split = (wide & 4u) != 0;              // the split path (K1g + K1s) serves static batching
  wide &= 3u;
  if (!knobs_valid(k, n_wl)) {
    bucket = 15;
    return 0;
  }
  // split path, min(C, B) = 1: every batch is one request, the chain a max-plus recursion (K1s scan_mode)
  if (SLO_SCAN && split && !wl[k.workload].batching && wl[k.workload].kind != 4 && (k.conc == 1 || k.max_num_seqs == 1)) {
    bucket = 0;
    return (uint32_t)kScanList;
  }
  // static batching needs G >= min(C, B) lanes: a batch has b <= min(C, B) members, the issue window
  // only matters for them, and s_{h+B-1} is needed only when B <= C.  Narrow groups pack more replicas
  // per warp (throughput); a launch too small to fill the GPU (`wide`) takes G >= max(C, B) instead, which
  // shortens each replica's dependency chain (latency)
  const uint32_t beff = min((uint32_t)k.conc, (uint32_t)k.max_num_seqs);
  // (wide == 2: a launch of at most one replica per SM — a lone replica's chain is shortest with the whole
  // warp, G = 32: a generation pass yields 32 requests)
  const uint32_t need = wide == 2 ? 32u : wide ? max((uint32_t)k.conc, (uint32_t)k.max_num_seqs) : beff;
  const bool spec = k.spec_on && k.draft_len > 0;
  bucket = min(14u, (31u - __clz(beff * beff)) + (spec ? 0u : 3u));
  if (wl[k.workload].kind == 4) {     // think time: the C pending chains live in the lanes, G >= max(C, B)
    const uint32_t tneed = wide == 2 ? 32u : max((uint32_t)k.conc, (uint32_t)k.max_num_seqs);
    const uint32_t base = wl[k.workload].batching ? 9u : 6u;
    return base + (tneed <= 8 ? 0u : (tneed <= 16 ? 1u : 2u));
  }
  if (split && wl[k.workload].batching && beff == 1) {   // split path, min(C, B) = 1: K1e's scan
    bucket = 0;
    return (uint32_t)kCScanList;
  }
  if (SLO_CG4 && split && wl[k.workload].batching && !wide && beff <= 4) {   // K1c, eight replicas per warp
    bucket = min(14u, (31u - __clz(beff)) + (spec ? 0u : 2u));
    return (uint32_t)kCG4List;
  }
  if (wl[k.workload].batching) {      // continuous batching, ~N*O/beff iterations: lane groups G >= min(C, B)
    // (at most min(C, B) requests run at once and a prefill admits at most that many; `wide`: G >= B)
    bucket = min(14u, (31u - __clz(beff)) + (spec ? 0u : 2u));
    const uint32_t cneed = wide ? (uint32_t)k.max_num_seqs : beff;
    return cneed <= 8 ? 3u : (cneed <= 16 ? 4u : 5u);
  }
  if (SLO_G4 && split && need <= 4) return (uint32_t)kG4List;   // K1s: eight replicas per warp
  return need <= 8 ? 0u : (need <= 16 ? 1u : 2u);
}

__global__ void slo_classify_count_kernel(const slo_knobs* __restrict__ cfg, const DevWorkload* __restrict__ wl,
                                          uint32_t n_seeds, uint32_t r_base, uint32_t n_chunk, uint32_t n_wl,
                                          uint32_t wide, uint32_t* __restrict__ ctl, const uint32_t* __restrict__ live) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_chunk) return;
  if (live && (r_base + t) / n_seeds >= *live) return;     // a skipped config: no work list, no outputs
  uint32_t bucket;
  const uint32_t cls = work_class(cfg[(r_base + t) / n_seeds], wl, n_wl, wide, bucket);
  atomicAdd(ctl + kCtlBucket + cls * 16 + bucket, 1u);     // per (class, bucket) counts
}

__global__ void slo_classify_kernel(const slo_knobs* __restrict__ cfg, const DevWorkload* __restrict__ wl,
                                    uint32_t n_seeds, uint32_t r_base, uint32_t n_chunk, uint32_t n_wl,
                                    uint32_t wide, uint32_t* __restrict__ ctl, uint32_t* __restrict__ lists,
                                    const uint32_t* __restrict__ live) {
  __shared__ uint32_t off[16 * kLists];
  if (threadIdx.x < kLists) {                      // exclusive offsets of the buckets inside each list
    uint32_t acc = 0;
    for (int bkt = 0; bkt < 16; ++bkt) {
      off[threadIdx.x * 16 + bkt] = acc;
      acc += ctl[kCtlBucket + threadIdx.x * 16 + bkt];
    }
    if (blockIdx.x == 0) ctl[threadIdx.x] = acc;   // list lengths (read by K1)
  }
  __syncthreads();
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_chunk) return;
  const uint32_t r = r_base + t;
  if (live && r / n_seeds >= *live) return;
  uint32_t bucket;
  const uint32_t cls = work_class(cfg[r / n_seeds], wl, n_wl, wide, bucket);
  const uint32_t pos = off[cls * 16 + bucket] + atomicAdd(ctl + kCtlBucket + 16 * kLists + cls * 16 + bucket, 1u);
  lists[(size_t)cls * n_chunk + pos] = r;
}

// ------------------------------------------------------------------------------------------------
// K1b: exact nearest-rank p99 (p50, p95) by radix select; goodput (Eq. 1)
// ------------------------------------------------------------------------------------------------
// Pass 1 histograms every value of the row by a log-scale digit (its highest set bit and the 4 bits below
// it: 464 bins, monotone in the value, each bucket a contiguous range whose values share all bits above bit
// t - 4, t = the highest set bit), which finds the bucket holding the wanted rank with a relative width of
// 1/16.  Pass 2 copies that bucket's values into shared memory (when they fit, kSelCap; for LL rows the 99th
// percentile's bucket holds a few dozen values): <= 256 of them are ranked by direct counting, more by 8-bit
// radix passes in shared memory.  A bucket that does not fit continues with 8-bit radix passes over the row.
constexpr uint32_t kSelCap = 1024, kLogBins = 512;

__device__ __forceinline__ uint32_t log_bin(uint32_t v) {   // v < 16: v; else 16 + 16 (t - 4) + 4 bits below t
  const uint32_t t = 31u - (uint32_t)__clz(v | 1u);
  return v < 16u ? v : 16u * (t - 3u) + ((v >> (t - 4u)) & 15u);
}

// every value of a global row, 16-B loads two deep per thread when the row is 16-B aligned (the loop is
// bound by load latency, not by bytes: a plain scalar loop keeps one load in flight per thread)
template <class F>
__device__ __forceinline__ void for_row(const uint32_t* __restrict__ row, uint32_t n, F f) {
  const uint32_t bs = blockDim.x;
  uint32_t e0 = 0;
  if ((reinterpret_cast<uintptr_t>(row) & 15u) == 0) {
    const uint4* r4 = reinterpret_cast<const uint4*>(row);
    const uint32_t n4 = n >> 2;
    for (uint32_t e = threadIdx.x; e < n4; e += 2 * bs) {
      const uint4 a = r4[e];
      const bool hb = e + bs < n4;
      const uint4 b = hb ? r4[e + bs] : uint4{0, 0, 0, 0};
      f(a.x); f(a.y); f(a.z); f(a.w);
      if (hb) { f(b.x); f(b.y); f(b.z); f(b.w); }
    }
    e0 = n4 << 2;
  }
  for (uint32_t e = e0 + threadIdx.x; e < n; e += bs) f(row[e]);
}

// warp 0: the bin holding the kk-th largest of hist[0, 8 * 32 * per) (per bins per lane, suffix sums over the
// lanes); writes the bin, the rank inside it and its count
template <int PER>
__device__ __forceinline__ void find_bin(const uint32_t* hist, uint32_t kk, uint32_t* s_dig, uint32_t* s_kk,
                                         uint32_t* s_cnt) {
  const int lane = threadIdx.x;
  uint32_t c[PER], sum = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    c[q] = hist[lane * PER + q];
    sum += c[q];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_down_sync(FULL, incl, d);
    if (lane + d < 32) incl += v;
  }
  if (incl >= kk && incl - sum < kk) {
    uint32_t above = incl - sum, dg = 0, kn = 0, cnt = 0;
#pragma unroll
    for (int q = PER - 1; q >= 0; --q) {
      if (kn == 0 && above + c[q] >= kk) {
        dg = (uint32_t)(PER * lane + q);
        kn = kk - above;
        cnt = c[q];
      }
      above += c[q];
    }
    *s_dig = dg;
    *s_kk = kn;
    *s_cnt = cnt;
  }
}

// one 8-bit radix pass: digit (v >> sh) & (2^w - 1) over the values of src whose bits >= sh + w equal those of
// prefix; returns the digit holding the kk-th largest and updates kk to the rank inside it
__device__ __forceinline__ uint32_t select_pass(const uint32_t* src, uint32_t n, uint32_t prefix, uint32_t sh,
                                                uint32_t w, uint32_t& kk, uint32_t* hist, uint32_t* s_dig,
                                                uint32_t* s_kk, uint32_t* s_cnt) {
  for (uint32_t i = threadIdx.x; i < 256u; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const uint32_t hs = sh + w;                      // bits >= hs must match the prefix
  const uint32_t dm = (1u << w) - 1u;
  for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) {
    const uint32_t v = src[e];
    if (hs >= 32 || (v >> hs) == (prefix >> hs)) atomicAdd(hist + ((v >> sh) & dm), 1u);
  }
  __syncthreads();
  if (threadIdx.x < 32) find_bin<8>(hist, kk, s_dig, s_kk, s_cnt);
  __syncthreads();
  kk = *s_kk;
  return *s_dig;
}

__global__ void __launch_bounds__(256) slo_select_kernel(const SimParams p) {
  __shared__ uint32_t hist[kLogBins];
  __shared__ uint32_t cand[kSelCap];
  __shared__ uint32_t s_digit, s_kk, s_cnt, s_m, s_res;
  const uint32_t N = p.warmup + p.seg;
  const uint32_t n = p.seg;                        // row length (stop rule: uncounted entries hold UINT32_MAX)

  const uint32_t live_cfg = p.live ? *p.live : 0xFFFFFFFFu;
  for (uint32_t t = blockIdx.x; t < p.n_chunk; t += gridDim.x) {
    const uint32_t r = p.r_base + t;
    if (p.live && r / p.n_seeds >= live_cfg) continue;   // a skipped config (slo_run_args.d_live_configs)
    const slo_replica_result pr = p.part[r];
    if (pr.flags & 1u) {
      if (threadIdx.x == 0) {
        p.p99[r] = 0xFFFFFFFFu;
        if (p.p50) p.p50[r] = 0xFFFFFFFFu;
        if (p.p95) p.p95[r] = 0xFFFFFFFFu;
        p.goodput[r] = -1.0;
        if (p.detail) p.detail[r] = pr;
      }
      continue;
    }
    const uint32_t* row = p.lat + (size_t)t * N + p.warmup;
    uint32_t res[3];
    const uint32_t nq = (p.p50 || p.p95) ? 3u : 1u;
    for (uint32_t qi = 0; qi < nq; ++qi) {          // p99, then p50 and p95 (nearest rank, ceil(q n))
      // nearest rank among the nm counted latencies; the n - nm uncounted ones are UINT32_MAX (the top), so
      // the rq-th smallest counted value is the (n - rq + 1)-th largest of the row
      const uint32_t nm = pr.n_measured;
      uint32_t rq = (uint32_t)(((qi == 0 ? 99ull : qi == 1 ? 50ull : 95ull) * nm + 99ull) / 100ull);
      if (rq == 0) rq = n;                           // no counted value (slo_select_rows): the row's largest
      uint32_t kk = n - rq + 1;
      // pass 1: log-scale histogram of the row
      for (uint32_t i = threadIdx.x; i < kLogBins; i += blockDim.x) hist[i] = 0;
      if (threadIdx.x == 0) s_m = 0;
      __syncthreads();
      for_row(row, n, [&](uint32_t v) { atomicAdd(hist + log_bin(v), 1u); });
      __syncthreads();
      if (threadIdx.x < 32) find_bin<16>(hist, kk, &s_digit, &s_kk, &s_cnt);
      __syncthreads();
      const uint32_t b = s_digit, m = s_cnt;
      kk = s_kk;
      uint32_t result;
      if (b < 16u) {                                 // an exact value
        result = b;
      } else {
        const uint32_t tb = b / 16u + 3u;            // the bucket's highest set bit
        const uint32_t lo = (16u | (b & 15u)) << (tb - 4u);   // its values: bits >= tb - 4 equal lo's
        uint32_t hi = tb - 4u;                       // bits [0, hi) still to select
        uint32_t prefix = lo;
        if (m <= kSelCap) {                          // pass 2: the bucket's values into shared memory
          for_row(row, n, [&](uint32_t v) {
            if ((v >> hi) == (lo >> hi)) cand[atomicAdd(&s_m, 1u)] = v;
          });
          __syncthreads();
          if (m <= blockDim.x) {                     // rank by counting: (greater, equal and earlier) = kk - 1
            if (threadIdx.x < m) {
              const uint32_t v = cand[threadIdx.x];
              uint32_t above = 0;
              for (uint32_t j = 0; j < m; ++j) {
                const uint32_t u = cand[j];
                above += (u > v || (u == v && j < threadIdx.x)) ? 1u : 0u;
              }
              if (above == kk - 1u) s_res = v;
            }
            __syncthreads();
            prefix = s_res;
            hi = 0;
          }
        }
        const uint32_t* src = m <= kSelCap ? cand : row;
        const uint32_t ns = m <= kSelCap ? m : n;
        while (hi > 0) {                             // the remaining digits, 8 bits at a time
          const uint32_t sh = hi >= 8u ? hi - 8u : 0u;
          prefix |= select_pass(src, ns, prefix, sh, hi - sh, kk, hist, &s_digit, &s_kk, &s_cnt) << sh;
          hi = sh;
        }
        result = prefix;
      }
      res[qi] = result;
      __syncthreads();
    }
    const uint32_t prefix = res[0];
    if (threadIdx.x == 0) {
      if (p.p50) p.p50[r] = res[1];
      if (p.p95) p.p95[r] = res[2];
      p.p99[r] = prefix;
      p.goodput[r] = (double)((uint64_t)pr.slo_met * 1000000ull) / (double)pr.window_us;
      if (p.detail) {
        slo_replica_result d = pr;
        d.p99_us = prefix;
        p.detail[r] = d;
      }
    }
    __syncthreads();
  }
}

}  // namespace slo
