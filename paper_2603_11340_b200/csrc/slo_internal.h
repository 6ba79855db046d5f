// slo_internal.h — shared between the kernels and the C-ABI glue of libslosim.so (not installed).
#pragma once
#include <cstdint>

#include "../../include/slo_sim.h"

namespace slo {

constexpr int kMaxWarpsPerBlock = 8;
constexpr int kDefaultWarpsPerBlock = 4;

struct DevWorkload {      // device copy of one slo_workload
  uint32_t kind, start_state;
  uint64_t gap_q16[2];
  uint64_t soj[2];
  uint32_t p_lo, p_ncw, p_off;
  uint32_t o_lo, o_ncw, o_off;
  slo_timing t;
  uint32_t stream_id, pad;
};

// Per-warp shared-memory state of K1 (followed by the p99 candidate buffer of `cap` u32).  Warp-uniform
// values that are touched rarely live here instead of in registers (K1 is register-bound).
struct WarpRing {
  uint64_t a[64];      // arrival time of request j at a[j & 63]
  uint64_t kap[64];    // kappa_k (k-th completion time, ascending) at kap[k & 63]
  uint32_t po[64];     // P | (O << 16)
  uint32_t w3[64];     // noise word of request j
  uint32_t hist[256];  // radix-select histogram
  uint32_t tm1[16];    // T_a - 1 for a = 1..gp (gp = #{a : T_a > 0})
  uint8_t guide[256];  // A(u) at the top of bucket u >> 24 | 0x80 if a threshold lies inside the bucket
  uint8_t slot[32];    // spec decode: lane of the s-th unfinished member
  // arrival-process state (touched once per 32 generated requests)
  uint64_t g[2];       // scaled mean gaps (Q48.16)
  uint64_t rho[2];     // floor((2^64 - 1) / g), 0 without arrivals
  uint64_t last;       // a of the last generated request (kind 0) or its tau (kinds 1, 2)
  uint64_t pstart, pD, pU, pLam;
  uint32_t ph, pstate;
  uint64_t nphase;     // PHASE blocks drawn
  uint64_t a_w;        // arrival time of the first measured request
  uint64_t alpha0, alpha1;
  uint32_t pre_base, pre_tok, noise, pad;
};
static_assert(sizeof(WarpRing) % 16 == 0, "WarpRing alignment");

struct SimParams {
  const slo_knobs* cfg;
  const uint64_t* seeds;
  const DevWorkload* wl;
  const uint32_t* tables;
  uint32_t* queue;
  uint32_t* p99;
  double* goodput;
  slo_replica_result* detail;
  uint32_t* lat;
  slo_stats* stats;
  uint32_t n_cfg, n_seeds, n_rep, n_wl;
  uint32_t warmup, seg, slo_us, crn;
  uint32_t topk, cap, warp_bytes, pad;
};

__global__ void slo_sim_kernel(const SimParams p);
__global__ void slo_aggregate_kernel(const slo_replica_result* detail, uint32_t n_cfg, uint32_t n_seeds,
                                     slo_config_agg* agg);
__global__ void slo_aggregate_reduce_kernel(const slo_config_agg* parts, uint32_t n_parts, uint32_t n_cfg,
                                            slo_config_agg* out);
__global__ void slo_climb_kernel(slo_space space, slo_score_params sp, slo_knobs* cands, uint32_t n_cand,
                                 const slo_config_agg* aggs, uint32_t n_parts, slo_climb_state* state,
                                 int64_t* scores);

// host+device neighbour generation
__host__ __device__ uint32_t neighbors_of(const slo_space& sp, const slo_knobs& K, slo_knobs* out, uint32_t cap);

size_t warp_bytes_for(uint32_t cap);

}  // namespace slo
