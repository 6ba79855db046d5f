// slo_internal.h — shared between the kernels and the C-ABI glue of libslosim.so (not installed).
#pragma once
#include <cstdint>

#include "../../include/slo_sim.h"

namespace slo {

constexpr int kMaxWarpsPerBlock = 8;
constexpr int kDefaultWarpsPerBlock = 4;
// K0 work lists: static batching by lane-group size G = 8, 16, 32 (>= min(C, B) narrow, >= max(C, B) wide, or
// 32 for a lone replica; K1), then continuous batching by G = 8, 16, 32 >= min(C, B) (wide: >= B) (K1c), then
// closed loops with think time (kind 4) by G = 8, 16, 32 >= max(C, B): static (K1t), continuous (K1c, think)
// and (split path only) list 12: static batching with min(C, B) = 1, every batch a single request (K1s's scan),
// list 13: static batching with G = 4 >= min(C, B) (K1s, eight replicas per warp), list 14: continuous batching
// with min(C, B) = 1 (K1e's scan), list 15: continuous batching with G = 4 >= min(C, B) (K1c)
constexpr int kLists = 16;
constexpr int kScanList = 12, kG4List = 13, kCScanList = 14, kCG4List = 15;
constexpr int kGenLists = 10;  // K1g's lists: 12, 13, 0, 1, 2 (static), 14, 15, 3, 4, 5 (continuous)
// control words: list lengths [kLists], K1 cursors [kLists], K0 per-(list, bucket) counts and cursors
// control words: list lengths [kLists], K1 cursors [kLists], K0 per-(list, bucket) counts and cursors
constexpr int kCtlBucket = 64, kCtlWords = kCtlBucket + 2 * 16 * kLists;

struct DevWorkload {      // device copy of one slo_workload
  uint32_t kind, start_state;
  uint64_t gap_q16[2];
  uint64_t soj[2];
  uint32_t p_lo, p_ncw, p_off, p_goff;   // cut points at tables[off], 256-entry bucket guide at tables[goff]
  uint32_t o_lo, o_ncw, o_off, o_goff;
  slo_timing t;
  uint32_t stream_id, batching;
};

struct SimParams {
  const slo_knobs* cfg;
  const uint64_t* seeds;
  const DevWorkload* wl;
  const uint32_t* tables;
  uint32_t* counts;            // [kLists] replicas per work list (K0); ctl[8..) K0 bucket counters
  uint32_t* cursor;            // [kLists] next list entry (K1)
  const uint32_t* lists;       // [kLists][n_chunk] replica indices: G = 8 / 16 / 32, continuous
  uint32_t* lat;               // [n_chunk][N] stored latency of every request of the chunk's replicas
  slo_replica_result* part;    // [n_rep] K1 -> K1b (the caller's detail buffer when given)
  uint32_t* p99;
  uint32_t* p50;               // optional further order statistics
  uint32_t* p95;
  double* goodput;
  slo_replica_result* detail;
  slo_stats* stats;
  uint32_t n_cfg, n_seeds, n_rep, n_wl;
  uint32_t r_base, n_chunk;    // this launch covers replicas [r_base, r_base + n_chunk)
  uint32_t warmup, seg, slo_us, crn;
  uint32_t warp_bytes, gpw;    // per-warp shared memory; K1s: lane groups per warp in use (1..4)
  uint32_t stop_n, stop_t;     // segment stop rule, 0, 0 = off
  const uint4* rec;            // split path: [n_chunk][N] request records written by K1g (nullptr: inline)
  const uint32_t* live;        // nullable: only configs [0, *live) are simulated (slo_run_args.d_live_configs)
};

template <bool STOP> __global__ void slo_sim_kernel_t(const SimParams p);       // K1 (STOP: §2.14 stop rule)
// K1s: the static-batching chain over K1g's request records (split path)
template <bool STOP> __global__ void slo_serve_kernel_t(const SimParams p);
// K1g: per-request records of the static-batching replicas (split path), one block per 2,048-request tile
constexpr int kGenThreads = 256, kGenPerThread = 8;
__global__ void slo_gen_kernel(const SimParams p, uint4* rec);
// K1c: continuous batching (§2.12); THINK: the kind-4 (think-time) lists 9-11
// (SPLIT: lists 3-5 fed by K1g's records, and first list 14, continuous min(C, B) = 1, by the max-plus scan K1e)
template <bool STOP, bool THINK, bool SPLIT> __global__ void slo_sim_cont_kernel_t(const SimParams p);
template <bool STOP> __global__ void slo_sim_think_kernel_t(const SimParams p); // K1t: think-time closed loop (§2.11)
__global__ void slo_classify_count_kernel(const slo_knobs* cfg, const DevWorkload* wl, uint32_t n_seeds,
                                          uint32_t r_base, uint32_t n_chunk, uint32_t n_wl, uint32_t wide,
                                          uint32_t* ctl, const uint32_t* live);
__global__ void slo_classify_kernel(const slo_knobs* cfg, const DevWorkload* wl, uint32_t n_seeds, uint32_t r_base,
                                    uint32_t n_chunk, uint32_t n_wl, uint32_t wide, uint32_t* ctl, uint32_t* lists,
                                    const uint32_t* live);
__global__ void slo_select_kernel(const SimParams p);
size_t group_warp_bytes();   // per-warp shared memory of K1
size_t serve_warp_bytes();   // per-warp shared memory of K1s
size_t cont_warp_bytes();    // per-warp shared memory of K1c
__global__ void slo_aggregate_kernel(const slo_replica_result* detail, uint32_t n_cfg, uint32_t n_seeds,
                                     slo_config_agg* agg);
__global__ void slo_aggregate_reduce_kernel(const slo_config_agg* parts, uint32_t n_parts, uint32_t n_cfg,
                                            slo_config_agg* out);
__global__ void slo_climb_kernel(slo_space space, slo_score_params sp, slo_knobs* cands, uint32_t n_cand,
                                 const slo_config_agg* aggs, uint32_t n_parts, slo_climb_state* state,
                                 int64_t* scores);

// lookahead climb (NEXT-4, slo_climb.cu): the round's candidate table U and last round's (the cache)
constexpr uint32_t kLookCap = SLO_LOOKAHEAD_CAP;
struct LookTable {
  uint32_t n_old, n_new, n_sim, overflow;     // overflow: |U| when it exceeded kLookCap (0 otherwise)
  uint32_t old_h[kLookCap], new_h[kLookCap];  // knob hashes
  int32_t map[kLookCap];                      // U entry i: >= 0 cached (old index), < 0 simulated (list -map - 1)
  slo_knobs old_k[kLookCap], new_k[kLookCap];
  slo_config_agg old_a[kLookCap];
};
__global__ void slo_lookahead_prepare_kernel(slo_space space, const slo_climb_state* state, LookTable* T,
                                             slo_knobs* sim);
__global__ void slo_lookahead_step_kernel(slo_space space, slo_score_params sp, LookTable* T,
                                          const slo_config_agg* aggs, uint32_t n_parts, uint32_t n_cand,
                                          slo_climb_state* state, slo_climb_state* traj);

// peer exchange (NEXT-4): window = [flags 2 x kXMaxRanks u64][inbox 2 parities x world x n_cfg slo_config_agg]
constexpr uint32_t kXMaxRanks = 16;
constexpr size_t kXHeader = 2 * kXMaxRanks * sizeof(uint64_t);
struct XState {                 // rank-local (not shared)
  unsigned long long epoch;     // completed exchanges
  unsigned int arrive_push, arrive_wait, error, pad;
};
__global__ void slo_aggregate_push_kernel(const slo_replica_result* detail, uint32_t n_cfg, uint32_t n_seeds,
                                          char* const* peers, uint32_t world, uint32_t rank, XState* st);
__global__ void slo_exchange_wait_kernel(const char* window, uint32_t n_cfg, uint32_t world, XState* st,
                                         slo_config_agg* out);

__global__ void slo_philox_peak_kernel(uint32_t iters, uint32_t* sink);   // K4: RNG roofline
// K6 exhaustive transform self-test (slo_selftest.cu): what 0 E_q, 1 a length table, 2 A(u), 3 noise factor
struct SelftestArgs {
  uint32_t what, arg0, arg1, arg2;
  uint32_t off, goff, lo, nbins, viol_slot, pad;
};
__global__ void slo_selftest_kernel(SelftestArgs a, const uint32_t* tables, uint64_t* out);
// K5 Pareto front (slo_pareto.cu): scratch bytes for n configs (cub temp part returned separately), launch
size_t pareto_scratch_bytes(uint32_t n, size_t* cub_bytes_out);
cudaError_t pareto_launch(const slo_config_agg* agg, uint32_t n, uint8_t* front, uint32_t* count, void* scratch,
                          size_t cub_bytes, cudaStream_t st);

// host+device neighbour generation
__host__ __device__ uint32_t neighbors_of(const slo_space& sp, const slo_knobs& K, slo_knobs* out, uint32_t cap);


}  // namespace slo
