/* include/slo_sim.h — C ABI of libslosim.so: the SLO-Tuner serving simulator (arXiv 2603.11340) as a
 * batched Monte-Carlo hot path on NVIDIA B200 (sm_100a).
 *
 * The paper's method:
 *   - discrete-event simulator (§2.2 "Simulator"): arrivals -> FCFS queue -> idle server forms a
 *     batch of up to B requests, optionally waiting up to max_wait -> prefill driven by the longest prompt
 *     -> decode depending on active sequences and speculative decoding;
 *   - goodput (Eq. 1) and empirical p99 per segment;
 *   - score S = goodput - lambda*max(0, p99 - SLO) - hw_cost (Eq. 2-3);
 *   - hill-climb control loop (Alg. 1; neighbour rule P:142).
 * The exact integer model both this library and the CPU oracle implement is DESIGN.md §2.
 *
 * Conventions
 *   - Every call returns slo_status; nothing throws or aborts.  On a non-OK status outputs are undefined.
 *   - "d_" pointers are CUDA device pointers (e.g. torch tensors' data_ptr()); "h_" pointers are host.
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).  Device calls validate
 *     host-visible arguments synchronously (SLO_E_INVAL, nothing enqueued), then enqueue on `stream` and
 *     return; results are valid once the stream reaches that point.
 *   - The caller owns every buffer it passes; slo_sim_create deep-copies the workload tables.
 *   - One handle may be used by one host thread at a time; distinct handles are independent.
 *   - All integer structs are little-endian PODs with the sizes stated (checked by static asserts).
 */
#ifndef SLO_SIM_H
#define SLO_SIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t slo_status;
#define SLO_OK 0
#define SLO_E_INVAL (-1)        /* null required pointer, zero size, bad table, reserved != 0, ...      */
#define SLO_E_NOMEM (-2)        /* device or host allocation failed                                   */
#define SLO_E_CUDA (-3)         /* a CUDA runtime call failed; text in slo_last_error                 */
#define SLO_E_RANGE (-4)        /* a size exceeds a documented limit                                  */
#define SLO_E_DEVICE (-5)       /* no usable sm_100 device                                            */
#define SLO_E_UNSUPPORTED (-6)

#define SLO_MAX_REQUESTS (1u << 22)   /* warmup_len + segment_len per replica                        */
#define SLO_MAX_LENGTH 4096u          /* largest prompt/output length a table may produce            */

typedef struct slo_sim slo_sim; /* opaque: one CUDA device, owns scratch and the copied workload tables */

/* Integer microsecond timing block.  Each value must be < 2^20 and the     */
/* worst-case step (gamma = 16, W = 4, n = 32) < 2^31 us, else slo_sim_create returns SLO_E_INVAL.        */
typedef struct {
  uint32_t pre_base_us, pre_tok_us;             /* prefill = f * (pre_base + pre_tok * max P) / 1e6      */
  uint32_t dec_base_us, dec_seq_us;             /* plain step  d(n) = dec_base + dec_seq * n             */
  uint32_t dr_base_us, dr_seq_us;               /* spec step   d(n) = g*W*(dr_base + dr_seq*n) + ver_base */
  uint32_t ver_base_us, ver_seq_us, ver_tok_us; /*            + ver_seq*n + ver_tok*(W*g+1)*n (R10, R28)  */
  uint32_t noise_step_ppm;                      /* per-batch Irwin-Hall noise step, <= 1960; 0 = none    */
} slo_timing;                                   /* 40 B */

/* Arrival process. */
typedef struct {
  uint32_t kind;                /* 0 Poisson, 1 MMPP-2 (exponential sojourns), 2 on/off (fixed sojourns), */
                                /* 3 closed loop: `conc` users with zero think time — every request is    */
                                /*   waiting from t = 0 and latency is measured from issue */
                                /* 4 closed loop with exponential think time of mean mean_gap_q16[0]      */
                                /*   (finite; 0 allowed): completion k starts user chain k + C after      */
                                /*   Z_k (THINK block (k, 4, 0)); static or continuous batching          */
                                /*                                                       */
  uint32_t start_state;         /* 0 or 1                                                               */
  uint64_t mean_gap_q16[2];     /* per-state mean gap, Q48.16 us, <= 2^48; UINT64_MAX = no arrivals     */
  uint64_t mean_sojourn_us[2];  /* kinds 1, 2: per-state mean/fixed sojourn, >= 1                       */
} slo_arrivals;                 /* 40 B */

/* One workload: arrivals, length tables, timing, CRN stream id. */
typedef struct {
  slo_arrivals arr;
  const uint32_t* prompt_cw;    /* host ptr, prompt_ncw non-decreasing Q32 cut points (copied at create) */
  uint32_t prompt_lo, prompt_ncw; /* P = prompt_lo + #{l : cw[l] <= u}; lo >= 1; lo + ncw <= 4096       */
  const uint32_t* output_cw;
  uint32_t output_lo, output_ncw;
  slo_timing timing;
  uint32_t stream_id;           /* cfgkey in CRN mode                                  */
  uint32_t batching;            /* 0: static batches; 1: continuous,         */
                                /* iteration-level (vLLM-style): prefill or */
                                /* decode iterations over a running set of <= max_num_seqs requests;     */
                                /* max_wait_us is not used.  Other values: SLO_E_INVAL at create.         */
} slo_workload;

/* One logical-knob configuration, 32 B.  Validity is checked per
 * replica on the device; an invalid record yields flags bit 0, p99 = UINT32_MAX, goodput = -1.0. */
typedef struct {
  uint8_t conc;                 /* client concurrency C in [1,32]                                        */
  uint8_t max_num_seqs;         /* batch limit B in [1,32]                                               */
  uint8_t draft_len;            /* gamma = k = num_speculative_tokens in [0,16]                          */
  uint8_t spec_on;              /* 0 or 1; 0 => gamma_eff = 0                                           */
  uint8_t draft_width;          /* W in [1,4]; alpha_eff = 1 - (1 - alpha)^W                             */
  uint8_t workload;             /* index into the create-time workload array                             */
  uint16_t rate_scale_q8;       /* offered-load multiplier, 256 = 1.0, >= 1                              */
  uint32_t accept_q16;          /* per-position acceptance alpha in [0, 65536]                           */
  uint32_t max_wait_us;         /* [0, 50000]                                                    */
  uint32_t reserved[4];         /* must be 0                                                             */
} slo_knobs;

/* Per-replica outputs, 32 B. flags: bit0 invalid knobs, bit1 a latency saturated u32,
 * bit2 the stop rule (slo_run_args) was not met before the segment's requests ran out. */
typedef struct {
  uint32_t p99_us, slo_met, n_measured, flags;
  uint64_t window_us, sum_latency_us;
} slo_replica_result;

/* Per-config aggregate over seeds, 32 B. */
typedef struct {
  uint64_t sum_p99_us, sum_slo_met, sum_window_us;
  uint32_t n_seeds, flags;
} slo_config_agg;

/* Work counters of one run (exact algorithmic work, summed over replicas), 64 B. */
typedef struct {
  uint64_t requests, batches, decode_steps, member_steps, philox_blocks, replicas, reserved[2];
} slo_stats;

typedef struct {
  uint32_t crn;                 /* 1 (default): cfgkey = workload.stream_id; 0: FNV-1a of the knob record */
  uint32_t warps_per_block;     /* 0 = default (4)                                                        */
  uint32_t blocks_per_sm;       /* 0 = as many as fit                                                     */
  uint32_t scratch_mb;          /* latency-row scratch per launch chunk in MiB; 0 = default (4096). A run */
                                /* whose rows exceed it is split into chunks of replicas (same results)  */
  uint32_t group_policy;        /* static-batching lane groups (results never depend on it): 0 auto      */
                                /* (whole warp for <= 1 replica per SM, else narrow G >= min(C,B)),       */
                                /* 1 narrow, 2 wide G >= max(C,B), 3 whole warp (G = 32); else INVAL      */
  uint32_t gen_policy;          /* static batching without think time (results never depend on it):      */
                                /* 0 auto (= 2), 1 inline generation inside K1, 2 split: K1g writes every */
                                /* request's 16-B record (16 B x chunk x N of scratch), K1s runs the     */
                                /* batch chain over them; else INVAL                                      */
  uint32_t reserved[2];         /* must be 0                                                              */
} slo_sim_opts;

typedef struct {                /* read-only launch facts of a handle                                    */
  int32_t device, sm_count, warps_per_block, blocks_per_sm;
  int32_t regs_per_thread, smem_per_warp_bytes, reserved[2];
} slo_sim_info;

/* Create a handle on CUDA device `device` with `n_wl` (1..255) workloads.  opts may be NULL.
 * Errors: SLO_E_INVAL (bad table / timing / arrivals), SLO_E_DEVICE, SLO_E_NOMEM, SLO_E_CUDA. */
slo_status slo_sim_create(int device, const slo_workload* wl, uint32_t n_wl, const slo_sim_opts* opts,
                          slo_sim** out);
/* Synchronise the handle's work and free everything it owns.  NULL is a no-op. */
slo_status slo_sim_destroy(slo_sim* h);
slo_status slo_sim_get_info(const slo_sim* h, slo_sim_info* info);

/* K1: simulate replicas r = c * n_seeds + s (config-major) for every (config c, seed s) pair.
 * Each replica simulates warmup_len + segment_len requests and writes
 *   d_p99_us[r] (u32, nearest-rank p99 of the measured latencies) and d_goodput[r] (f64, Eq. 1);
 * optionally d_detail[r], d_latencies[r * (warmup_len + segment_len) + i] (every request's stored
 * latency, debug/parity only) and *d_stats (one slo_stats accumulated over the launch, overwritten).
 * Limits: n_configs * n_seeds < 2^31, warmup_len + segment_len <= SLO_MAX_REQUESTS, slo_us < UINT32_MAX.
 * Errors: SLO_E_INVAL (null required pointer, segment_len == 0, n == 0), SLO_E_RANGE, SLO_E_CUDA. */
slo_status slo_sim_run_batch(slo_sim* h, const slo_knobs* d_configs, uint32_t n_configs,
                             const uint64_t* d_seeds, uint32_t n_seeds, uint32_t segment_len,
                             uint32_t warmup_len, uint32_t slo_us, uint32_t* d_p99_us, double* d_goodput,
                             slo_replica_result* d_detail, uint32_t* d_latencies, slo_stats* d_stats,
                             void* stream);

/* Extended form of slo_sim_run_batch (the latter is slo_sim_run with the extra outputs NULL). */
typedef struct {
  const slo_knobs* d_configs;   uint32_t n_configs;
  const uint64_t* d_seeds;      uint32_t n_seeds;
  uint32_t segment_len, warmup_len, slo_us;
  uint32_t* d_p99_us;           /* [R] nearest-rank p99 (required)                                       */
  double* d_goodput;            /* [R] Eq. (1) (required)                                                 */
  slo_replica_result* d_detail; /* [R] or NULL                                                            */
  uint32_t* d_latencies;        /* [R x (warmup_len + segment_len)] or NULL                              */
  slo_stats* d_stats;           /* or NULL                                                                */
  uint32_t* d_p50_us;           /* [R] nearest-rank p50 or NULL                             */
  uint32_t* d_p95_us;           /* [R] nearest-rank p95 or NULL                                           */
  /* segment stop rule, both 0 = off (R15's fixed count): the segment ends at
   * the first measured completion t* with >= stop_min_completions measured completions and
   * t* - t0 >= stop_min_time_us; only requests completing by t* count (n_measured varies), later ones
   * store latency UINT32_MAX; flags bit 2 if the segment's requests ran out first.  Work counters then
   * count what was simulated up to the stop.  The kernels stop simulating at t*, which is exact only if no
   * later batch or iteration can also end at t*: with a stop rule every workload must have
   * pre_base + pre_tok >= 3 and dec_base + dec_seq >= 3 and ver_base + ver_seq + ver_tok >= 3 (every batch and
   * iteration then lasts >= 1 us under any noise factor >= 0.4004), else SLO_E_INVAL. */
  uint32_t stop_min_completions, stop_min_time_us;
  /* device u32 or NULL: only configs [0, *d_live_configs) are simulated; replicas of later configs are skipped
   * entirely (nothing written for them, not counted) — a graph-captured caller with a fixed n_configs and a
   * count known only on the device (the lookahead climb's simulation list) pays nothing for its padding */
  const uint32_t* d_live_configs;
} slo_run_args;
slo_status slo_sim_run(slo_sim* h, const slo_run_args* args, void* stream);

/* The same call on HOST buffers (end-to-end use): copies h_configs / h_seeds to the handle's device
 * scratch, runs K1 on `stream`, copies the outputs back and synchronises `stream` before returning.
 * h_detail and h_stats may be NULL.  Pinned host memory makes the copies asynchronous DMA. */
slo_status slo_sim_run_batch_host(slo_sim* h, const slo_knobs* h_configs, uint32_t n_configs,
                                  const uint64_t* h_seeds, uint32_t n_seeds, uint32_t segment_len,
                                  uint32_t warmup_len, uint32_t slo_us, uint32_t* h_p99_us,
                                  double* h_goodput, slo_replica_result* h_detail, slo_stats* h_stats,
                                  void* stream);

/* K2: d_agg[c] = sum over seeds s of d_detail[c * n_seeds + s] (integer sums, flags OR). */
slo_status slo_aggregate(slo_sim* h, const slo_replica_result* d_detail, uint32_t n_configs,
                         uint32_t n_seeds, slo_config_agg* d_agg, void* stream);
/* d_out[c] = sum over parts p of d_parts[p * n_configs + c] (e.g. per-rank aggregates after an
 * all-gather; integer sums make the result independent of rank order). */
slo_status slo_aggregate_reduce(slo_sim* h, const slo_config_agg* d_parts, uint32_t n_parts,
                                uint32_t n_configs, slo_config_agg* d_out, void* stream);

/* Climb space.  dims: 0 conc, 1 max_num_seqs, 2 draft_len, 3 draft_width,
 * 4 max_wait_us.  stencil: 0 paper-live (<= 7 neighbours), 1 sim (<= 8), 2 wide-32 (<= 31). */
typedef struct {
  uint32_t stencil;
  int32_t lo[5], hi[5], step[5];
} slo_space;

/* Eq. (2)-(3) and Alg. 1 parameters in fixed point.  Live controller: 5000, 10000,
 * 10000, 20000, 20000, w_W = w_k = 0, viol_mult 1, ema 0.  The paper's simulator controller (P:173-174,
 * P:188) sets viol_mult = 10, w_W/w_k > 0 and ema_beta_q16 > 0. */
typedef struct {
  int64_t lambda_milli, w_conc_micro, w_max_micro, w_spec_micro, delta_micro;
  uint32_t slo_us, strict_alg1;
  int64_t w_W_micro, w_k_micro;   /* draft/verifier cost w_W*W + w_k*(k_max - gamma) when speculating */
  uint32_t viol_mult;             /* violation term multiplier: 1 live, 10 simulator ("10 lambda")     */
  uint32_t k_max;                 /* verifier-cadence reference of w_k (16)                             */
  uint32_t ema_beta_q16;          /* EMA weight of the current point's p99 in Q16; 0 = raw p99          */
  uint32_t reserved;              /* must be 0                                                          */
} slo_score_params;             /* 80 B */

typedef struct {
  slo_knobs K, K_best;
  int64_t S_best_micro;
  uint32_t step, has_best;
  int32_t moved;                /* last step: 1 if K moved                                               */
  uint32_t argmax;              /* last step: index of K* among the candidates                           */
  uint32_t n_next;              /* number of valid candidates written for the next step                  */
  uint32_t has_ema;             /* ema_p99_us holds a value                                              */
  uint64_t ema_p99_us;          /* EMA of the current point's seed-mean p99 (ema_beta_q16 > 0)           */
} slo_climb_state;              /* 104 B */

/* Host helper: neighbours of K, written to out[0..*n) (cap >= 31 recommended). */
slo_status slo_neighbors(const slo_space* space, const slo_knobs* K, slo_knobs* out, uint32_t cap,
                         uint32_t* n);

/* K3 (device-resident Alg. 1 step, one warp):
 *   aggregates d_aggs[p * n_cand + k] summed over p < n_parts are the measurements of candidate
 *   d_cands[k] (d_cands[0] must equal state.K); computes every score (Eq. 3, INT64_MIN for invalid),
 *   argmax over k >= 1 (lowest index on ties), the move rule, best-so-far, then OVERWRITES
 *   d_cands[0..n_cand) with [K', neighbours(K'), padding] for the next step (padding records have
 *   conc = 0, i.e. are invalid and cost nothing).  d_scores (nullable) receives the scores.
 * n_cand in [1, 32]. */
slo_status slo_hillclimb_step(slo_sim* h, const slo_space* space, const slo_score_params* sp,
                              slo_knobs* d_cands, uint32_t n_cand, const slo_config_agg* d_aggs,
                              uint32_t n_parts, slo_climb_state* d_state, int64_t* d_scores,
                              void* stream);

/* ---- Peer exchange of the per-config aggregates (SV §8(f) NEXT-4) ----------------------
 * The one exchange of the method — pooling the per-config aggregates over ranks before the score and the
 * argmax (Eq. 1 pooled over seeds, R17; Alg. 1) — done by the aggregation kernel itself: every
 * rank's K2x pushes its aggregates straight into every peer's exchange window over NVLink (CUDA IPC
 * peer pointers, one process per GPU), then publishes an epoch flag; K2w waits for all flags and sums the
 * parts in rank order (integer sums: bit-identical to the NCCL all-gather + slo_aggregate_reduce path).
 * Windows are double-buffered by epoch parity, so a rank can never overwrite a part a peer has not read.
 * Usage: slo_exchange_create on every rank -> all-gather the 64-byte handles (any transport, e.g. a
 * torch.distributed group) -> slo_exchange_open -> slo_aggregate_exchange per step (stream-ordered, graph-
 * capturable; all ranks must call it the same number of times).  A rank that waits > 30 s for a peer gives
 * up (results undefined) and latches an error readable with slo_exchange_error. */
#define SLO_EXCHANGE_MAX_RANKS 16u
#define SLO_EXCHANGE_HANDLE_BYTES 64u
typedef struct slo_exchange slo_exchange;
/* Allocate this rank's window for n_cfg aggregates among `world` ranks (2..16) on h's device and write its
 * CUDA IPC handle (64 B) to h_handle_out.  Errors: SLO_E_INVAL, SLO_E_RANGE, SLO_E_NOMEM, SLO_E_CUDA. */
slo_status slo_exchange_create(slo_sim* h, uint32_t world, uint32_t rank, uint32_t n_cfg, slo_exchange** out,
                               void* h_handle_out);
/* Map the peers' windows: h_handles = world x 64 B in rank order (this rank's own entry is ignored). */
slo_status slo_exchange_open(slo_exchange* x, const void* h_handles);
/* K2x + K2w: d_pooled[c] = sum over ranks r of (sum over seeds s of rank r's d_detail[c * n_seeds_r + s]),
 * n_seeds = this rank's seed count.  d_pooled (n_cfg records) feeds slo_hillclimb_step with n_parts = 1. */
slo_status slo_aggregate_exchange(slo_sim* h, slo_exchange* x, const slo_replica_result* d_detail,
                                  uint32_t n_seeds, slo_config_agg* d_pooled, void* stream);
/* Synchronising read of the latched error word (0 = ok, 1 = a wait for a peer timed out). */
slo_status slo_exchange_error(slo_exchange* x, uint32_t* h_err);
slo_status slo_exchange_destroy(slo_exchange* x);

/* K5: the Pareto front of a sweep ("the resulting Pareto front").
 * For each of n_cfg aggregates (slo_aggregate output, device), d_on_front[c] = 1 iff config c is valid (no
 * invalid seed, n_seeds > 0) and no valid config dominates it on (minimise floor(sum_p99 / n_seeds) us,
 * maximise floor(sum_slo_met * 10^12 / sum_window) micro-rps) — dominate = no worse in both, better in one;
 * equal points do not dominate each other.  *d_count (nullable, device) = number of front configs.
 * O(n log n) on the device (two radix sorts and two scans; scratch owned by the handle).
 * Errors: SLO_E_INVAL (null pointers, n_cfg == 0), SLO_E_NOMEM, SLO_E_CUDA. */
slo_status slo_pareto_front(slo_sim* h, const slo_config_agg* d_agg, uint32_t n_cfg, uint8_t* d_on_front,
                            uint32_t* d_count, void* stream);

/* K4 (measurement only): the RNG roofline.  Every thread of a full-occupancy grid (sm_count x 8 blocks x
 * 256 threads) draws `iters` Philox4x32-10 blocks with distinct counters and XOR-folds them
 * into d_sink[thread] (so nothing is dead code); blocks drawn = sm_count * 2048 * iters.  The caller times
 * it on `stream` (bench.py reports blocks/s next to the simulator's).  d_sink: >= sm_count * 2048 u32. */
slo_status slo_philox_peak(slo_sim* h, uint32_t iters, uint32_t* d_sink, void* stream);

/* Measurement hook (bench.py's per-kernel roofline): while enabled, every run call records CUDA events on its
 * stream around each launch chunk's K0 (classify), K1g (split-path generation; 0 when inline), the chain kernels
 * (K1 / K1s / K1t / K1c) and K1b (select); slo_sim_profile_read waits for them and returns the summed elapsed
 * milliseconds h_ms[0..4] = (K0, K1g, chain, K1b, simulation = end of K0 to start of K1b) (h_ms: >= 5 doubles)
 * and the number of chunks, then clears the marks.  Calls made while the stream is being captured into a
 * CUDA graph record nothing.  Errors: SLO_E_INVAL (null), SLO_E_CUDA. */
slo_status slo_sim_profile(slo_sim* h, uint32_t enable);
slo_status slo_sim_profile_read(slo_sim* h, double* h_ms, uint32_t* h_chunks);

/* K6 (test instrumentation): exhaustive self-test of the integer transforms the simulation kernels use —
 * the SAME device functions, over all 2^32 inputs (SURVEY §8(c) pins table) — so tests can compare them with
 * the oracle (E_q) and with exact closed forms (lengths, acceptance, noise).  `what`:
 *   SLO_SELFTEST_EXP    : d_out[b] (b < 4096) = sum over u in [b 2^20, (b+1) 2^20) of
 *                         (E_q(u) ^ (u * 0x9E3779B97F4A7C15)) * 0xBF58476D1CE4E5B9 mod 2^64;
 *                         d_out[4096] = #{u : E_q(u) > E_q(u - 1)}.  out_len >= 4097.
 *   SLO_SELFTEST_LENGTH : workload arg0, table arg1 (0 prompt, 1 output): d_out[l - lo] =
 *                         #{u : length(u) = l} for l = lo .. lo + ncw; d_out[ncw + 1] = #{u : length(u) <
 *                         length(u - 1)} + out-of-range values.  out_len >= ncw + 2.
 *   SLO_SELFTEST_ACCEPT : accept_q16 arg0, draft_width arg1, gamma arg2: d_out[A] = #{u : A(u) =
 *                         A}, A = 0..16; d_out[17] = #{u : A(u) > A(u - 1)}.  out_len >= 18.  (K1 / K1c's 256-entry
 *                         byte guide.)
 *   SLO_SELFTEST_ACCEPT2: the same through K1g's 4096-entry fine guide (K1g).
 *   SLO_SELFTEST_NOISE  : noise_step_ppm arg0: d_out[k] = #{w : f(w) = 10^6 + (k - 510) arg0},
 *                         k = 0..1020; d_out[1021] = #{w : f(w) off that lattice}.  out_len >= 1022.
 * d_out (device, u64) is zeroed by the call; results are valid after `stream` completes.
 * Errors: SLO_E_INVAL (null pointers, unknown `what`, bad arguments, short out_len), SLO_E_CUDA. */
enum { SLO_SELFTEST_EXP = 0, SLO_SELFTEST_LENGTH = 1, SLO_SELFTEST_ACCEPT = 2, SLO_SELFTEST_NOISE = 3,
       SLO_SELFTEST_ACCEPT2 = 4 };
slo_status slo_selftest_transforms(slo_sim* h, uint32_t what, uint32_t arg0, uint32_t arg1, uint32_t arg2,
                                   uint64_t* d_out, uint32_t out_len, void* stream);

/* K1b on caller rows (SV §8(a) a9; "p99", S:123 / S:165 nearest rank): for each of n_rows contiguous rows
 * of row_len u32 values (device, [n_rows][row_len], row r at d_rows + r * row_len), the exact nearest-rank
 * order statistics among its first-counted values: with m = d_n_measured ? min(d_n_measured[r], row_len) :
 * row_len counted values and the row_len - m others equal to UINT32_MAX (the convention the simulation's stop
 * rule uses, §2.14), p_q = the ceil(q m)-th smallest value of the row (q = 0.99, 0.50, 0.95; m = 0 gives the
 * row's largest value, UINT32_MAX under that convention).  d_p99_us is required ([n_rows]); d_p50_us and
 * d_p95_us are optional (NULL: not computed).  The same kernel and code path as slo_sim_run_batch's select step;
 * enqueued on `stream`, results valid after it completes.  Uses handle scratch (32 B + 8 B per row).
 * Errors: SLO_E_INVAL (null handle / rows / d_p99_us, n_rows == 0, row_len == 0), SLO_E_RANGE (n_rows * row_len
 * >= 2^40), SLO_E_NOMEM, SLO_E_CUDA. */
slo_status slo_select_rows(slo_sim* h, const uint32_t* d_rows, uint32_t n_rows, uint32_t row_len,
                           const uint32_t* d_n_measured, uint32_t* d_p99_us, uint32_t* d_p50_us, uint32_t* d_p95_us,
                           void* stream);

/* Lookahead climb (SV §8(f) NEXT-4 "neighbour-of-neighbour lookahead"; Alg. 1).  A round takes two
 * Alg. 1 steps from one batch of simulations: U(K) = {K} u N(K) u (union over c in N(K) of N(c)) holds every
 * candidate the next two steps can score, whichever way the first step moves (<= 272 records for the wide-32
 * stencil), and a record's aggregate depends only on the record and the seeds (its Philox key is (seed, config
 * key), §2.1), so records the previous round measured are taken from its table (the cache) and only the rest
 * are simulated.  The trajectory is the plain climb's (slo_hillclimb_step with n_cand candidates) step for step.
 * d_table: SLO_LOOKAHEAD_TABLE_BYTES of device memory, zero-filled before the first round (empty cache).
 *   slo_lookahead_prepare: builds U(state.K), looks it up in the cache and writes the records to simulate into
 *     d_sim[0 .. SLO_LOOKAHEAD_CAP) (the rest padded with invalid records, conc = 0) and their count into the
 *     table's 3rd u32 word (byte offset 8); the caller then runs slo_sim_run on d_sim x seeds with
 *     d_live_configs = d_table + 8 bytes (the padding is then skipped entirely; slo_sim_run_batch also works,
 *     simulating the padding as invalid records) and slo_aggregate into SLO_LOOKAHEAD_CAP aggregates (n_parts rank
 *     parts of them, [part][SLO_LOOKAHEAD_CAP], for a seed-sharded multi-GPU climb);
 *   slo_lookahead_step: assembles U's aggregates (cache or the new parts, summed), takes two steps on *d_state
 *     (n_cand in [2, 32], the plain climb's candidate count), writes the state after each into d_traj[0..2)
 *     and keeps U's table as the next round's cache.
 * Enqueued on `stream` (graph-capturable: fixed launch sizes).  Errors: SLO_E_INVAL (null pointers, bad space or
 * score parameters, n_cand / n_parts out of range), SLO_E_CUDA.  A U larger than the capacity (not reachable
 * with the built-in stencils) is recorded in the table's 4th word. */
#define SLO_LOOKAHEAD_CAP 320
#define SLO_LOOKAHEAD_TABLE_BYTES 34576
slo_status slo_lookahead_prepare(slo_sim* h, const slo_space* space, const slo_climb_state* d_state, void* d_table,
                                 slo_knobs* d_sim, void* stream);
slo_status slo_lookahead_step(slo_sim* h, const slo_space* space, const slo_score_params* sp, void* d_table,
                              const slo_config_agg* d_aggs, uint32_t n_parts, uint32_t n_cand,
                              slo_climb_state* d_state, slo_climb_state* d_traj, void* stream);

const char* slo_status_string(slo_status s);
const char* slo_last_error(const slo_sim* h); /* detail of the last failing call on h (NULL h: global) */

#ifdef __cplusplus
}
#endif
#endif /* SLO_SIM_H */
