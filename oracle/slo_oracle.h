/* oracle/slo_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, single-threaded CPU oracle of the SLO-Tuner serving simulator (arXiv 2603.11340,
 * §2.2 "Simulator") as specified in DESIGN.md §2.  It shares no code, header, table or
 * constant generator with the CUDA path (paper_2603_11340_b200/csrc, include/slo_sim.h).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it.
 */
#ifndef SLO_ORACLE_H
#define SLO_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint32_t kind;              /* 0 Poisson, 1 MMPP-2 (exponential sojourns), 2 on/off (fixed sojourns),
                                 3 closed loop: C users, zero think time (every a_i = 0, latency from issue),
                                 4 closed loop with exponential think time of mean mean_gap_q16[0]
                                    */
  uint32_t start_state;
  uint64_t mean_gap_q16[2];   /* Q48.16 us; UINT64_MAX = no arrivals in that state */
  uint64_t mean_sojourn_us[2];
} orc_arrivals;

typedef struct {
  uint32_t pre_base_us, pre_tok_us, dec_base_us, dec_seq_us, dr_base_us, dr_seq_us,
           ver_base_us, ver_seq_us, ver_tok_us, noise_step_ppm;
} orc_timing;

typedef struct {
  orc_arrivals arr;
  const uint32_t* prompt_cw; uint32_t prompt_lo, prompt_ncw;   /* ncw cut points */
  const uint32_t* output_cw; uint32_t output_lo, output_ncw;
  orc_timing timing;
  uint32_t stream_id;
  uint32_t batching;          /* 0 static batches (§2.6), 1 continuous / iteration-level (§2.12) */
} orc_workload;

/* Knob record; its 32-byte little-endian layout is normative (FNV-1a key mode). */
typedef struct {
  uint8_t conc, max_num_seqs, draft_len, spec_on, draft_width, workload;
  uint16_t rate_scale_q8;
  uint32_t accept_q16, max_wait_us;
  uint32_t reserved[4];
} orc_knobs;

typedef struct {
  uint32_t p99_us, slo_met, n_measured, flags;
  uint64_t window_us, sum_latency_us;
  double goodput;           /* (double)(slo_met * 10^6) / (double)window_us, Eq. (1) */
  uint32_t p50_us, p95_us;  /* nearest-rank p50 and p95 */
} orc_result;

typedef struct {
  uint64_t philox_blocks;   /* REQ + PHASE + SPEC blocks the definition consumes */
  uint64_t batches;
  uint64_t decode_steps;    /* sum over batches of the batch's step count */
  uint64_t member_steps;    /* sum over requests of S_m */
} orc_counters;

typedef struct {            /* per-request trace (optional) */
  uint64_t a, s, form, c;
  uint32_t batch, steps, P, O;
} orc_req;

/* Philox4x32-10 block (Salmon et al. SC'11). */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* E_q(u) */
uint64_t orc_exp_q32(uint32_t u);
/* length = lo + #{l : cw[l] <= u} */
uint32_t orc_length(const uint32_t* cw, uint32_t ncw, uint32_t lo, uint32_t u);
/* acceptance thresholds T_1..T_gamma; returns alpha_eff */
uint32_t orc_thresholds(uint32_t accept_q16, uint32_t width, uint32_t gamma, uint64_t* T);
/* batch noise factor f (ppm) from a word's four bytes */
uint32_t orc_noise_factor(uint32_t w, uint32_t step_ppm);
/* FNV-1a-32 over the 32 knob bytes */
uint32_t orc_fnv1a_knobs(const orc_knobs* k);
/* 1 if the knob record is valid */
int orc_knobs_valid(const orc_knobs* k, uint32_t n_wl);

/* Per-request draws of the Philox mode: a_i, P_i, O_i, w3_i for i < n (arrays of length n). */
int orc_request_draws(const orc_workload* wl, const orc_knobs* k, uint64_t seed, uint32_t crn,
                      uint32_t n, uint64_t* a, uint32_t* P, uint32_t* O, uint32_t* w3);

/* The first n bursty phases (kinds 1, 2) of a replica: start instant, duration D_p,
 * operational capacity U_p and state.  Returns -1 for other arrival kinds. */
int orc_phases(const orc_workload* wl, const orc_knobs* k, uint64_t seed, uint32_t crn, uint32_t n,
               uint64_t* start, uint64_t* D, uint64_t* U, uint32_t* state);

/* Full replica in Philox mode. latencies[N] (stored u32), trace[N], counters nullable.
 * Returns 0, or <0 on an argument error (invalid knobs are not an error: flags bit 0). */
int orc_run(const orc_workload* wl, uint32_t n_wl, const orc_knobs* k, uint64_t seed, uint32_t crn,
            uint32_t segment_len, uint32_t warmup_len, uint32_t slo_us,
            orc_result* res, uint32_t* latencies, orc_req* trace, orc_counters* cnt);

/* DESIGN.md §2.14 segment stop rule: at least n_min measured completions and t_min_us since t0 (0, 0 = off). */
typedef struct {
  uint32_t n_min, t_min_us;
} orc_stop;

int orc_run_stop(const orc_workload* wl, uint32_t n_wl, const orc_knobs* k, uint64_t seed, uint32_t crn,
                 uint32_t segment_len, uint32_t warmup_len, uint32_t slo_us, uint32_t stop_n_min,
                 uint32_t stop_t_min_us, orc_result* res, uint32_t* latencies, orc_req* trace, orc_counters* cnt);

/* Trace mode: explicit arrivals a[n], lengths P[n], O[n], per-request noise factor f[n] (ppm, used when
 * the request heads a batch / a prefill), and per-request accepted-prefix draws A_val[A_off[i] + j] for
 * decode step j of request i (A_off has n+1 entries).  gamma_eff is given directly.  With `continuous`
 * the decode iterations carry no noise (f_it = 10^6). */
int orc_run_trace(const orc_timing* tm, uint32_t conc, uint32_t max_num_seqs, uint32_t gamma_eff,
                  uint32_t max_wait_us, uint32_t issue_origin, uint32_t continuous, uint32_t n,
                  const uint64_t* a, const uint32_t* P,
                  const uint32_t* O, const uint32_t* f, const uint32_t* A_off, const uint32_t* A_val,
                  uint32_t warmup_len, uint32_t slo_us,
                  orc_result* res, uint32_t* latencies, orc_req* trace, orc_counters* cnt);

/* ... with a draft width W (>= 1) in the speculative step cost (R28) and a stop rule (§2.14) */
int orc_run_trace_stop(const orc_timing* tm, uint32_t conc, uint32_t max_num_seqs, uint32_t gamma_eff,
                       uint32_t draft_width, uint32_t max_wait_us, uint32_t issue_origin, uint32_t continuous, uint32_t n,
                       const uint64_t* a, const uint32_t* P, const uint32_t* O, const uint32_t* f,
                       const uint32_t* A_off, const uint32_t* A_val, uint32_t warmup_len, uint32_t slo_us,
                       uint32_t stop_n_min, uint32_t stop_t_min_us, orc_result* res, uint32_t* latencies,
                       orc_req* trace, orc_counters* cnt);

#ifdef __cplusplus
}
#endif
#endif
