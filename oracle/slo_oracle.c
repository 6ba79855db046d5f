/* oracle/slo_oracle.c — TEST INFRASTRUCTURE ONLY (see slo_oracle.h).
 *
 * A plain, slow, obviously-correct single-threaded discrete-event simulator of the SLO-Tuner serving
 * model, written step by step from DESIGN.md §2 in the paper's order:
 *   arrivals -> FCFS queue -> idle server forms a batch of up to B requests,
 *   optionally waiting up to max_wait -> prefill driven by the longest prompt ->
 *   decode depending on the number of active sequences and on speculation ->
 *   per-request latencies -> p99 and goodput (Eq. 1).
 * It walks every event instant and every decode step explicitly (no event skipping, no closed forms),
 * recomputes a full Philox block for every word it needs, sorts to get the percentile, and uses 128-bit
 * intermediates for every product.
 */
#include "slo_oracle.h"

#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define ORC_MAX_N (1u << 22)
#define U32MAX 0xFFFFFFFFu
#define U64MAX 0xFFFFFFFFFFFFFFFFull

/* ---------------------------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11, "Parallel random numbers: as  */
/* easy as 1, 2, 3"): round = two 32x32->64 multiplies and xors; key bumped by the Weyl constants.   */
/* ---------------------------------------------------------------------------------------------- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)x0;
    uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)x2;
    uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
    uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
    uint32_t y0 = hi1 ^ x1 ^ k0;
    uint32_t y1 = lo1;
    uint32_t y2 = hi0 ^ x3 ^ k1;
    uint32_t y3 = lo0;
    x0 = y0; x1 = y1; x2 = y2; x3 = y3;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

static void block(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t out[4]) {
  uint32_t ctr[4] = {c0, c1, c2, 0};
  uint32_t key[2] = {k0, k1};
  orc_philox4x32_10(ctr, key, out);
}

/* ---------------------------------------------------------------------------------------------- */
/* E_q(u) ~ 2^32 * (-ln((u+1)/2^32)), integer only.                                */
/* ---------------------------------------------------------------------------------------------- */
static const int64_t LOG2_POLY[11] = {0,          3098163621LL, -1549061789LL, 1032354281LL,
                                      -771198690LL, 601767258LL, -455160697LL, 300247864LL,
                                      -151331885LL, 49215561LL,  -7511879LL};

uint64_t orc_exp_q32(uint32_t u) {
  uint64_t x = (uint64_t)u + 1u;
  if (x == (1ull << 32)) return 0;
  int e = 0; /* floor(log2 x): position of the leading one, found by a plain scan */
  for (int bit = 31; bit >= 0; --bit) {
    if (x & (1ull << bit)) { e = bit; break; }
  }
  uint64_t m = x << (31 - e);                 /* [2^31, 2^32) */
  int64_t t = (int64_t)(m - (1ull << 31));    /* Q0.31 */
  int64_t acc = LOG2_POLY[10];
  for (int k = 9; k >= 0; --k) {
    int64_t prod;
    if (__builtin_mul_overflow(acc, t, &prod)) abort(); /* cannot happen (pinned by tests) */
    acc = LOG2_POLY[k] + (prod >> 31);        /* arithmetic shift = floor division by 2^31 */
  }
  uint64_t y = ((uint64_t)(32 - e) << 31) - (uint64_t)acc;
  return (uint64_t)(((u128)y * (u128)2977044472u) >> 31);
}

/* lengths by counting cut points (the definition, no search). */
uint32_t orc_length(const uint32_t* cw, uint32_t ncw, uint32_t lo, uint32_t u) {
  uint32_t count = 0;
  for (uint32_t l = 0; l < ncw; ++l)
    if (cw[l] <= u) ++count;
  return lo + count;
}

/* alpha_eff = 1 - (1 - alpha)^W in Q16 with floors; T_a = floor(T_{a-1} alpha_eff / 2^16). */
uint32_t orc_thresholds(uint32_t accept_q16, uint32_t width, uint32_t gamma, uint64_t* T) {
  uint64_t r = 65536;
  for (uint32_t w = 0; w < width; ++w) r = (r * (65536u - accept_q16)) / 65536u;
  uint32_t alpha_eff = (uint32_t)(65536u - r);
  uint64_t prev = 1ull << 32;
  for (uint32_t a = 1; a <= gamma; ++a) {
    T[a - 1] = (prev * alpha_eff) / 65536u;
    prev = T[a - 1];
  }
  return alpha_eff;
}

static uint32_t accepted_prefix(uint32_t u, const uint64_t* T, uint32_t gamma) {
  uint32_t A = 0;
  for (uint32_t a = 1; a <= gamma; ++a)
    if ((uint64_t)u < T[a - 1]) ++A;
  return A;
}

/* batch noise factor ("light noise"): f = 10^6 + (b0+b1+b2+b3 - 510) * step_ppm from
 * the four bytes of a word (the head's w3, or an ITER word under continuous batching). */
uint32_t orc_noise_factor(uint32_t w, uint32_t step_ppm) {
  int64_t bytesum = (int64_t)(w & 0xFF) + (int64_t)((w >> 8) & 0xFF) + (int64_t)((w >> 16) & 0xFF) + (int64_t)(w >> 24);
  return (uint32_t)(1000000 + (bytesum - 510) * (int64_t)step_ppm);
}

/* knob record bytes (little-endian), FNV-1a-32. */
static void knob_bytes(const orc_knobs* k, uint8_t b[32]) {
  memset(b, 0, 32);
  b[0] = k->conc; b[1] = k->max_num_seqs; b[2] = k->draft_len; b[3] = k->spec_on;
  b[4] = k->draft_width; b[5] = k->workload;
  b[6] = (uint8_t)(k->rate_scale_q8 & 0xFF); b[7] = (uint8_t)(k->rate_scale_q8 >> 8);
  for (int i = 0; i < 4; ++i) b[8 + i] = (uint8_t)(k->accept_q16 >> (8 * i));
  for (int i = 0; i < 4; ++i) b[12 + i] = (uint8_t)(k->max_wait_us >> (8 * i));
  for (int w = 0; w < 4; ++w)
    for (int i = 0; i < 4; ++i) b[16 + 4 * w + i] = (uint8_t)(k->reserved[w] >> (8 * i));
}

uint32_t orc_fnv1a_knobs(const orc_knobs* k) {
  uint8_t b[32];
  knob_bytes(k, b);
  uint32_t h = 2166136261u;
  for (int i = 0; i < 32; ++i) {
    h ^= b[i];
    h *= 16777619u;
  }
  return h;
}

/* DESIGN.md §3 */
int orc_knobs_valid(const orc_knobs* k, uint32_t n_wl) {
  if (k->conc < 1 || k->conc > 32) return 0;
  if (k->max_num_seqs < 1 || k->max_num_seqs > 32) return 0;
  if (k->draft_len > 16) return 0;
  if (k->spec_on > 1) return 0;
  if (k->draft_width < 1 || k->draft_width > 4) return 0;
  if (k->workload >= n_wl) return 0;
  if (k->rate_scale_q8 < 1) return 0;
  if (k->accept_q16 > 65536u) return 0;
  if (k->max_wait_us > 50000u) return 0;
  for (int i = 0; i < 4; ++i)
    if (k->reserved[i] != 0) return 0;
  return 1;
}

static uint64_t scaled_gap(uint64_t mean_gap_q16, uint32_t rate_scale_q8) {
  if (mean_gap_q16 == U64MAX) return U64MAX;
  return (uint64_t)(((u128)mean_gap_q16 * 256u) / rate_scale_q8);
}

/* operational capacity of a phase: U = min(2^62, floor(D * rho / 2^16)) */
static uint64_t capacity(uint64_t D, uint64_t rho) {
  u128 x = ((u128)D * (u128)rho) >> 16;
  return x > ((u128)1 << 62) ? (1ull << 62) : (uint64_t)x;
}

/* ---------------------------------------------------------------------------------------------- */
/* bursty phases (kinds 1, 2): phase p is in state (start_state + p) mod 2, lasts D_p    */
/* (an exponential sojourn from PHASE block p for kind 1, the fixed sojourn for kind 2) and holds U_p     */
/* operational-time units (its expected arrival count D_p / g_s in Q32 units, reading R26).              */
/* ---------------------------------------------------------------------------------------------- */
typedef struct {
  uint32_t p, state;
  uint64_t start, D, U, Lambda;   /* start instant, duration, operational capacity, operational start */
} phase_t;

static void phase_setup(phase_t* ph, const orc_workload* W, uint32_t k0, uint32_t k1, const uint64_t rho[2]) {
  ph->state = (W->arr.start_state + ph->p) & 1u;
  if (W->arr.kind == 1) {
    uint32_t w[4];
    block(k0, k1, ph->p, 2, 0, w);
    ph->D = (uint64_t)(((u128)orc_exp_q32(w[0]) * W->arr.mean_sojourn_us[ph->state]) >> 32);
  } else {
    ph->D = W->arr.mean_sojourn_us[ph->state];
  }
  ph->U = capacity(ph->D, rho[ph->state]);
}

static void phase_first(phase_t* ph, const orc_workload* W, uint32_t k0, uint32_t k1, const uint64_t rho[2]) {
  ph->p = 0;
  ph->start = 0;
  ph->Lambda = 0;
  phase_setup(ph, W, k0, k1, rho);
}

static void phase_next(phase_t* ph, const orc_workload* W, uint32_t k0, uint32_t k1, const uint64_t rho[2]) {
  ph->Lambda += ph->U;
  ph->start += ph->D;
  ph->p += 1;
  phase_setup(ph, W, k0, k1, rho);
}

static void replica_keys(const orc_workload* wl, const orc_knobs* k, uint64_t seed, uint32_t crn, uint32_t* k0,
                         uint32_t* k1, uint64_t g[2], uint64_t rho[2]) {
  const orc_workload* W = &wl[k->workload];
  uint32_t cfgkey = crn ? W->stream_id : orc_fnv1a_knobs(k);
  *k0 = (uint32_t)seed;
  *k1 = (uint32_t)(seed >> 32) ^ cfgkey;
  g[0] = scaled_gap(W->arr.mean_gap_q16[0], k->rate_scale_q8);
  g[1] = scaled_gap(W->arr.mean_gap_q16[1], k->rate_scale_q8);
  /* per-state rate rho_s = floor((2^64 - 1) / g_s), 0 for a state without arrivals;
   * g = 0 only for kind 4, a zero mean think time (rho is used by kinds 1 and 2) */
  rho[0] = g[0] == U64MAX || g[0] == 0 ? 0 : U64MAX / g[0];
  rho[1] = g[1] == U64MAX || g[1] == 0 ? 0 : U64MAX / g[1];
}

int orc_phases(const orc_workload* wl, const orc_knobs* k, uint64_t seed, uint32_t crn, uint32_t n,
               uint64_t* start, uint64_t* D, uint64_t* U, uint32_t* state) {
  const orc_workload* W = &wl[k->workload];
  if (W->arr.kind != 1 && W->arr.kind != 2) return -1;
  uint32_t k0, k1;
  uint64_t g[2], rho[2];
  replica_keys(wl, k, seed, crn, &k0, &k1, g, rho);
  phase_t ph;
  phase_first(&ph, W, k0, k1, rho);
  for (uint32_t q = 0; q < n; ++q) {
    start[q] = ph.start;
    D[q] = ph.D;
    U[q] = ph.U;
    state[q] = ph.state;
    phase_next(&ph, W, k0, k1, rho);
  }
  return 0;
}

/* ---------------------------------------------------------------------------------------------- */
/* request draws a_i, P_i, O_i, w3_i                                         */
/* ---------------------------------------------------------------------------------------------- */
int orc_request_draws(const orc_workload* wl, const orc_knobs* k, uint64_t seed, uint32_t crn,
                      uint32_t n, uint64_t* a, uint32_t* P, uint32_t* O, uint32_t* w3) {
  const orc_workload* W = &wl[k->workload];
  uint32_t k0, k1;
  uint64_t g[2], rho[2];
  replica_keys(wl, k, seed, crn, &k0, &k1, g, rho);
  const uint32_t kind = W->arr.kind;
  phase_t ph = {0, 0, 0, 0, 0, 0};
  if (kind == 1 || kind == 2) phase_first(&ph, W, k0, k1, rho);
  uint64_t prev = 0, tau = 0;
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t w[4];
    block(k0, k1, i, 0, 0, w);
    uint64_t E = orc_exp_q32(w[0]);
    if (kind >= 3) {           /* closed loop (3: zero think time, 4: exponential think time):
                                  a_i = 0; kind 4's issue instants come from the think draws in simulate() */
      a[i] = 0;
    } else if (kind == 0) {
      uint64_t gap = (uint64_t)(((u128)E * g[0]) >> 48);
      a[i] = prev + gap;
      prev = a[i];
    } else {                   /* Cox time change: operational epoch tau_i -> the phase holding it */
      tau += E;
      while (tau >= ph.Lambda + ph.U) phase_next(&ph, W, k0, k1, rho);
      uint64_t off = (uint64_t)(((u128)(tau - ph.Lambda) * g[ph.state]) >> 48);
      if (off > ph.D - 1) off = ph.D - 1;
      a[i] = ph.start + off;
    }
    P[i] = orc_length(W->prompt_cw, W->prompt_ncw, W->prompt_lo, w[1]);
    O[i] = orc_length(W->output_cw, W->output_ncw, W->output_lo, w[2]);
    w3[i] = w[3];
  }
  return (int)((kind == 1 || kind == 2) ? ph.p + 1 : 0); /* phases drawn (kind 1 consumes one block each) */
}

/* ---------------------------------------------------------------------------------------------- */
/* the event loop                                                                 */
/* ---------------------------------------------------------------------------------------------- */
typedef struct {
  int philox;                 /* 1: draws from SPEC blocks; 0: explicit A arrays */
  uint32_t k0, k1;
  const uint64_t* T;
  const uint32_t* A_off;
  const uint32_t* A_val;
  int bad;                    /* trace ran out of A values */
} adraw;

static uint32_t draw_A(adraw* d, uint32_t i, uint32_t j, uint32_t gamma) {
  if (d->philox) {
    uint32_t w[4];
    block(d->k0, d->k1, i, 1, j / 4u, w);
    return accepted_prefix(w[j % 4u], d->T, gamma);
  }
  if (d->A_off[i] + j >= d->A_off[i + 1]) {
    d->bad = 1;
    return 0;
  }
  return d->A_val[d->A_off[i] + j];
}

/* DESIGN.md §2.6 decode step cost with n active sequences; with speculation (R10, factorised per R28,
 * P:98 "draft width W and verifier cadence k", "wider drafts add verifier and compute cost"):
 * W draft branches of gamma tokens each cost gamma*W*(dr_base + dr_seq*n), and the verifier scores the
 * W*gamma drafted tokens plus one per sequence: ver_base + ver_seq*n + ver_tok*(W*gamma + 1)*n.  W = 1 is
 * R10's cost exactly. */
static uint64_t step_cost(const orc_timing* tm, uint32_t gamma, uint32_t width, uint64_t n) {
  if (gamma == 0) return (uint64_t)tm->dec_base_us + (uint64_t)tm->dec_seq_us * n;
  const uint64_t drafted = (uint64_t)gamma * width;
  return drafted * ((uint64_t)tm->dr_base_us + (uint64_t)tm->dr_seq_us * n) +
         (uint64_t)tm->ver_base_us + (uint64_t)tm->ver_seq_us * n +
         (uint64_t)tm->ver_tok_us * (drafted + 1) * n;
}

/* DESIGN.md §2.11 kind 4 — closed loop with exponential think time: the k-th completion (k = 0, 1, ...)
 * starts user chain q = k + C (if q < N), which becomes ready at c + Z_k, Z_k = floor(E_q(w0) * g / 2^48)
 * with w0 from the THINK block (k, 4, 0) and g the scaled mean think time (Q48.16 us). */
typedef struct {
  int on;
  uint32_t k0, k1;
  uint64_t g;
} thinkdraw;

static uint64_t think_time(const thinkdraw* th, uint32_t k) {
  uint32_t w[4];
  block(th->k0, th->k1, k, 4, 0, w);
  return (uint64_t)(((u128)orc_exp_q32(w[0]) * th->g) >> 48);
}

static int cmp_u64(const void* x, const void* y) {
  uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
  return (a > b) - (a < b);
}

static int cmp_u32(const void* x, const void* y) {
  uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
  return (a > b) - (a < b);
}

/* DESIGN.md §2.8 (+ §2.14 stop rule) — replica outputs from the completion times c[] of all N requests.
 * Without a stop rule every measured request (i >= warmup) counts.  With one (n_min, t_min), the segment
 * ends at t* = the k-th smallest measured completion time for the smallest k >= max(n_min, 1) with
 * c_(k) - t0 >= t_min (t0 = origin of request `warmup`); only requests with c <= t* count and every request
 * completing after t* stores the sentinel latency U32MAX; if no k qualifies, every measured request counts
 * and flags bit 2 is set (the source ran out first). */
static void outputs(uint32_t N, uint32_t warmup, uint32_t slo_us, const uint64_t* c, const uint64_t* origin,
                    const orc_stop* stop, orc_result* res, uint32_t* lat) {
  const uint32_t nm = N - warmup;
  const uint64_t t0 = origin[warmup];
  uint64_t tstar = U64MAX;
  uint32_t flags = 0;
  if (stop && (stop->n_min || stop->t_min_us)) {
    uint64_t* cm = (uint64_t*)malloc((size_t)nm * sizeof(uint64_t));
    if (!cm) abort();
    memcpy(cm, c + warmup, (size_t)nm * sizeof(uint64_t));
    qsort(cm, nm, sizeof(uint64_t), cmp_u64);
    const uint32_t need = stop->n_min > 0 ? stop->n_min : 1u;
    int found = 0;
    for (uint32_t k = need; k <= nm; ++k) {
      if (cm[k - 1] >= t0 + stop->t_min_us) {
        tstar = cm[k - 1];
        found = 1;
        break;
      }
    }
    if (!found) flags |= 4u;
    free(cm);
  }
  uint32_t n = 0, slo_met = 0;
  uint64_t sum = 0, cmax = 0;
  uint32_t* sorted = (uint32_t*)malloc((size_t)nm * sizeof(uint32_t));
  if (!sorted) abort();
  for (uint32_t i = 0; i < N; ++i) {
    const uint64_t l = c[i] - origin[i];
    const int inc = c[i] <= tstar;
    lat[i] = !inc ? U32MAX : (l > U32MAX ? U32MAX : (uint32_t)l);
    if (i >= warmup && inc) {
      if (l > U32MAX) flags |= 2u;
      if (l <= slo_us) ++slo_met;
      sum += l;
      if (c[i] > cmax) cmax = c[i];
      sorted[n++] = lat[i];
    }
  }
  qsort(sorted, n, sizeof(uint32_t), cmp_u32);
  res->p99_us = sorted[(uint32_t)((99ull * n + 99ull) / 100ull) - 1]; /* nearest rank, ceil(0.99 n) */
  res->p50_us = sorted[(uint32_t)((50ull * n + 99ull) / 100ull) - 1]; /* ceil(0.50 n) */
  res->p95_us = sorted[(uint32_t)((95ull * n + 99ull) / 100ull) - 1]; /* ceil(0.95 n) */
  res->slo_met = slo_met;
  res->n_measured = n;
  res->flags = flags;
  const uint64_t T = cmax - t0;
  res->window_us = T < 1 ? 1 : T;
  res->sum_latency_us = sum;
  res->goodput = (double)((uint64_t)slo_met * 1000000ull) / (double)res->window_us;
  free(sorted);
}

static int simulate(const orc_timing* tm, uint32_t C, uint32_t B, uint32_t gamma, uint32_t width, uint32_t mw,
                    uint32_t issue_origin,
                    uint32_t N, const uint64_t* a, const uint32_t* P, const uint32_t* O,
                    const uint32_t* f, adraw* ad, const thinkdraw* th, uint32_t warmup, uint32_t slo_us,
                    const orc_stop* stop, orc_result* res, uint32_t* latencies, orc_req* trace, orc_counters* cnt) {
  uint64_t* s = (uint64_t*)calloc(N, sizeof(uint64_t));
  uint64_t* form = (uint64_t*)calloc(N, sizeof(uint64_t));
  uint64_t* c = (uint64_t*)calloc(N, sizeof(uint64_t));
  uint32_t* steps = (uint32_t*)calloc(N, sizeof(uint32_t));
  uint32_t* batch_of = (uint32_t*)calloc(N, sizeof(uint32_t));
  uint32_t* pend = (uint32_t*)calloc(B, sizeof(uint32_t));
  uint32_t* rem = (uint32_t*)calloc(B, sizeof(uint32_t));
  uint32_t* lat = (uint32_t*)calloc(N, sizeof(uint32_t));
  /* kind 4: ordinal of each request's completion, and the ready user chains (ready time, chain id) */
  uint32_t* kord = (uint32_t*)calloc(N, sizeof(uint32_t));
  uint64_t* rdy_t = (uint64_t*)calloc(C, sizeof(uint64_t));
  uint32_t* rdy_q = (uint32_t*)calloc(C, sizeof(uint32_t));
  uint32_t* order = (uint32_t*)calloc(B, sizeof(uint32_t));
  if (!s || !form || !c || !steps || !batch_of || !pend || !rem || !lat || !kord || !rdy_t || !rdy_q || !order) abort();

  uint32_t na = 0, ni = 0, nb = 0, inflight = 0, ndone = 0, npend = 0, nbatches = 0, nrdy = 0, nord = 0;
  int busy = 0;
  uint64_t decode_steps = 0, member_steps = 0, spec_blocks = 0, think_blocks = 0;
  if (th->on) /* the first C chains are ready at t = 0 */
    for (uint32_t q = 0; q < C && q < N; ++q) {
      rdy_t[nrdy] = 0;
      rdy_q[nrdy++] = q;
    }

  while (ndone < N) {
    /* next event instant: an arrival (kind 4: a chain's think ends), a completion, or a max_wait deadline of
     * an idle server */
    uint64_t t = U64MAX;
    if (!th->on && na < N && a[na] < t) t = a[na];
    for (uint32_t q = 0; q < nrdy; ++q)
      if (rdy_t[q] < t) t = rdy_t[q];
    for (uint32_t q = 0; q < npend; ++q)
      if (c[pend[q]] < t) t = c[pend[q]];
    if (!busy && nb < ni && mw > 0 && s[nb] + mw < t) t = s[nb] + mw;
    if (t == U64MAX) abort(); /* no event can happen: impossible for a valid model */

    /* (1) completions at t */
    for (uint32_t q = 0; q < npend;) {
      if (c[pend[q]] == t) {
        --inflight;
        ++ndone;
        if (th->on && kord[pend[q]] + C < N) { /* kind 4: the user thinks, then chain k + C is ready */
          rdy_t[nrdy] = t + think_time(th, kord[pend[q]]);
          rdy_q[nrdy++] = kord[pend[q]] + C;
          ++think_blocks;
        }
        pend[q] = pend[npend - 1];
        --npend;
      } else {
        ++q;
      }
    }
    if (busy && npend == 0) busy = 0;
    /* (2) arrivals at t, in index order (kind 4: the chains ready at t, in chain order, arrive and issue at
     * once; request index = issue order) */
    if (th->on) {
      for (;;) {
        uint32_t best = U32MAX;
        for (uint32_t q = 0; q < nrdy; ++q)
          if (rdy_t[q] == t && (best == U32MAX || rdy_q[q] < rdy_q[best])) best = q;
        if (best == U32MAX) break;
        rdy_t[best] = rdy_t[nrdy - 1];
        rdy_q[best] = rdy_q[nrdy - 1];
        --nrdy;
        ++na;
      }
    } else {
      while (na < N && a[na] == t) ++na;
    }
    /* (3) issues at t, in index order, while fewer than C are in flight */
    while (ni < na && inflight < C) {
      s[ni] = t;
      ++inflight;
      ++ni;
    }
    /* (4) batch formation by an idle server */
    if (!busy && nb < ni) {
      uint32_t q = ni - nb;
      if (mw == 0 || q >= B || t >= s[nb] + mw) {
        uint32_t b = q < B ? q : B;
        uint32_t h = nb;
        uint64_t fh = f[h];
        uint32_t maxP = 0;
        for (uint32_t m = h; m < h + b; ++m)
          if (P[m] > maxP) maxP = P[m];
        uint64_t Dp = (uint64_t)(((u128)fh * ((u128)tm->pre_base_us + (u128)tm->pre_tok_us * maxP)) /
                                 1000000u);
        /* decode, step by step */
        uint32_t active = b;
        for (uint32_t m = 0; m < b; ++m) rem[m] = O[h + m];
        u128 cum = 0;
        uint32_t j = 0;
        while (active > 0) {
          uint64_t n = active;
          cum += step_cost(tm, gamma, width, n);
          for (uint32_t m = 0; m < b; ++m) {
            if (rem[m] == 0) continue;
            uint32_t e = 1;
            if (gamma > 0) {
              uint32_t A = draw_A(ad, h + m, j, gamma);
              e = A + 1 < rem[m] ? A + 1 : rem[m];
            }
            rem[m] -= e;
            steps[h + m] += 1;
            if (rem[m] == 0) {
              c[h + m] = t + Dp + (uint64_t)(((u128)fh * cum) / 1000000u);
              --active;
            }
          }
          ++j;
        }
        decode_steps += j;
        /* completion ordinals (kind 4 think draws): in time order, i.e. by step count, then request index */
        for (uint32_t m = 0; m < b; ++m) order[m] = h + m;
        for (uint32_t x = 1; x < b; ++x)
          for (uint32_t y = x; y > 0 && steps[order[y]] < steps[order[y - 1]]; --y) {
            uint32_t tmp = order[y];
            order[y] = order[y - 1];
            order[y - 1] = tmp;
          }
        for (uint32_t m = 0; m < b; ++m) kord[order[m]] = nord++;
        for (uint32_t m = h; m < h + b; ++m) {
          form[m] = t;
          batch_of[m] = nbatches;
          member_steps += steps[m];
          if (gamma > 0) spec_blocks += (steps[m] + 3u) / 4u;
          pend[npend++] = m;
        }
        ++nbatches;
        nb += b;
        busy = 1;
      }
    }
  }

  /* outputs; latency from arrival (open loop, R2) or from issue (closed loop, §2.11) */
  const uint64_t* origin = issue_origin ? s : a;
  outputs(N, warmup, slo_us, c, origin, stop, res, lat);
  if (latencies) memcpy(latencies, lat, (size_t)N * sizeof(uint32_t));
  if (trace) {
    for (uint32_t i = 0; i < N; ++i) {
      trace[i].a = a[i];
      trace[i].s = s[i];
      trace[i].form = form[i];
      trace[i].c = c[i];
      trace[i].batch = batch_of[i];
      trace[i].steps = steps[i];
      trace[i].P = P[i];
      trace[i].O = O[i];
    }
  }
  if (cnt) {
    cnt->batches = nbatches;
    cnt->decode_steps = decode_steps;
    cnt->member_steps = member_steps;
    cnt->philox_blocks = spec_blocks + think_blocks; /* caller adds REQ and PHASE blocks */
  }
  free(s); free(form); free(c); free(steps); free(batch_of); free(pend); free(rem); free(lat);
  free(kord); free(rdy_t); free(rdy_q); free(order);
  return ad->bad ? -2 : 0;
}

/* ---------------------------------------------------------------------------------------------- */
/* continuous (iteration-level) batching: the same instants and gate, but the server  */
/* runs one prefill or decode iteration at a time over a running set of at most B requests.           */
/* ---------------------------------------------------------------------------------------------- */
typedef struct {
  int philox;                 /* decode-iteration noise from ITER blocks (Philox mode) */
  uint32_t k0, k1, step_ppm;
} itnoise;

static uint64_t iter_noise(const itnoise* nz, uint64_t it) {
  if (!nz->philox || nz->step_ppm == 0) return 1000000u;
  uint32_t w[4];
  block(nz->k0, nz->k1, (uint32_t)it, 3, 0, w);
  return orc_noise_factor(w[0], nz->step_ppm);
}

static int simulate_cont(const orc_timing* tm, uint32_t C, uint32_t B, uint32_t gamma, uint32_t width,
                         uint32_t issue_origin,
                         uint32_t N, const uint64_t* a, const uint32_t* P, const uint32_t* O,
                         const uint32_t* f, adraw* ad, const itnoise* nz, const thinkdraw* th, uint32_t warmup,
                         uint32_t slo_us, const orc_stop* stop, orc_result* res, uint32_t* latencies,
                         orc_req* trace, orc_counters* cnt) {
  uint64_t* s = (uint64_t*)calloc(N, sizeof(uint64_t));
  uint64_t* form = (uint64_t*)calloc(N, sizeof(uint64_t));   /* admission (prefill start) */
  uint64_t* c = (uint64_t*)calloc(N, sizeof(uint64_t));
  uint32_t* steps = (uint32_t*)calloc(N, sizeof(uint32_t));
  uint32_t* batch_of = (uint32_t*)calloc(N, sizeof(uint32_t)); /* prefill iteration that admitted it */
  uint32_t* rem = (uint32_t*)calloc(N, sizeof(uint32_t));
  uint32_t* run = (uint32_t*)calloc(B, sizeof(uint32_t));
  uint32_t* fin = (uint32_t*)calloc(B, sizeof(uint32_t));
  uint32_t* lat = (uint32_t*)calloc(N, sizeof(uint32_t));
  uint64_t* rdy_t = (uint64_t*)calloc(C, sizeof(uint64_t));     /* kind 4: ready user chains */
  uint32_t* rdy_q = (uint32_t*)calloc(C, sizeof(uint32_t));
  if (!s || !form || !c || !steps || !batch_of || !rem || !run || !fin || !lat || !rdy_t || !rdy_q) abort();

  uint32_t nrdy = 0;
  uint64_t think_blocks = 0;
  if (th->on) /* the first C chains are ready at t = 0 */
    for (uint32_t q = 0; q < C && q < N; ++q) {
      rdy_t[nrdy] = 0;
      rdy_q[nrdy++] = q;
    }
  uint32_t na = 0, ni = 0, nq = 0, inflight = 0, ndone = 0, nrun = 0;
  uint32_t join_lo = 0, join_hi = 0;      /* requests being prefilled: they join R at the iteration end */
  uint32_t nfin = 0;                      /* running members finishing at the iteration end */
  int busy = 0;
  uint64_t t = 0, iter_end = 0, it = 0, prefills = 0, decode_iters = 0, member_steps = 0, spec_blocks = 0;

  while (ndone < N) {
    uint64_t tn = U64MAX;
    if (busy) tn = iter_end;
    if (!th->on && na < N && a[na] < tn) tn = a[na];
    for (uint32_t q = 0; q < nrdy; ++q)
      if (rdy_t[q] < tn) tn = rdy_t[q];
    if (tn == U64MAX) abort();
    t = tn;
    /* (1) the iteration ending at t: completions leave, prefilled requests join */
    if (busy && iter_end == t) {
      for (uint32_t q = 0; q < nfin; ++q) { /* fin[] is in admission = request-index order */
        c[fin[q]] = t;
        --inflight;
        if (th->on && ndone + C < N) { /* kind 4: completion ndone starts chain ndone + C after Z_ndone */
          rdy_t[nrdy] = t + think_time(th, ndone);
          rdy_q[nrdy++] = ndone + C;
          ++think_blocks;
        }
        ++ndone;
      }
      uint32_t kept = 0;                              /* drop finished members, keep admission order */
      for (uint32_t q = 0; q < nrun; ++q)
        if (rem[run[q]] != 0) run[kept++] = run[q];
      nrun = kept;
      for (uint32_t m = join_lo; m < join_hi; ++m) run[nrun++] = m;
      nfin = 0;
      join_lo = join_hi = 0;
      busy = 0;
    }
    /* (2) arrivals at t (kind 4: the chains ready at t, in chain order) */
    if (th->on) {
      for (;;) {
        uint32_t best = U32MAX;
        for (uint32_t q = 0; q < nrdy; ++q)
          if (rdy_t[q] == t && (best == U32MAX || rdy_q[q] < rdy_q[best])) best = q;
        if (best == U32MAX) break;
        rdy_t[best] = rdy_t[nrdy - 1];
        rdy_q[best] = rdy_q[nrdy - 1];
        --nrdy;
        ++na;
      }
    } else {
      while (na < N && a[na] == t) ++na;
    }
    /* (3) issues at t while fewer than C are in flight */
    while (ni < na && inflight < C) {
      s[ni] = t;
      ++inflight;
      ++ni;
    }
    /* (4) a free server starts the next iteration */
    if (!busy) {
      if (nrun < B && nq < ni) {                        /* prefill the first k queued requests */
        uint32_t k = ni - nq < B - nrun ? ni - nq : B - nrun;
        uint32_t maxP = 0;
        for (uint32_t m = nq; m < nq + k; ++m) {
          if (P[m] > maxP) maxP = P[m];
          form[m] = t;
          batch_of[m] = (uint32_t)prefills;
          rem[m] = O[m];
        }
        uint64_t D = (uint64_t)(((u128)f[nq] * ((u128)tm->pre_base_us + (u128)tm->pre_tok_us * maxP)) / 1000000u);
        join_lo = nq;
        join_hi = nq + k;
        nq += k;
        ++prefills;
        iter_end = t + D;
        busy = 1;
      } else if (nrun > 0) {                            /* one decode iteration of the running set */
        uint64_t fi = iter_noise(nz, it);
        uint64_t D = (uint64_t)(((u128)fi * step_cost(tm, gamma, width, nrun)) / 1000000u);
        for (uint32_t q = 0; q < nrun; ++q) {
          uint32_t m = run[q];
          uint32_t e = 1;
          if (gamma > 0) {
            uint32_t A = draw_A(ad, m, steps[m], gamma);
            e = A + 1 < rem[m] ? A + 1 : rem[m];
          }
          rem[m] -= e;
          steps[m] += 1;
          if (rem[m] == 0) fin[nfin++] = m;
        }
        ++it;
        ++decode_iters;
        iter_end = t + D;
        busy = 1;
      }
    }
  }
  for (uint32_t m = 0; m < N; ++m) {
    member_steps += steps[m];
    if (gamma > 0) spec_blocks += (steps[m] + 3u) / 4u;
  }

  const uint64_t* origin = issue_origin ? s : a;
  outputs(N, warmup, slo_us, c, origin, stop, res, lat);
  if (latencies) memcpy(latencies, lat, (size_t)N * sizeof(uint32_t));
  if (trace) {
    for (uint32_t i = 0; i < N; ++i) {
      trace[i].a = a[i];
      trace[i].s = s[i];
      trace[i].form = form[i];
      trace[i].c = c[i];
      trace[i].batch = batch_of[i];
      trace[i].steps = steps[i];
      trace[i].P = P[i];
      trace[i].O = O[i];
    }
  }
  if (cnt) {
    cnt->batches = prefills;                 /* continuous mode: prefill iterations */
    cnt->decode_steps = decode_iters;        /* continuous mode: decode iterations */
    cnt->member_steps = member_steps;
    cnt->philox_blocks = spec_blocks + ((nz->philox && nz->step_ppm) ? decode_iters : 0) + think_blocks;
  }
  free(s); free(form); free(c); free(steps); free(batch_of); free(rem); free(run); free(fin); free(lat);
  free(rdy_t); free(rdy_q);
  return ad->bad ? -2 : 0;
}

static void invalid_result(orc_result* res) {
  memset(res, 0, sizeof(*res));
  res->p99_us = U32MAX;
  res->flags = 1u;
  res->goodput = -1.0;
}

int orc_run(const orc_workload* wl, uint32_t n_wl, const orc_knobs* k, uint64_t seed, uint32_t crn,
            uint32_t segment_len, uint32_t warmup_len, uint32_t slo_us,
            orc_result* res, uint32_t* latencies, orc_req* trace, orc_counters* cnt) {
  return orc_run_stop(wl, n_wl, k, seed, crn, segment_len, warmup_len, slo_us, 0, 0, res, latencies, trace, cnt);
}

int orc_run_stop(const orc_workload* wl, uint32_t n_wl, const orc_knobs* k, uint64_t seed, uint32_t crn,
                 uint32_t segment_len, uint32_t warmup_len, uint32_t slo_us, uint32_t stop_n_min,
                 uint32_t stop_t_min_us, orc_result* res, uint32_t* latencies, orc_req* trace, orc_counters* cnt) {
  const orc_stop stop = {stop_n_min, stop_t_min_us};
  if (!wl || !k || !res || segment_len == 0 || n_wl == 0) return -1;
  if ((uint64_t)segment_len + warmup_len > ORC_MAX_N) return -1;
  if (slo_us == U32MAX) return -1;
  if (cnt) memset(cnt, 0, sizeof(*cnt));
  if (!orc_knobs_valid(k, n_wl)) {
    invalid_result(res);
    return 0;
  }
  uint32_t N = segment_len + warmup_len;
  const orc_workload* W = &wl[k->workload];
  uint64_t* a = (uint64_t*)malloc((size_t)N * sizeof(uint64_t));
  uint32_t* P = (uint32_t*)malloc((size_t)N * sizeof(uint32_t));
  uint32_t* O = (uint32_t*)malloc((size_t)N * sizeof(uint32_t));
  uint32_t* w3 = (uint32_t*)malloc((size_t)N * sizeof(uint32_t));
  uint32_t* f = (uint32_t*)malloc((size_t)N * sizeof(uint32_t));
  if (!a || !P || !O || !w3 || !f) abort();
  int phases = orc_request_draws(wl, k, seed, crn, N, a, P, O, w3);
  for (uint32_t i = 0; i < N; ++i) f[i] = orc_noise_factor(w3[i], W->timing.noise_step_ppm); /* §2.4 */
  uint32_t gamma = k->spec_on ? k->draft_len : 0;
  uint64_t T[16];
  orc_thresholds(k->accept_q16, k->draft_width, gamma, T);
  uint32_t cfgkey = crn ? W->stream_id : orc_fnv1a_knobs(k);
  adraw ad = {1, (uint32_t)seed, (uint32_t)(seed >> 32) ^ cfgkey, T, NULL, NULL, 0};
  int rc;
  const int closed = W->arr.kind == 3 || W->arr.kind == 4;
  const thinkdraw th = {W->arr.kind == 4, (uint32_t)seed, (uint32_t)(seed >> 32) ^ cfgkey,
                        scaled_gap(W->arr.mean_gap_q16[0], k->rate_scale_q8)};
  if (th.on && W->arr.mean_gap_q16[0] == U64MAX) { /* kind 4 needs a finite mean think time */
    free(a); free(P); free(O); free(w3); free(f);
    return -1;
  }
  if (W->batching == 1) {
    itnoise nz = {1, (uint32_t)seed, (uint32_t)(seed >> 32) ^ cfgkey, W->timing.noise_step_ppm};
    rc = simulate_cont(&W->timing, k->conc, k->max_num_seqs, gamma, k->draft_width, closed, N, a, P, O, f, &ad, &nz, &th,
                       warmup_len, slo_us, &stop, res, latencies, trace, cnt);
  } else {
    rc = simulate(&W->timing, k->conc, k->max_num_seqs, gamma, k->draft_width, k->max_wait_us, closed, N, a, P, O, f, &ad, &th,
                  warmup_len, slo_us, &stop, res, latencies, trace, cnt);
  }
  if (cnt) cnt->philox_blocks += N + (W->arr.kind == 1 ? (uint64_t)phases : 0);
  free(a); free(P); free(O); free(w3); free(f);
  return rc;
}

int orc_run_trace(const orc_timing* tm, uint32_t conc, uint32_t max_num_seqs, uint32_t gamma_eff,
                  uint32_t max_wait_us, uint32_t issue_origin, uint32_t continuous, uint32_t n,
                  const uint64_t* a, const uint32_t* P,
                  const uint32_t* O, const uint32_t* f, const uint32_t* A_off, const uint32_t* A_val,
                  uint32_t warmup_len, uint32_t slo_us,
                  orc_result* res, uint32_t* latencies, orc_req* trace, orc_counters* cnt) {
  return orc_run_trace_stop(tm, conc, max_num_seqs, gamma_eff, 1, max_wait_us, issue_origin, continuous, n, a, P, O,
                            f, A_off, A_val, warmup_len, slo_us, 0, 0, res, latencies, trace, cnt);
}

int orc_run_trace_stop(const orc_timing* tm, uint32_t conc, uint32_t max_num_seqs, uint32_t gamma_eff,
                       uint32_t draft_width, uint32_t max_wait_us, uint32_t issue_origin, uint32_t continuous, uint32_t n,
                       const uint64_t* a, const uint32_t* P,
                       const uint32_t* O, const uint32_t* f, const uint32_t* A_off, const uint32_t* A_val,
                       uint32_t warmup_len, uint32_t slo_us, uint32_t stop_n_min, uint32_t stop_t_min_us,
                       orc_result* res, uint32_t* latencies, orc_req* trace, orc_counters* cnt) {
  const orc_stop stop = {stop_n_min, stop_t_min_us};
  if (!tm || !a || !P || !O || !f || !res || n == 0 || warmup_len >= n) return -1;
  if (conc < 1 || max_num_seqs < 1 || draft_width < 1) return -1;
  if (gamma_eff > 0 && (!A_off || !A_val)) return -1;
  for (uint32_t i = 1; i < n; ++i)
    if (a[i] < a[i - 1]) return -1;
  for (uint32_t i = 0; i < n; ++i)
    if (O[i] < 1) return -1;
  if (cnt) memset(cnt, 0, sizeof(*cnt));
  adraw ad = {0, 0, 0, NULL, A_off, A_val, 0};
  const thinkdraw th = {0, 0, 0, 0};
  if (continuous) {
    itnoise nz = {0, 0, 0, 0};
    return simulate_cont(tm, conc, max_num_seqs, gamma_eff, draft_width, issue_origin, n, a, P, O, f, &ad, &nz, &th, warmup_len,
                         slo_us, &stop, res, latencies, trace, cnt);
  }
  return simulate(tm, conc, max_num_seqs, gamma_eff, draft_width, max_wait_us, issue_origin, n, a, P, O, f, &ad, &th, warmup_len,
                  slo_us, &stop, res, latencies, trace, cnt);
}
