/* examples/c_api_demo.c — the C-ABI of libslosim.so used from plain C (no Python, no torch).
 *
 * Simulates BASELINE config C1 shaped replicas (C = 8, B = 16, Poisson 10 req/s, 2,000 requests) plus a
 * speculative knob record, 4 seeds each, with an integer-only workload: prompt = 40 tokens, output uniform on
 * [1, 64] (cut points l * 2^32 / 64), LL timing.  Prints one line per replica:
 *   replica p99_us goodput(%.17g) slo_met window_us
 * Build: gcc -O2 -I include examples/c_api_demo.c -L paper_2603_11340_b200 -lslosim \
 *            -Wl,-rpath,$PWD/paper_2603_11340_b200 -o c_api_demo      (libslosim.so carries the CUDA runtime)
 */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "slo_sim.h"

#define CHECK(x)                                                                             \
  do {                                                                                       \
    slo_status s_ = (x);                                                                     \
    if (s_ != SLO_OK) {                                                                      \
      fprintf(stderr, "%s: %s (%s)\n", #x, slo_status_string(s_), slo_last_error(NULL));     \
      return 1;                                                                              \
    }                                                                                        \
  } while (0)

int main(void) {
  uint32_t out_cw[63];
  for (uint32_t l = 1; l < 64; ++l) out_cw[l - 1] = (uint32_t)(((uint64_t)l << 32) / 64u);
  slo_workload wl;
  memset(&wl, 0, sizeof wl);
  wl.arr.kind = 0;                                   /* Poisson, mean gap 100,000 us in Q48.16 */
  wl.arr.mean_gap_q16[0] = wl.arr.mean_gap_q16[1] = 100000ull << 16;
  wl.prompt_cw = NULL;                               /* point mass: P = prompt_lo */
  wl.prompt_lo = 40;
  wl.prompt_ncw = 0;
  wl.output_cw = out_cw;
  wl.output_lo = 1;
  wl.output_ncw = 63;
  slo_timing t = {2000, 60, 7000, 200, 1500, 50, 8000, 300, 20, 338};
  wl.timing = t;
  wl.stream_id = 0;
  wl.batching = 0;

  slo_sim* h = NULL;
  CHECK(slo_sim_create(0, &wl, 1, NULL, &h));

  slo_knobs k[2];
  memset(k, 0, sizeof k);
  k[0].conc = 8; k[0].max_num_seqs = 16; k[0].draft_width = 1; k[0].rate_scale_q8 = 256; k[0].accept_q16 = 32768;
  k[1] = k[0];
  k[1].max_num_seqs = 8; k[1].draft_len = 8; k[1].spec_on = 1;
  uint64_t seeds[4] = {1, 2, 3, 0x5EED0000ull};
  const uint32_t R = 2 * 4, N = 2000, slo = 1200000;

  uint32_t p99[8];
  double gp[8];
  slo_replica_result det[8];
  slo_stats st;
  /* the host entry point: copies in, K0/K1/K1b on the stream, copies out, synchronises */
  CHECK(slo_sim_run_batch_host(h, k, 2, seeds, 4, N, 0, slo, p99, gp, det, &st, NULL));
  for (uint32_t r = 0; r < R; ++r)
    printf("%u %u %.17g %u %llu\n", r, p99[r], gp[r], det[r].slo_met, (unsigned long long)det[r].window_us);
  printf("requests %llu batches %llu philox_blocks %llu\n", (unsigned long long)st.requests,
         (unsigned long long)st.batches, (unsigned long long)st.philox_blocks);
  CHECK(slo_sim_destroy(h));
  return 0;
}
