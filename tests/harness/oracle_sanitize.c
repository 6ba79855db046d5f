/* tests/harness/oracle_sanitize.c — TEST INFRASTRUCTURE (ASan/UBSan on the oracle).  A standalone
 * driver compiled together with oracle/slo_oracle.c under -fsanitize=address,undefined: it runs the oracle over
 * every arrival kind (Poisson, MMPP-2, on/off, closed loop, think time), both batching modes, speculation on and
 * off, warmup and the stop rule, and prints one checksum line.  Any out-of-bounds access, use of uninitialised
 * stack or undefined integer behaviour aborts with the sanitizer's report.  It holds none of the method's
 * arithmetic: it only calls the oracle. */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../oracle/slo_oracle.h"

int main(void) {
  /* a small output-length table (cut points, Q32) and a point-mass prompt */
  static const uint32_t out_cw[] = {400000000u, 1200000000u, 2500000000u, 3600000000u, 4100000000u};
  orc_workload wl[10];
  memset(wl, 0, sizeof wl);
  const uint64_t gap = 100000ull << 16, NOA = ~0ull;
  for (int w = 0; w < 10; ++w) {
    orc_workload* x = &wl[w];
    x->prompt_cw = NULL; x->prompt_lo = 40; x->prompt_ncw = 0;
    x->output_cw = out_cw; x->output_lo = 8; x->output_ncw = 5;
    x->timing = (orc_timing){2000, 60, 7000, 200, 1500, 50, 8000, 300, 20, w % 3 ? 338u : 0u};
    x->stream_id = (uint32_t)w;
    x->batching = (uint32_t)(w >= 5);
    const uint32_t kind = (uint32_t)(w % 5);
    x->arr.kind = kind;
    x->arr.mean_gap_q16[0] = gap;
    x->arr.mean_gap_q16[1] = kind == 1 ? gap / 5 : (kind == 2 ? NOA : gap);
    x->arr.mean_sojourn_us[0] = 2000000; x->arr.mean_sojourn_us[1] = 1000000;
    if (kind == 4) x->arr.mean_gap_q16[0] = 30000ull << 16;   /* think time */
  }
  uint64_t check = 0;
  int runs = 0;
  for (int w = 0; w < 10; ++w)
    for (int v = 0; v < 6; ++v) {
      orc_knobs k;
      memset(&k, 0, sizeof k);
      k.conc = (uint8_t)(1 + (v * 7 + w) % 16); k.max_num_seqs = (uint8_t)(1 + (v * 5 + 3 * w) % 12);
      k.draft_len = (uint8_t)(v % 3 ? 4 * (v % 3) : 0); k.spec_on = k.draft_len > 0; k.draft_width = (uint8_t)(1 + v % 2);
      k.workload = (uint8_t)w; k.rate_scale_q8 = (uint16_t)(256 + 64 * v); k.accept_q16 = 32768u + 4000u * (uint32_t)v;
      k.max_wait_us = v == 4 ? 20000u : 0u;
      uint32_t lat[400];
      orc_result res;
      orc_counters cnt;
      const uint32_t warm = v % 2 ? 17u : 0u, seg = 400u - warm;
      int rc = orc_run(wl, 10, &k, 0x5EED0000ull + (uint64_t)(w * 16 + v), 1, seg, warm, 1200000u, &res, lat, NULL, &cnt);
      if (rc) { printf("orc_run rc=%d (w=%d v=%d)\n", rc, w, v); return 1; }
      for (uint32_t i = 0; i < seg + warm; ++i) check = check * 1315423911ull + lat[i];
      check ^= res.p99_us ^ res.slo_met ^ cnt.philox_blocks;
      rc = orc_run_stop(wl, 10, &k, 0xABCDull + (uint64_t)v, 1, seg, warm, 1200000u, 50u, 3000000u, &res, lat, NULL,
                        &cnt);
      if (rc) { printf("orc_run_stop rc=%d (w=%d v=%d)\n", rc, w, v); return 1; }
      check ^= (uint64_t)res.n_measured << 17;
      runs += 2;
    }
  printf("oracle sanitize ok: %d runs, checksum %016llx\n", runs, (unsigned long long)check);
  return 0;
}
