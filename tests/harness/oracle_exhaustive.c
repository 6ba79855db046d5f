/* tests/harness/oracle_exhaustive.c — TEST INFRASTRUCTURE: exhaustive sweeps of the oracle's integer
 * transforms over all 2^32 inputs (SURVEY §8(c) pins table), linked against oracle/libslo_oracle.so.
 * It holds none of the method's arithmetic: it only calls the oracle and counts / hashes what it returns.
 *
 *   exp_scan   : per 2^20-input block, an order-free hash of E_q(u) — the golden values the
 *                device's exhaustive test compares against; also E_q's monotonicity violations and its
 *                largest deviation from -ln((u+1)/2^32) computed by libm in double.
 *   noise_scan : the histogram of the noise factor f(w) over every word w, on the lattice
 *                10^6 + (k - 510) step, k = 0..1020, plus the number of off-lattice values and the exact sum. */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "../../oracle/slo_oracle.h"

/* order-free per-input mix for the block hashes (test hash; the device test restates it) */
static inline uint64_t mix(uint32_t u, uint64_t v) {
  return (v ^ ((uint64_t)u * 0x9E3779B97F4A7C15ull)) * 0xBF58476D1CE4E5B9ull;
}

void exp_scan(uint64_t* block_hash /* [4096] */, uint64_t* nonmono, double* maxerr) {
  uint64_t nm = 0;
  double me = 0.0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : nm) reduction(max : me)
  for (int b = 0; b < 4096; ++b) {
    uint64_t h = 0;
    uint32_t u0 = (uint32_t)b << 20;
    uint64_t prev = u0 == 0 ? UINT64_MAX : orc_exp_q32(u0 - 1u);
    for (uint32_t k = 0; k < (1u << 20); ++k) {
      const uint32_t u = u0 + k;
      const uint64_t v = orc_exp_q32(u);
      h += mix(u, v);
      nm += v > prev;
      prev = v;
      const double ex = -log(((double)u + 1.0) * 0x1p-32);
      const double e = fabs((double)v * 0x1p-32 - ex);
      if (e > me) me = e;
    }
    block_hash[b] = h;
  }
  *nonmono = nm;
  *maxerr = me;
}

void noise_scan(uint32_t step_ppm, uint64_t* counts /* [1021] */, uint64_t* off_lattice, uint64_t* sum_lo,
                uint64_t* sum_hi) {
  memset(counts, 0, 1021 * sizeof(uint64_t));
  uint64_t off = 0;
  unsigned __int128 sum = 0;
  const int64_t base = 1000000 - 510 * (int64_t)step_ppm;
#pragma omp parallel
  {
    uint64_t loc[1021];
    memset(loc, 0, sizeof(loc));
    uint64_t loff = 0;
    unsigned __int128 lsum = 0;
#pragma omp for schedule(static)
    for (int64_t hi = 0; hi < 65536; ++hi) {
      for (uint32_t lo = 0; lo < 65536; ++lo) {
        const uint32_t w = ((uint32_t)hi << 16) | lo;
        const int64_t f = (int64_t)orc_noise_factor(w, step_ppm);
        lsum += (unsigned __int128)f;
        const int64_t d = f - base;
        if (step_ppm == 0 ? f != 1000000 : (d < 0 || d % step_ppm != 0 || d / step_ppm > 1020)) {
          ++loff;
        } else {
          ++loc[step_ppm == 0 ? 510 : d / step_ppm];
        }
      }
    }
#pragma omp critical
    {
      for (int k = 0; k < 1021; ++k) counts[k] += loc[k];
      off += loff;
      sum += lsum;
    }
  }
  *off_lattice = off;
  *sum_lo = (uint64_t)sum;
  *sum_hi = (uint64_t)(sum >> 64);
}
