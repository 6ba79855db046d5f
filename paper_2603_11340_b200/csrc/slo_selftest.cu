// slo_selftest.cu — K6: exhaustive self-test of the integer transforms K1/K1c use (SURVEY §8(c) pins table).
//
// Every 2^32 input of E_q, a length table's lookup (§2.4), the acceptance prefix A(u) (§2.5)
// (both guides: K1 / K1c's byte guide and K1g's two-level guide) and the noise factor (§2.4) is evaluated with the SAME device functions the simulation kernels call
// (slo_device.cuh), and reduced to order-free block hashes / histograms that tests compare with the oracle
// (E_q) or with exact closed forms (lengths: #{u -> l} = cw[l] - cw[l-1]; acceptance: #{u : A(u) >= a} = T_a;
// noise: the 4-fold byte convolution).  One CUDA block per 2^20 inputs (4096 blocks), 256 threads, each thread
// a contiguous run of 4096 inputs so monotonicity is checked against the previous input.
#include <cstdint>

#include "slo_device.cuh"
#include "slo_internal.h"

namespace slo {

__device__ __forceinline__ uint64_t selftest_mix(uint32_t u, uint64_t v) {   // test hash (restated in tests)
  return (v ^ ((uint64_t)u * 0x9E3779B97F4A7C15ull)) * 0xBF58476D1CE4E5B9ull;
}

__global__ void __launch_bounds__(256) slo_selftest_kernel(SelftestArgs a, const uint32_t* __restrict__ tables,
                                                           uint64_t* __restrict__ out) {
  extern __shared__ __align__(16) uint32_t sh[];        // histogram bins (what 1-3)
  __shared__ uint32_t tm1[16];
  __shared__ uint8_t guide[256];
  __shared__ uint8_t guide2[kGuideFine];
  __shared__ unsigned long long s_hash, s_viol;
  const uint32_t nb = a.nbins;
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
  if (threadIdx.x == 0) {
    s_hash = 0;
    s_viol = 0;
  }
  uint32_t gp = 0;
  if (a.what == 2 || a.what == 4) {
    gp = accept_thresholds(a.arg0, a.arg1, a.arg2, tm1, threadIdx.x == 0);
    __syncthreads();
    if (a.what == 2) accept_guide(tm1, gp, guide, threadIdx.x, blockDim.x);
    else accept_guide_fine(tm1, gp, guide2, threadIdx.x, blockDim.x);
    __syncthreads();
    if (a.what == 4) accept_guide_fine_mark(tm1, gp, guide2, threadIdx.x);
  }
  __syncthreads();

  const uint32_t u0 = (blockIdx.x << 20) + threadIdx.x * 4096u;
  auto value = [&](uint32_t u) -> uint64_t {
    switch (a.what) {
      case 0: return exp_q32(u);
      case 1: return length_guided(tables, a.off, a.goff, a.lo, u) - a.lo;
      case 2: return accepted_guided(guide, tm1, u, gp);
      case 4: return accepted_fine(guide2[u >> 20], tm1, u, gp);
      default: return noise_factor(u, a.arg0);
    }
  };
  uint64_t prev = u0 == 0 ? 0 : value(u0 - 1u);
  uint64_t h = 0, viol = 0;
  for (uint32_t k = 0; k < 4096u; ++k) {
    const uint32_t u = u0 + k;
    const uint64_t v = value(u);
    if (a.what == 0) {
      h += selftest_mix(u, v);
      viol += (u > 0 && v > prev);                     // E_q increase (R27: expected, counted)
    } else if (a.what == 1 || a.what == 2 || a.what == 4) {
      if (v < nb) atomicAdd(&sh[v], 1u);
      else ++viol;                                     // out of range
      // lengths must be non-decreasing in u, A non-increasing
      viol += (u > 0 && (a.what == 1 ? v < prev : v > prev));
    } else {
      const int64_t d = (int64_t)v - (int64_t)(1000000 - 510 * (int64_t)a.arg0);
      const bool on = a.arg0 == 0 ? v == 1000000u : (d >= 0 && d % a.arg0 == 0 && d / a.arg0 <= 1020);
      if (on) atomicAdd(&sh[a.arg0 == 0 ? 510 : (uint32_t)(d / a.arg0)], 1u);
      else ++viol;
    }
    prev = v;
  }
  if (h) atomicAdd(&s_hash, (unsigned long long)h);
  if (viol) atomicAdd(&s_viol, (unsigned long long)viol);
  __syncthreads();
  if (a.what == 0) {
    if (threadIdx.x == 0) {
      out[blockIdx.x] = s_hash;
      if (s_viol) atomicAdd((unsigned long long*)&out[4096], s_viol);
    }
  } else {
    for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x)
      if (sh[i]) atomicAdd((unsigned long long*)&out[i], (unsigned long long)sh[i]);
    if (threadIdx.x == 0 && s_viol) atomicAdd((unsigned long long*)&out[a.viol_slot], s_viol);
  }
}

}  // namespace slo
