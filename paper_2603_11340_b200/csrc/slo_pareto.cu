// slo_pareto.cu — K5: the Pareto front of a sweep.
//
// Objectives per config from its aggregate over seeds: mean p99 = floor(sum_p99 / n) (minimise) and
// goodput = floor(sum_slo_met * 10^12 / sum_window) micro-rps (maximise).  The front is found in
// O(n log n) on the device instead of the definition's O(n^2): sort by (p99 ascending, goodput descending)
// with two stable radix sorts; then a point is dominated iff some point of an earlier p99 group has goodput
// >= its own (an exclusive prefix max, read at its group's first position), or the first point of its own
// group has a strictly larger goodput.  Equal points never dominate each other.
#include <cub/cub.cuh>

#include "slo_internal.h"

namespace slo {

__global__ void pareto_objectives_kernel(const slo_config_agg* __restrict__ agg, uint32_t n, uint32_t* __restrict__ p99,
                                         unsigned long long* __restrict__ gp, uint32_t* __restrict__ idx,
                                         uint8_t* __restrict__ valid) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const slo_config_agg a = agg[i];
  const bool ok = a.n_seeds > 0 && !(a.flags & 1u) && a.sum_window_us > 0;
  uint32_t p = 0xFFFFFFFFu;
  unsigned long long g = 0;
  if (ok) {
    p = (uint32_t)(a.sum_p99_us / a.n_seeds);                      // each p99 < 2^32, so the mean is too
    const unsigned __int128 q = ((unsigned __int128)a.sum_slo_met * 1000000000000ull) / a.sum_window_us;
    g = q > (unsigned __int128)~0ull ? ~0ull : (unsigned long long)q;
  }
  p99[i] = p;
  gp[i] = g;
  idx[i] = i;
  valid[i] = ok;
}

template <typename T>
__global__ void gather_kernel(const T* __restrict__ src, const uint32_t* __restrict__ idx, uint32_t n, T* __restrict__ dst) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void group_start_kernel(const uint32_t* __restrict__ p99s, uint32_t n, uint32_t* __restrict__ start) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) start[i] = (i == 0 || p99s[i] != p99s[i - 1]) ? i : 0u;
}

__global__ void pareto_mark_kernel(const unsigned long long* __restrict__ gps, const unsigned long long* __restrict__ exmax,
                                   const uint32_t* __restrict__ gstart, const uint32_t* __restrict__ idxs,
                                   const uint8_t* __restrict__ valid, uint32_t n, uint8_t* __restrict__ front,
                                   uint32_t* __restrict__ count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t g0 = gstart[i];
  const unsigned long long g = gps[i];
  const bool dominated = (g0 > 0 && exmax[g0] >= g) || gps[g0] > g;
  const uint32_t c = idxs[i];
  const bool on = valid[c] && !dominated;
  front[c] = on;
  if (on && count) atomicAdd(count, 1u);
}

struct MaxU64 {
  __device__ __forceinline__ unsigned long long operator()(unsigned long long a, unsigned long long b) const {
    return a > b ? a : b;
  }
};
struct MaxU32 {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

// scratch layout inside one device buffer (bytes); returns the bytes needed for n configs
size_t pareto_scratch_bytes(uint32_t n, size_t* cub_bytes_out) {
  size_t c1 = 0, c2 = 0, c3 = 0, c4 = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, c1, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                            (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
  cub::DeviceRadixSort::SortPairs(nullptr, c2, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)n);
  cub::DeviceScan::ExclusiveScan(nullptr, c3, (unsigned long long*)nullptr, (unsigned long long*)nullptr, MaxU64(),
                                 0ull, (int)n);
  cub::DeviceScan::InclusiveScan(nullptr, c4, (uint32_t*)nullptr, (uint32_t*)nullptr, MaxU32(), (int)n);
  size_t cb = c1;
  if (c2 > cb) cb = c2;
  if (c3 > cb) cb = c3;
  if (c4 > cb) cb = c4;
  cb = (cb + 255) & ~(size_t)255;
  *cub_bytes_out = cb;
  const size_t per = 2 * sizeof(uint32_t) /*p99 a,b*/ + 2 * sizeof(unsigned long long) /*gp a,b*/ +
                     2 * sizeof(uint32_t) /*idx a,b*/ + sizeof(unsigned long long) /*exmax*/ + sizeof(uint32_t) /*gstart*/ +
                     1 /*valid*/;
  return cb + (size_t)n * per + 8 * 256;
}

cudaError_t pareto_launch(const slo_config_agg* agg, uint32_t n, uint8_t* front, uint32_t* count, void* scratch,
                          size_t cub_bytes, cudaStream_t st) {
  char* base = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* p = base;
    base += (bytes + 255) & ~(size_t)255;
    return p;
  };
  void* cubtmp = take(cub_bytes);
  uint32_t* p99a = (uint32_t*)take(4ull * n);
  uint32_t* p99b = (uint32_t*)take(4ull * n);
  unsigned long long* gpa = (unsigned long long*)take(8ull * n);
  unsigned long long* gpb = (unsigned long long*)take(8ull * n);
  uint32_t* idxa = (uint32_t*)take(4ull * n);
  uint32_t* idxb = (uint32_t*)take(4ull * n);
  unsigned long long* exmax = (unsigned long long*)take(8ull * n);
  uint32_t* gstart = (uint32_t*)take(4ull * n);
  uint8_t* valid = (uint8_t*)take(n);
  const unsigned T = 256, Bk = (n + T - 1) / T;
  cudaError_t e;
  if (count && (e = cudaMemsetAsync(count, 0, sizeof(uint32_t), st)) != cudaSuccess) return e;
  pareto_objectives_kernel<<<Bk, T, 0, st>>>(agg, n, p99a, gpa, idxa, valid);
  size_t cb = cub_bytes;
  // 1. goodput descending (stable), 2. p99 ascending (stable): order (p99 asc, goodput desc)
  if ((e = cub::DeviceRadixSort::SortPairsDescending(cubtmp, cb, gpa, gpb, idxa, idxb, (int)n, 0, 64, st)) != cudaSuccess)
    return e;
  gather_kernel<uint32_t><<<Bk, T, 0, st>>>(p99a, idxb, n, p99b);
  cb = cub_bytes;
  if ((e = cub::DeviceRadixSort::SortPairs(cubtmp, cb, p99b, p99a, idxb, idxa, (int)n, 0, 32, st)) != cudaSuccess)
    return e;
  gather_kernel<unsigned long long><<<Bk, T, 0, st>>>(gpa, idxa, n, gpb);   // gpa still holds gp by config
  cb = cub_bytes;
  if ((e = cub::DeviceScan::ExclusiveScan(cubtmp, cb, gpb, exmax, MaxU64(), 0ull, (int)n, st)) != cudaSuccess) return e;
  group_start_kernel<<<Bk, T, 0, st>>>(p99a, n, p99b);
  cb = cub_bytes;
  if ((e = cub::DeviceScan::InclusiveScan(cubtmp, cb, p99b, gstart, MaxU32(), (int)n, st)) != cudaSuccess) return e;
  pareto_mark_kernel<<<Bk, T, 0, st>>>(gpb, exmax, gstart, idxa, valid, n, front, count);
  return cudaGetLastError();
}

}  // namespace slo
