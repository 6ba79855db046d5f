// slo_abi.cu — the C ABI of libslosim.so (include/slo_sim.h): handle, validation, stream-ordered launches.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <array>
#include <vector>

#include "slo_internal.h"
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: host ranges around each launch phase (nsys / ncu timelines)

static_assert(sizeof(slo_knobs) == 32, "slo_knobs must be 32 B");
static_assert(sizeof(slo_replica_result) == 32, "slo_replica_result must be 32 B");
static_assert(sizeof(slo_config_agg) == 32, "slo_config_agg must be 32 B");
static_assert(sizeof(slo_stats) == 64, "slo_stats must be 64 B");
static_assert(sizeof(slo_timing) == 40, "slo_timing must be 40 B");
static_assert(sizeof(slo_arrivals) == 40, "slo_arrivals must be 40 B");
static_assert(sizeof(slo_climb_state) == 104, "slo_climb_state must be 104 B");
static_assert(sizeof(slo_score_params) == 80, "slo_score_params must be 80 B");

// K1b block size by row length: short rows take smaller blocks (their per-row histogram scans and barriers, not
// the loads, dominate; C5s's 2,000-value rows: 6.1 ms at 256 threads, 4.7 at 128, 4.2 at 64)
static int sel_threads_for(uint32_t n) { return n <= 2048u ? 64 : (n <= 4096u ? 128 : 256); }

struct slo_sim {
  int device = 0;
  int sm_count = 0;
  int warps_per_block = slo::kDefaultWarpsPerBlock;
  int blocks_per_sm_opt = 0;
  uint32_t n_wl = 0;
  uint32_t crn = 1;
  bool any_cont = false;            // a workload uses continuous batching: launch K1c
  bool any_think = false;           // a static-batching workload has think time (kind 4): launch K1t
  bool any_cont_think = false;      // a continuous-batching workload has think time: launch K1c on lists 9-11
  bool any_cont_plain = false;      // a continuous-batching workload without think time: K1c on lists 3-5
  uint32_t group_policy = 0;        // slo_sim_opts.group_policy
  uint32_t gen_policy = 0;          // slo_sim_opts.gen_policy
  bool any_static_plain = false;    // a static-batching workload without think time (K1 / K1g + K1s)
  std::vector<slo::DevWorkload> h_wl;  // host copy of the device workload descriptors
  slo::DevWorkload* d_wl = nullptr;
  uint32_t* d_tables = nullptr;
  uint32_t* d_ctl = nullptr;        // [slo::kCtlWords]: list lengths, K1 cursors, K0 bucket counts/cursors
  // run scratch (grow-only): work lists, latency rows, per-replica partial results
  uint32_t* d_lists = nullptr;
  size_t lists_cap = 0;
  uint32_t* d_lat = nullptr;
  size_t lat_cap = 0;
  slo_replica_result* d_part = nullptr;
  size_t part_cap = 0;
  uint4* d_rec = nullptr;           // split path: K1g's request records, [chunk][N]
  size_t rec_cap = 0;
  size_t lat_budget = (size_t)4 << 30;  // bytes of latency rows per launch chunk
  char* d_pareto = nullptr;         // K5 scratch (grow-only)
  size_t pareto_cap = 0;
  // host-entry scratch
  void* d_scratch = nullptr;
  size_t scratch_bytes = 0;
  int regs = 0;
  int sel_bps[3] = {1, 1, 1};       // K1b resident blocks per SM at 64 / 128 / 256 threads (grid: one wave)
  double* d_sel_gp = nullptr;       // slo_select_rows: the goodput K1b writes (unused)
  size_t sel_gp_cap = 0;
  bool pinned = false;              // scratch referenced by a captured CUDA graph: never regrown (ensure())
  // measurement hook (slo_sim_profile): events around each chunk's K0 | simulation kernels | K1b
  bool profile = false;
  std::vector<cudaEvent_t> ev_free;             // recycled events
  std::vector<std::array<cudaEvent_t, 7>> ev_marks;  // recorded, not yet read

  std::string err;
};

namespace {

thread_local std::string g_err;

slo_status fail(slo_sim* h, slo_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  g_err = buf;
  return s;
}

#define CUDA_TRY(h, call)                                                                   \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) return fail((h), SLO_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

struct NvtxRange {               // scoped NVTX range (free when no profiler is attached)
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// bucket guide of a length table: for the 2^24-wide bucket b of u, entry b packs
// lo_b = #{l : cw[l] <= b 2^24} and hi_b = #{l : cw[l] <= b 2^24 + 2^24 - 1}; the count for any u in the bucket
// lies in [lo_b, hi_b], so lo_b == hi_b answers at once and otherwise a search over cw[lo_b, hi_b) does
void append_guide(std::vector<uint32_t>& t, const uint32_t* cw, uint32_t ncw) {
  uint32_t lo = 0, hi = 0;
  for (uint32_t b = 0; b < 256; ++b) {
    const uint32_t umin = b << 24, umax = umin | 0xFFFFFFu;
    while (lo < ncw && cw[lo] <= umin) ++lo;
    if (hi < lo) hi = lo;
    while (hi < ncw && cw[hi] <= umax) ++hi;
    t.push_back(lo | (hi << 16));
  }
}

bool table_ok(const uint32_t* cw, uint32_t ncw, uint32_t lo) {
  if (lo < 1 || (uint64_t)lo + ncw > SLO_MAX_LENGTH) return false;
  if (ncw > 0 && cw == nullptr) return false;
  for (uint32_t i = 1; i < ncw; ++i)
    if (cw[i] < cw[i - 1]) return false;
  return true;
}

// slo_select_rows: the replica records K1b reads (n_measured; window 1 so its goodput division is defined)
__global__ void select_rows_part_kernel(slo_replica_result* part, uint32_t n, uint32_t row_len,
                                        const uint32_t* __restrict__ nm) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t m = nm ? (nm[r] < row_len ? nm[r] : row_len) : row_len;
  part[r] = slo_replica_result{0, 0, m, 0, 1, 0};
}

}  // namespace

// grow-only device scratch owned by the handle (callers synchronise before a regrow).  A call made while `st`
// is being captured into a CUDA graph pins the handle's scratch: the graph holds its pointers, so every later
// call that would regrow (free + reallocate) the scratch is refused instead of leaving the graph dangling.
template <typename T>
slo_status ensure(slo_sim* h, T*& ptr, size_t& cap, size_t need, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) h->pinned = true;
  if (need <= cap) return SLO_OK;
  if (h->pinned)
    return fail(h, SLO_E_RANGE, "scratch of %zu B needed, but this handle's scratch is held by a captured CUDA graph "
                "(use a separate handle for larger runs)", need * sizeof(T));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  cap = 0;
  if (cudaMalloc(&ptr, need * sizeof(T)) != cudaSuccess) return fail(h, SLO_E_NOMEM, "scratch of %zu B", need * sizeof(T));
  cap = need;
  return SLO_OK;
}

extern "C" {

const char* slo_status_string(slo_status s) {
  switch (s) {
    case SLO_OK: return "ok";
    case SLO_E_INVAL: return "invalid argument";
    case SLO_E_NOMEM: return "out of memory";
    case SLO_E_CUDA: return "CUDA error";
    case SLO_E_RANGE: return "size out of range";
    case SLO_E_DEVICE: return "no usable device";
    case SLO_E_UNSUPPORTED: return "unsupported";
    default: return "unknown status";
  }
}

const char* slo_last_error(const slo_sim* h) { return h ? h->err.c_str() : g_err.c_str(); }

slo_status slo_sim_create(int device, const slo_workload* wl, uint32_t n_wl, const slo_sim_opts* opts,
                          slo_sim** out) {
  if (!out || !wl || n_wl == 0 || n_wl > 255) return fail(nullptr, SLO_E_INVAL, "create: bad arguments");
  *out = nullptr;
  slo_sim_opts o{};
  o.crn = 1;
  if (opts) {
    o = *opts;
    for (int i = 0; i < 2; ++i)
      if (o.reserved[i]) return fail(nullptr, SLO_E_INVAL, "create: opts.reserved must be 0");
    if (o.group_policy > 3) return fail(nullptr, SLO_E_INVAL, "create: opts.group_policy must be 0..3");
    if (o.gen_policy > 2) return fail(nullptr, SLO_E_INVAL, "create: opts.gen_policy must be 0..2");
    if (o.crn > 1) return fail(nullptr, SLO_E_INVAL, "create: opts.crn must be 0 or 1");
    if (o.warps_per_block > (uint32_t)slo::kMaxWarpsPerBlock)
      return fail(nullptr, SLO_E_INVAL, "create: warps_per_block > %d", slo::kMaxWarpsPerBlock);
  }
  // ---- validate the workloads (include/slo_sim.h)
  std::vector<slo::DevWorkload> hw(n_wl);
  std::vector<uint32_t> tables;
  for (uint32_t w = 0; w < n_wl; ++w) {
    const slo_workload& x = wl[w];
    const uint64_t NOA = ~0ull;
    if (x.arr.kind > 4 || x.arr.start_state > 1) return fail(nullptr, SLO_E_INVAL, "workload %u: bad arrival kind", w);
    if (x.arr.kind == 4 && x.arr.mean_gap_q16[0] == NOA)
      return fail(nullptr, SLO_E_INVAL, "workload %u: think time needs a finite mean (mean_gap_q16[0])", w);
    for (int s = 0; s < 2; ++s)
      if (x.arr.mean_gap_q16[s] != NOA && x.arr.mean_gap_q16[s] > (1ull << 48))
        return fail(nullptr, SLO_E_INVAL, "workload %u: mean_gap_q16 > 2^48", w);
    if (x.arr.kind == 0 && (x.arr.mean_gap_q16[0] == NOA || x.arr.mean_gap_q16[0] == 0))
      return fail(nullptr, SLO_E_INVAL, "workload %u: Poisson needs a finite positive gap", w);
    if (x.arr.kind == 1 || x.arr.kind == 2) {
      if (x.arr.mean_gap_q16[0] == NOA && x.arr.mean_gap_q16[1] == NOA)
        return fail(nullptr, SLO_E_INVAL, "workload %u: no state has arrivals", w);
      for (int s = 0; s < 2; ++s) {
        if (x.arr.mean_sojourn_us[s] < 1 || x.arr.mean_sojourn_us[s] > (1ull << 40))
          return fail(nullptr, SLO_E_INVAL, "workload %u: sojourn out of [1, 2^40]", w);
        if (x.arr.mean_gap_q16[s] == 0) return fail(nullptr, SLO_E_INVAL, "workload %u: zero gap", w);
      }
    }
    if (!table_ok(x.prompt_cw, x.prompt_ncw, x.prompt_lo) || !table_ok(x.output_cw, x.output_ncw, x.output_lo))
      return fail(nullptr, SLO_E_INVAL, "workload %u: bad length table", w);
    const uint32_t* tv = &x.timing.pre_base_us;
    for (int i = 0; i < 9; ++i)
      if (tv[i] >= (1u << 20)) return fail(nullptr, SLO_E_INVAL, "workload %u: timing value >= 2^20", w);
    if (x.timing.noise_step_ppm > 1960) return fail(nullptr, SLO_E_INVAL, "workload %u: noise_step_ppm > 1960", w);
    {   // worst-case decode step d(n) over gamma <= 16, W <= 4, n <= 32 (R10, R28) must stay below 2^31 us: K1c
        // keeps a step's duration in 32 bits
      const slo_timing& t = x.timing;
      const uint64_t dmax_spec = 64ull * (t.dr_base_us + 32ull * t.dr_seq_us) + t.ver_base_us + 32ull * t.ver_seq_us +
                                 65ull * 32ull * t.ver_tok_us;
      const uint64_t dmax_plain = t.dec_base_us + 32ull * t.dec_seq_us;
      if (dmax_spec >= (1ull << 31) || dmax_plain >= (1ull << 31))
        return fail(nullptr, SLO_E_INVAL, "workload %u: worst-case decode step cost >= 2^31 us", w);
    }
    if (x.batching > 1) return fail(nullptr, SLO_E_INVAL, "workload %u: batching must be 0 or 1", w);
    slo::DevWorkload& d = hw[w];
    memset(&d, 0, sizeof d);
    d.kind = x.arr.kind;
    d.start_state = x.arr.start_state;
    d.gap_q16[0] = x.arr.mean_gap_q16[0];
    d.gap_q16[1] = x.arr.mean_gap_q16[1];
    d.soj[0] = x.arr.mean_sojourn_us[0];
    d.soj[1] = x.arr.mean_sojourn_us[1];
    d.p_lo = x.prompt_lo;
    d.p_ncw = x.prompt_ncw;
    d.p_off = (uint32_t)tables.size();
    tables.insert(tables.end(), x.prompt_cw, x.prompt_cw + x.prompt_ncw);
    d.p_goff = (uint32_t)tables.size();
    append_guide(tables, x.prompt_cw, x.prompt_ncw);
    d.o_lo = x.output_lo;
    d.o_ncw = x.output_ncw;
    d.o_off = (uint32_t)tables.size();
    tables.insert(tables.end(), x.output_cw, x.output_cw + x.output_ncw);
    d.o_goff = (uint32_t)tables.size();
    append_guide(tables, x.output_cw, x.output_ncw);
    d.t = x.timing;
    d.stream_id = x.stream_id;
    d.batching = x.batching;
  }
  if (tables.empty()) tables.push_back(0);

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(nullptr, SLO_E_DEVICE, "create: no CUDA device %d", device);
  cudaDeviceProp prop;
  // the library carries sm_100a SASS only (no PTX): any other architecture could create a handle but fail
  // every launch with "no kernel image", so it is refused here
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10 || prop.minor != 0)
    return fail(nullptr, SLO_E_DEVICE, "create: device %d is not sm_100 (B200)", device);
  DeviceGuard g(device);

  slo_sim* h = new (std::nothrow) slo_sim();
  if (!h) return fail(nullptr, SLO_E_NOMEM, "create: host allocation");
  h->device = device;
  h->sm_count = prop.multiProcessorCount;
  h->n_wl = n_wl;
  for (uint32_t w = 0; w < n_wl; ++w) h->any_cont |= wl[w].batching == 1;
  for (uint32_t w = 0; w < n_wl; ++w) {
    h->any_think |= wl[w].arr.kind == 4 && wl[w].batching == 0;
    h->any_cont_think |= wl[w].arr.kind == 4 && wl[w].batching == 1;
    h->any_cont_plain |= wl[w].arr.kind != 4 && wl[w].batching == 1;
    h->any_static_plain |= wl[w].arr.kind != 4 && wl[w].batching == 0;
  }
  h->crn = o.crn;
  if (o.warps_per_block) h->warps_per_block = (int)o.warps_per_block;
  h->blocks_per_sm_opt = (int)o.blocks_per_sm;
  if (o.scratch_mb) h->lat_budget = (size_t)o.scratch_mb << 20;
  h->group_policy = o.group_policy;
  h->gen_policy = o.gen_policy;
  h->h_wl = hw;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, slo::slo_sim_kernel_t<false>) != cudaSuccess) {
    cudaGetLastError();
    slo_sim_destroy(h);
    return fail(nullptr, SLO_E_DEVICE, "create: no sm_100a kernel image for device %d", device);
  }
  h->regs = fa.numRegs;
  for (int i = 0; i < 3; ++i)
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&h->sel_bps[i], slo::slo_select_kernel, 64 << i, 0) !=
            cudaSuccess || h->sel_bps[i] < 1)
      h->sel_bps[i] = 1;
  cudaError_t e;
  if ((e = cudaMalloc(&h->d_wl, sizeof(slo::DevWorkload) * n_wl)) != cudaSuccess ||
      (e = cudaMalloc(&h->d_tables, sizeof(uint32_t) * tables.size())) != cudaSuccess ||
      (e = cudaMalloc(&h->d_ctl, sizeof(uint32_t) * slo::kCtlWords)) != cudaSuccess) {
    slo_sim_destroy(h);
    return fail(nullptr, SLO_E_NOMEM, "create: cudaMalloc: %s", cudaGetErrorString(e));
  }
  if ((e = cudaMemcpy(h->d_wl, hw.data(), sizeof(slo::DevWorkload) * n_wl, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(h->d_tables, tables.data(), sizeof(uint32_t) * tables.size(), cudaMemcpyHostToDevice)) !=
          cudaSuccess) {
    slo_sim_destroy(h);
    return fail(nullptr, SLO_E_CUDA, "create: cudaMemcpy: %s", cudaGetErrorString(e));
  }
  *out = h;
  return SLO_OK;
}

slo_status slo_sim_profile(slo_sim* h, uint32_t enable) {
  if (!h) return fail(nullptr, SLO_E_INVAL, "profile: null handle");
  h->profile = enable != 0;
  return SLO_OK;
}

slo_status slo_sim_profile_read(slo_sim* h, double* h_ms, uint32_t* h_chunks) {
  if (!h || !h_ms) return fail(h, SLO_E_INVAL, "profile_read: null argument");
  DeviceGuard g(h->device);
  h_ms[0] = h_ms[1] = h_ms[2] = h_ms[3] = h_ms[4] = 0.0;
  // marks per chunk: 0/1 around K0, 2/3 around K1g, 4/5 around the chain kernels, 5/6 K1b; 1/5 the simulation
  static const int from[5] = {0, 2, 4, 5, 1}, to[5] = {1, 3, 5, 6, 5};
  for (auto& m : h->ev_marks) {
    CUDA_TRY(h, cudaEventSynchronize(m[6]));
    CUDA_TRY(h, cudaEventSynchronize(m[3]));
    for (int i = 0; i < 5; ++i) {
      float ms = 0.0f;
      CUDA_TRY(h, cudaEventElapsedTime(&ms, m[from[i]], m[to[i]]));
      h_ms[i] += ms;
    }
    for (int i = 0; i < 7; ++i) h->ev_free.push_back(m[i]);
  }
  if (h_chunks) *h_chunks = (uint32_t)h->ev_marks.size();
  h->ev_marks.clear();
  return SLO_OK;
}

slo_status slo_sim_destroy(slo_sim* h) {
  if (!h) return SLO_OK;
  {
    DeviceGuard g(h->device);
    cudaDeviceSynchronize();
    if (h->d_wl) cudaFree(h->d_wl);
    if (h->d_tables) cudaFree(h->d_tables);
    if (h->d_ctl) cudaFree(h->d_ctl);
    if (h->d_lists) cudaFree(h->d_lists);
    if (h->d_lat) cudaFree(h->d_lat);
    if (h->d_part) cudaFree(h->d_part);
    if (h->d_rec) cudaFree(h->d_rec);
    if (h->d_scratch) cudaFree(h->d_scratch);
    if (h->d_pareto) cudaFree(h->d_pareto);
    if (h->d_sel_gp) cudaFree(h->d_sel_gp);
    for (auto& m : h->ev_marks)
      for (cudaEvent_t e : m) cudaEventDestroy(e);
    for (cudaEvent_t e : h->ev_free) cudaEventDestroy(e);

  }
  delete h;
  return SLO_OK;
}

static int blocks_per_sm_for(slo_sim* h, size_t smem) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slo::slo_sim_kernel_t<false>, h->warps_per_block * 32, smem) !=
          cudaSuccess ||
      occ < 1)
    occ = 1;
  if (h->blocks_per_sm_opt > 0 && h->blocks_per_sm_opt < occ) occ = h->blocks_per_sm_opt;
  return occ;
}

slo_status slo_sim_get_info(const slo_sim* hc, slo_sim_info* info) {
  if (!hc || !info) return fail(nullptr, SLO_E_INVAL, "get_info: null");
  slo_sim* h = const_cast<slo_sim*>(hc);
  DeviceGuard g(h->device);
  const size_t wb = slo::group_warp_bytes();
  memset(info, 0, sizeof *info);
  info->device = h->device;
  info->sm_count = h->sm_count;
  info->warps_per_block = h->warps_per_block;
  info->blocks_per_sm = blocks_per_sm_for(h, wb * h->warps_per_block);
  info->regs_per_thread = h->regs;
  info->smem_per_warp_bytes = (int32_t)wb;
  return SLO_OK;
}

static slo_status launch_sim(slo_sim* h, const slo_knobs* d_configs, uint32_t n_configs, const uint64_t* d_seeds,
                             uint32_t n_seeds, uint32_t segment_len, uint32_t warmup_len, uint32_t slo_us,
                             uint32_t* d_p99, double* d_goodput, slo_replica_result* d_detail, uint32_t* d_lat,
                             slo_stats* d_stats, uint32_t* d_p50, uint32_t* d_p95, cudaStream_t st,
                             uint32_t stop_n = 0, uint32_t stop_t = 0, const uint32_t* d_live = nullptr) {
  const uint32_t n_rep = (uint32_t)((uint64_t)n_configs * n_seeds);
  const uint32_t N = warmup_len + segment_len;
  // replicas per launch chunk: the latency rows of a chunk stay within the budget (a caller-provided
  // latency buffer is written in place, chunk by chunk)
  // (K1 indexes a chunk's rows with 32-bit offsets: chunk * N < 2^31 elements)
  uint64_t chunk = h->lat_budget / ((uint64_t)N * 4u);
  if (chunk * N >= (1ull << 31)) chunk = ((1ull << 31) - 1) / N;
  if (chunk < 1) chunk = 1;
  if (chunk > n_rep) chunk = n_rep;
  // static batching without think time runs the split path (K1g records, K1s chain) unless gen_policy = 1 asks
  // for K1's inline generation
  const bool split = (h->any_static_plain || h->any_cont_plain) && h->gen_policy != 1;
  slo_status s;
  if ((s = ensure(h, h->d_lists, h->lists_cap, (size_t)slo::kLists * chunk, st)) != SLO_OK) return s;
  if (!d_lat && (s = ensure(h, h->d_lat, h->lat_cap, (size_t)chunk * N, st)) != SLO_OK) return s;
  if (!d_detail && (s = ensure(h, h->d_part, h->part_cap, (size_t)n_rep, st)) != SLO_OK) return s;
  // 16 B of K1g records per request of the chunk
  if (split && (s = ensure(h, h->d_rec, h->rec_cap, (size_t)chunk * N, st)) != SLO_OK) return s;

  int gen_bps = 1, serve_bps = 1;
  const size_t serve_smem = slo::serve_warp_bytes() * h->warps_per_block;
  if (split) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&gen_bps, slo::slo_gen_kernel, slo::kGenThreads, 0) != cudaSuccess ||
        gen_bps < 1)
      gen_bps = 1;
    if (serve_smem > 48 * 1024) {
      CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_serve_kernel_t<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)serve_smem));
      CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_serve_kernel_t<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)serve_smem));
    }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&serve_bps, slo::slo_serve_kernel_t<false>, h->warps_per_block * 32,
                                                      serve_smem) != cudaSuccess || serve_bps < 1)
      serve_bps = 1;
    if (h->blocks_per_sm_opt > 0 && h->blocks_per_sm_opt < serve_bps) serve_bps = h->blocks_per_sm_opt;
  }

  slo::SimParams p{};
  p.cfg = d_configs;
  p.seeds = d_seeds;
  p.wl = h->d_wl;
  p.tables = h->d_tables;
  p.counts = h->d_ctl;
  p.cursor = h->d_ctl + slo::kLists;
  p.lists = h->d_lists;
  p.part = d_detail ? d_detail : h->d_part;
  p.p99 = d_p99;
  p.p50 = d_p50;
  p.p95 = d_p95;
  p.goodput = d_goodput;
  p.detail = d_detail;
  p.stats = d_stats;
  p.n_cfg = n_configs;
  p.n_seeds = n_seeds;
  p.n_rep = n_rep;
  p.n_wl = h->n_wl;
  p.warmup = warmup_len;
  p.seg = segment_len;
  p.slo_us = slo_us;
  p.crn = h->crn;
  p.stop_n = stop_n;
  p.stop_t = stop_t;
  p.live = d_live;
  p.warp_bytes = (uint32_t)slo::group_warp_bytes();
  const size_t smem = (size_t)p.warp_bytes * h->warps_per_block;
  if (smem > 48 * 1024)
  {
    CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_kernel_t<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_kernel_t<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (h->any_think) {
      CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_think_kernel_t<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
      CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_think_kernel_t<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    }
  }
  const int bps = blocks_per_sm_for(h, smem);
  int cont_bps = 1;
  slo::SimParams pc{};
  const size_t cont_smem = slo::cont_warp_bytes() * h->warps_per_block;
  if (h->any_cont || h->any_cont_think) {
    if (cont_smem > 48 * 1024)
    {
      CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_cont_kernel_t<false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)cont_smem));
      CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_cont_kernel_t<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)cont_smem));
      CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_cont_kernel_t<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)cont_smem));
      CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_cont_kernel_t<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)cont_smem));
      CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_cont_kernel_t<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)cont_smem));
      CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_cont_kernel_t<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)cont_smem));
    }
    // occupancy is register-bound; give the group rings the whole carveout so smem never binds first
    CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_cont_kernel_t<false, false, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_cont_kernel_t<true, false, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_cont_kernel_t<false, true, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_cont_kernel_t<true, true, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_cont_kernel_t<false, false, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CUDA_TRY(h, cudaFuncSetAttribute(slo::slo_sim_cont_kernel_t<true, false, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cont_bps, slo::slo_sim_cont_kernel_t<false, false, false>, h->warps_per_block * 32,
                                                      cont_smem) != cudaSuccess || cont_bps < 1)
      cont_bps = 1;
    if (h->blocks_per_sm_opt > 0 && h->blocks_per_sm_opt < cont_bps) cont_bps = h->blocks_per_sm_opt;
  }
  // K1b reads each row from L2 (a just-written row stays there across the radix passes): staging rows of up
  // to 43 KB in shared memory capped residency at 5 blocks/SM and measured 1.5 % slower on C2
  if (d_stats) CUDA_TRY(h, cudaMemsetAsync(d_stats, 0, sizeof(slo_stats), st));
  bool prof = h->profile;
  if (prof) {                                     // no event marks inside a graph capture
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) prof = false;
  }
  std::array<cudaEvent_t, 7> ev{};
  auto mark = [&](int i, cudaStream_t on) -> slo_status {
    if (!prof) return SLO_OK;
    if (h->ev_free.empty()) {
      cudaEvent_t e;
      CUDA_TRY(h, cudaEventCreate(&e));
      h->ev_free.push_back(e);
    }
    ev[i] = h->ev_free.back();
    h->ev_free.pop_back();
    CUDA_TRY(h, cudaEventRecord(ev[i], on));
    if (i == 6) h->ev_marks.push_back(ev);
    return SLO_OK;
  };

  for (uint64_t r0 = 0; r0 < n_rep; r0 += chunk) {
    const uint32_t nc = (uint32_t)((n_rep - r0) < chunk ? (n_rep - r0) : chunk);
    p.r_base = (uint32_t)r0;
    p.n_chunk = nc;
    p.lists = h->d_lists;
    p.lat = d_lat ? d_lat + r0 * N : h->d_lat;
    NvtxRange chunk_range("slo_sim_run chunk");
    if ((s = mark(0, st)) != SLO_OK) return s;
    CUDA_TRY(h, cudaMemsetAsync(h->d_ctl, 0, sizeof(uint32_t) * slo::kCtlWords, st));
    // lane groups: narrow (G >= min(C, B), up to four replicas per warp) by default — measured best from
    // 512-replica climb steps (one 8-GPU rank of C4) up to the full sweeps; a chunk of at most one replica per
    // SM runs each replica on a whole warp (C1: shortest chain); wide (G >= max(C, B)) only when forced
    const uint32_t wide = (h->group_policy == 3 ? 2u
                           : h->group_policy == 2 ? 1u
                           : h->group_policy == 1 ? 0u
                           : nc <= (uint32_t)h->sm_count && !split ? 2u : 0u) | (split ? 4u : 0u);   // bit 2: split
    // (a lone replica runs K1's inline generation fastest on a whole warp; K1s's chain is shortest on narrow
    // groups, spread one replica per warp by gpw below)
    slo::slo_classify_count_kernel<<<(nc + 255) / 256, 256, 0, st>>>(d_configs, h->d_wl, n_seeds, (uint32_t)r0, nc,
                                                                    h->n_wl, wide, h->d_ctl, d_live);
    CUDA_TRY(h, cudaGetLastError());
    slo::slo_classify_kernel<<<(nc + 255) / 256, 256, 0, st>>>(d_configs, h->d_wl, n_seeds, (uint32_t)r0, nc, h->n_wl,
                                                              wide, h->d_ctl, h->d_lists, d_live);
    CUDA_TRY(h, cudaGetLastError());
    if ((s = mark(1, st)) != SLO_OK) return s;
    uint64_t blocks = (uint64_t)bps * h->sm_count;
    const uint64_t need = ((uint64_t)nc + 4u * h->warps_per_block - 1) / (4u * h->warps_per_block);
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    const bool stop = (p.stop_n | p.stop_t) != 0;
    if (split) {   // K1g: every request's record at full width, then K1s: the batch chain over the records
      p.rec = h->d_rec;
      // K1s lane groups per warp: the fewest that still fit every replica of the chunk into the resident warp
      // slots (one wave) — the chain is latency-bound, so a small launch runs one replica per warp
      const uint64_t slots = (uint64_t)serve_bps * h->sm_count * h->warps_per_block;
      uint64_t gpw = (nc + slots - 1) / slots;
      if (gpw < 1) gpw = 1;
      if (gpw > 8) gpw = 8;
      uint64_t gblocks = (uint64_t)gen_bps * h->sm_count;
      if (gblocks > (uint64_t)nc * ((N + 255) / 256)) gblocks = (uint64_t)nc * ((N + 255) / 256);
      uint64_t sblocks = (uint64_t)serve_bps * h->sm_count;
      const uint64_t sneed = ((uint64_t)nc + gpw * h->warps_per_block - 1) / (gpw * h->warps_per_block);
      if (sblocks > sneed) sblocks = sneed;
      if (sblocks < 1) sblocks = 1;
      if ((s = mark(2, st)) != SLO_OK) return s;
      nvtxRangePushA("K1g generate");
      slo::slo_gen_kernel<<<(unsigned)gblocks, slo::kGenThreads, 0, st>>>(p, h->d_rec);
      CUDA_TRY(h, cudaGetLastError());
      nvtxRangePop();
      if ((s = mark(3, st)) != SLO_OK || (s = mark(4, st)) != SLO_OK) return s;
      NvtxRange chain_range("K1s chains");
      slo::SimParams ps = p;
      ps.gpw = (uint32_t)gpw;
      ps.warp_bytes = (uint32_t)slo::serve_warp_bytes();
      if (h->any_static_plain) {
        stop ? slo::slo_serve_kernel_t<true><<<(unsigned)sblocks, h->warps_per_block * 32, serve_smem, st>>>(ps)
             : slo::slo_serve_kernel_t<false><<<(unsigned)sblocks, h->warps_per_block * 32, serve_smem, st>>>(ps);
        CUDA_TRY(h, cudaGetLastError());
      }
      p.rec = nullptr;
    } else {
      if ((s = mark(2, st)) != SLO_OK || (s = mark(3, st)) != SLO_OK || (s = mark(4, st)) != SLO_OK)
        return s;                                     // (no K1g: an empty interval)
      stop ? slo::slo_sim_kernel_t<true><<<(unsigned)blocks, h->warps_per_block * 32, smem, st>>>(p)
           : slo::slo_sim_kernel_t<false><<<(unsigned)blocks, h->warps_per_block * 32, smem, st>>>(p);
    }
    CUDA_TRY(h, cudaGetLastError());
    if (h->any_think) {  // K1t: closed loops with think time (same group layout and grid as K1)
      if (p.stop_n | p.stop_t)
        slo::slo_sim_think_kernel_t<true><<<(unsigned)blocks, h->warps_per_block * 32, smem, st>>>(p);
      else
        slo::slo_sim_think_kernel_t<false><<<(unsigned)blocks, h->warps_per_block * 32, smem, st>>>(p);
      CUDA_TRY(h, cudaGetLastError());
    }
    // K1c over the continuous-batching lists (one launch for lists 3-5, one for the think-time lists 9-11)
    NvtxRange cont_range("K1c continuous");
    for (uint32_t think = 0; think < 2; ++think) {
      if (!(think ? h->any_cont_think : h->any_cont_plain)) continue;
      uint64_t cblocks = (uint64_t)cont_bps * h->sm_count;   // (one replica per warp at most: the K1e scans)
      const uint64_t cneed = ((uint64_t)nc + h->warps_per_block - 1) / h->warps_per_block;
      if (cblocks > cneed) cblocks = cneed;
      pc = p;
      pc.warp_bytes = (uint32_t)slo::cont_warp_bytes();
      const dim3 cg((unsigned)cblocks), cb(h->warps_per_block * 32);
      if (think)
        (p.stop_n | p.stop_t) ? slo::slo_sim_cont_kernel_t<true, true, false><<<cg, cb, cont_smem, st>>>(pc)
                              : slo::slo_sim_cont_kernel_t<false, true, false><<<cg, cb, cont_smem, st>>>(pc);
      else if (split) {   // lists 3-5 from K1g's records
        pc.rec = h->d_rec;
        (p.stop_n | p.stop_t) ? slo::slo_sim_cont_kernel_t<true, false, true><<<cg, cb, cont_smem, st>>>(pc)
                              : slo::slo_sim_cont_kernel_t<false, false, true><<<cg, cb, cont_smem, st>>>(pc);
      } else {
        (p.stop_n | p.stop_t) ? slo::slo_sim_cont_kernel_t<true, false, false><<<cg, cb, cont_smem, st>>>(pc)
                              : slo::slo_sim_cont_kernel_t<false, false, false><<<cg, cb, cont_smem, st>>>(pc);
      }
      CUDA_TRY(h, cudaGetLastError());
    }
    if ((s = mark(5, st)) != SLO_OK) return s;
    // one wave of resident blocks: a grid-stride second wave would start its rows late
    // (fewer rows than SMs: latency-bound, every row takes a full 256-thread block)
    const uint32_t sel_threads = nc < (uint32_t)h->sm_count ? 256u : (uint32_t)sel_threads_for(p.seg);
    const uint32_t sel_wave = (uint32_t)h->sm_count * (uint32_t)h->sel_bps[sel_threads == 64 ? 0 : (sel_threads == 128 ? 1 : 2)];
    const uint32_t sel_blocks = nc < sel_wave ? nc : sel_wave;
    nvtxRangePushA("K1b select");
    slo::slo_select_kernel<<<sel_blocks, sel_threads, 0, st>>>(p);
    nvtxRangePop();
    CUDA_TRY(h, cudaGetLastError());
    if ((s = mark(6, st)) != SLO_OK) return s;
  }
  return SLO_OK;
}

static slo_status check_run_args(slo_sim* h, uint32_t n_configs, uint32_t n_seeds, uint32_t segment_len,
                                 uint32_t warmup_len, uint32_t slo_us) {
  if (n_configs == 0 || n_seeds == 0 || segment_len == 0)
    return fail(h, SLO_E_INVAL, "run_batch: n_configs, n_seeds and segment_len must be > 0");
  if ((uint64_t)n_configs * n_seeds >= (1ull << 31)) return fail(h, SLO_E_RANGE, "run_batch: too many replicas");
  if ((uint64_t)segment_len + warmup_len > SLO_MAX_REQUESTS)
    return fail(h, SLO_E_RANGE, "run_batch: warmup_len + segment_len > %u", SLO_MAX_REQUESTS);
  if (slo_us == 0xFFFFFFFFu) return fail(h, SLO_E_RANGE, "run_batch: slo_us must be < UINT32_MAX");
  return SLO_OK;
}

slo_status slo_sim_run(slo_sim* h, const slo_run_args* a, void* stream) {
  if (!h) return fail(nullptr, SLO_E_INVAL, "run: null handle");
  if (!a || !a->d_configs || !a->d_seeds || !a->d_p99_us || !a->d_goodput)
    return fail(h, SLO_E_INVAL, "run: null pointer");
  slo_status s = check_run_args(h, a->n_configs, a->n_seeds, a->segment_len, a->warmup_len, a->slo_us);
  if (s != SLO_OK) return s;
  if (a->stop_min_completions || a->stop_min_time_us) {
    // the kernels end a replica at t*: exact only if nothing else can complete at t* after it, i.e. every batch
    // / iteration lasts >= 1 us.  floor(f x / 10^6) >= 1 for x >= 3 and f >= 10^6 - 510 * 1960 = 400,400 ppm.
    for (uint32_t w = 0; w < h->n_wl; ++w) {
      const slo_timing& t = h->h_wl[w].t;
      if ((uint64_t)t.pre_base_us + t.pre_tok_us < 3 || (uint64_t)t.dec_base_us + t.dec_seq_us < 3 ||
          (uint64_t)t.ver_base_us + t.ver_seq_us + t.ver_tok_us < 3)
        return fail(h, SLO_E_INVAL, "run: a stop rule needs every batch and iteration to last >= 1 us (workload %u "
                    "allows a zero-duration one)", w);
    }
  }
  DeviceGuard g(h->device);
  return launch_sim(h, a->d_configs, a->n_configs, a->d_seeds, a->n_seeds, a->segment_len, a->warmup_len, a->slo_us,
                    a->d_p99_us, a->d_goodput, a->d_detail, a->d_latencies, a->d_stats, a->d_p50_us, a->d_p95_us,
                    (cudaStream_t)stream, a->stop_min_completions, a->stop_min_time_us, a->d_live_configs);
}

slo_status slo_sim_run_batch(slo_sim* h, const slo_knobs* d_configs, uint32_t n_configs, const uint64_t* d_seeds,
                             uint32_t n_seeds, uint32_t segment_len, uint32_t warmup_len, uint32_t slo_us,
                             uint32_t* d_p99_us, double* d_goodput, slo_replica_result* d_detail,
                             uint32_t* d_latencies, slo_stats* d_stats, void* stream) {
  slo_run_args a{};
  a.d_configs = d_configs;
  a.n_configs = n_configs;
  a.d_seeds = d_seeds;
  a.n_seeds = n_seeds;
  a.segment_len = segment_len;
  a.warmup_len = warmup_len;
  a.slo_us = slo_us;
  a.d_p99_us = d_p99_us;
  a.d_goodput = d_goodput;
  a.d_detail = d_detail;
  a.d_latencies = d_latencies;
  a.d_stats = d_stats;
  return slo_sim_run(h, &a, stream);
}

slo_status slo_sim_run_batch_host(slo_sim* h, const slo_knobs* h_configs, uint32_t n_configs, const uint64_t* h_seeds,
                                  uint32_t n_seeds, uint32_t segment_len, uint32_t warmup_len, uint32_t slo_us,
                                  uint32_t* h_p99_us, double* h_goodput, slo_replica_result* h_detail,
                                  slo_stats* h_stats, void* stream) {
  if (!h) return fail(nullptr, SLO_E_INVAL, "run_batch_host: null handle");
  if (!h_configs || !h_seeds || !h_p99_us || !h_goodput) return fail(h, SLO_E_INVAL, "run_batch_host: null pointer");
  slo_status s = check_run_args(h, n_configs, n_seeds, segment_len, warmup_len, slo_us);
  if (s != SLO_OK) return s;
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t R = (uint64_t)n_configs * n_seeds;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t o_cfg = 0, o_seed = al(o_cfg + 32ull * n_configs), o_p99 = al(o_seed + 8ull * n_seeds),
               o_gp = al(o_p99 + 4ull * R), o_det = al(o_gp + 8ull * R), o_st = al(o_det + (h_detail ? 32ull * R : 0)),
               total = al(o_st + sizeof(slo_stats));
  if (total > h->scratch_bytes) {
    CUDA_TRY(h, cudaStreamSynchronize(st));
    if (h->d_scratch) cudaFree(h->d_scratch);
    h->d_scratch = nullptr;
    h->scratch_bytes = 0;
    if (cudaMalloc(&h->d_scratch, total) != cudaSuccess) return fail(h, SLO_E_NOMEM, "run_batch_host: scratch");
    h->scratch_bytes = total;
  }
  char* b = (char*)h->d_scratch;
  CUDA_TRY(h, cudaMemcpyAsync(b + o_cfg, h_configs, 32ull * n_configs, cudaMemcpyHostToDevice, st));
  CUDA_TRY(h, cudaMemcpyAsync(b + o_seed, h_seeds, 8ull * n_seeds, cudaMemcpyHostToDevice, st));
  s = launch_sim(h, (const slo_knobs*)(b + o_cfg), n_configs, (const uint64_t*)(b + o_seed), n_seeds, segment_len,
                 warmup_len, slo_us, (uint32_t*)(b + o_p99), (double*)(b + o_gp),
                 h_detail ? (slo_replica_result*)(b + o_det) : nullptr, nullptr,
                 h_stats ? (slo_stats*)(b + o_st) : nullptr, nullptr, nullptr, st);
  if (s != SLO_OK) return s;
  CUDA_TRY(h, cudaMemcpyAsync(h_p99_us, b + o_p99, 4ull * R, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(h_goodput, b + o_gp, 8ull * R, cudaMemcpyDeviceToHost, st));
  if (h_detail) CUDA_TRY(h, cudaMemcpyAsync(h_detail, b + o_det, 32ull * R, cudaMemcpyDeviceToHost, st));
  if (h_stats) CUDA_TRY(h, cudaMemcpyAsync(h_stats, b + o_st, sizeof(slo_stats), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  return SLO_OK;
}

slo_status slo_aggregate(slo_sim* h, const slo_replica_result* d_detail, uint32_t n_configs, uint32_t n_seeds,
                         slo_config_agg* d_agg, void* stream) {
  if (!h) return fail(nullptr, SLO_E_INVAL, "aggregate: null handle");
  if (!d_detail || !d_agg || n_configs == 0 || n_seeds == 0) return fail(h, SLO_E_INVAL, "aggregate: bad arguments");
  DeviceGuard g(h->device);
  const unsigned threads = 256, warps = threads / 32;
  const unsigned blocks = (unsigned)((n_configs + warps - 1) / warps);
  slo::slo_aggregate_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(d_detail, n_configs, n_seeds, d_agg);
  CUDA_TRY(h, cudaGetLastError());
  return SLO_OK;
}

slo_status slo_aggregate_reduce(slo_sim* h, const slo_config_agg* d_parts, uint32_t n_parts, uint32_t n_configs,
                                slo_config_agg* d_out, void* stream) {
  if (!h) return fail(nullptr, SLO_E_INVAL, "aggregate_reduce: null handle");
  if (!d_parts || !d_out || n_parts == 0 || n_configs == 0) return fail(h, SLO_E_INVAL, "aggregate_reduce: bad arguments");
  DeviceGuard g(h->device);
  const unsigned threads = 256;
  slo::slo_aggregate_reduce_kernel<<<(n_configs + threads - 1) / threads, threads, 0, (cudaStream_t)stream>>>(
      d_parts, n_parts, n_configs, d_out);
  CUDA_TRY(h, cudaGetLastError());
  return SLO_OK;
}

static bool space_ok(const slo_space* sp) {
  if (!sp || sp->stencil > 2) return false;
  for (int d = 0; d < 5; ++d) {
    if (sp->lo[d] < 0 || sp->lo[d] > sp->hi[d] || sp->step[d] < 0) return false;
    if (d < 4 && sp->hi[d] > 255) return false;
  }
  return true;
}

slo_status slo_neighbors(const slo_space* space, const slo_knobs* K, slo_knobs* out, uint32_t cap, uint32_t* n) {
  if (!space_ok(space) || !K || !n || (cap > 0 && !out)) return fail(nullptr, SLO_E_INVAL, "neighbors: bad arguments");
  *n = slo::neighbors_of(*space, *K, out, cap);
  return SLO_OK;
}

slo_status slo_hillclimb_step(slo_sim* h, const slo_space* space, const slo_score_params* sp, slo_knobs* d_cands,
                              uint32_t n_cand, const slo_config_agg* d_aggs, uint32_t n_parts,
                              slo_climb_state* d_state, int64_t* d_scores, void* stream) {
  if (!h) return fail(nullptr, SLO_E_INVAL, "hillclimb_step: null handle");
  if (!space_ok(space) || !sp || !d_cands || !d_aggs || !d_state || n_cand == 0 || n_cand > 32 || n_parts == 0)
    return fail(h, SLO_E_INVAL, "hillclimb_step: bad arguments");
  if (sp->lambda_milli < 0 || sp->delta_micro < 0 || sp->viol_mult < 1 || sp->ema_beta_q16 > 65536 || sp->reserved)
    return fail(h, SLO_E_INVAL, "hillclimb_step: bad score parameters");
  DeviceGuard g(h->device);
  slo::slo_climb_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(*space, *sp, d_cands, n_cand, d_aggs, n_parts, d_state,
                                                            d_scores);
  CUDA_TRY(h, cudaGetLastError());
  return SLO_OK;
}

static_assert(sizeof(slo::LookTable) == SLO_LOOKAHEAD_TABLE_BYTES, "SLO_LOOKAHEAD_TABLE_BYTES");

slo_status slo_lookahead_prepare(slo_sim* h, const slo_space* space, const slo_climb_state* d_state, void* d_table,
                                 slo_knobs* d_sim, void* stream) {
  if (!h) return fail(nullptr, SLO_E_INVAL, "lookahead_prepare: null handle");
  if (!space_ok(space) || !d_state || !d_table || !d_sim) return fail(h, SLO_E_INVAL, "lookahead_prepare: bad arguments");
  DeviceGuard g(h->device);
  slo::slo_lookahead_prepare_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(*space, d_state, (slo::LookTable*)d_table,
                                                                         d_sim);
  CUDA_TRY(h, cudaGetLastError());
  return SLO_OK;
}

slo_status slo_lookahead_step(slo_sim* h, const slo_space* space, const slo_score_params* sp, void* d_table,
                              const slo_config_agg* d_aggs, uint32_t n_parts, uint32_t n_cand,
                              slo_climb_state* d_state, slo_climb_state* d_traj, void* stream) {
  if (!h) return fail(nullptr, SLO_E_INVAL, "lookahead_step: null handle");
  if (!space_ok(space) || !sp || !d_table || !d_aggs || !d_state || !d_traj || n_cand < 2 || n_cand > 32 ||
      n_parts == 0)
    return fail(h, SLO_E_INVAL, "lookahead_step: bad arguments");
  if (sp->lambda_milli < 0 || sp->delta_micro < 0 || sp->viol_mult < 1 || sp->ema_beta_q16 > 65536 || sp->reserved)
    return fail(h, SLO_E_INVAL, "lookahead_step: bad score parameters");
  DeviceGuard g(h->device);
  slo::slo_lookahead_step_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(*space, *sp, (slo::LookTable*)d_table, d_aggs,
                                                                    n_parts, n_cand, d_state, d_traj);
  CUDA_TRY(h, cudaGetLastError());
  return SLO_OK;
}

// ---- peer exchange (NEXT-4) ----------------------------------------------------------------------
struct slo_exchange {
  slo_sim* h = nullptr;
  uint32_t world = 0, rank = 0, n_cfg = 0;
  char* window = nullptr;          // this rank's window (exported)
  size_t bytes = 0;
  slo::XState* st = nullptr;       // rank-local epoch / counters / error
  char** d_peers = nullptr;        // device copy of the window base of every rank
  char* h_peers[slo::kXMaxRanks] = {};
  bool opened = false;
};

slo_status slo_exchange_create(slo_sim* h, uint32_t world, uint32_t rank, uint32_t n_cfg, slo_exchange** out,
                               void* h_handle_out) {
  if (!h || !out || !h_handle_out || n_cfg == 0 || rank >= world) return fail(h, SLO_E_INVAL, "exchange_create: bad arguments");
  if (world < 2 || world > slo::kXMaxRanks) return fail(h, SLO_E_RANGE, "exchange_create: world must be in [2, %u]", slo::kXMaxRanks);
  *out = nullptr;
  DeviceGuard g(h->device);
  slo_exchange* x = new (std::nothrow) slo_exchange();
  if (!x) return fail(h, SLO_E_NOMEM, "exchange_create: host allocation");
  x->h = h;
  x->world = world;
  x->rank = rank;
  x->n_cfg = n_cfg;
  x->bytes = slo::kXHeader + (size_t)2 * world * n_cfg * sizeof(slo_config_agg);
  cudaError_t e;
  if ((e = cudaMalloc(&x->window, x->bytes)) != cudaSuccess || (e = cudaMalloc(&x->st, sizeof(slo::XState))) != cudaSuccess ||
      (e = cudaMalloc(&x->d_peers, sizeof(char*) * slo::kXMaxRanks)) != cudaSuccess) {
    slo_exchange_destroy(x);
    return fail(h, SLO_E_NOMEM, "exchange_create: cudaMalloc: %s", cudaGetErrorString(e));
  }
  cudaIpcMemHandle_t hd;
  if ((e = cudaMemset(x->window, 0, x->bytes)) != cudaSuccess || (e = cudaMemset(x->st, 0, sizeof(slo::XState))) != cudaSuccess ||
      (e = cudaIpcGetMemHandle(&hd, x->window)) != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess) {
    slo_exchange_destroy(x);
    return fail(h, SLO_E_CUDA, "exchange_create: %s", cudaGetErrorString(e));
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == SLO_EXCHANGE_HANDLE_BYTES, "IPC handle size");
  memcpy(h_handle_out, &hd, sizeof hd);
  *out = x;
  return SLO_OK;
}

slo_status slo_exchange_open(slo_exchange* x, const void* h_handles) {
  if (!x || !h_handles || x->opened) return fail(x ? x->h : nullptr, SLO_E_INVAL, "exchange_open: bad arguments");
  DeviceGuard g(x->h->device);
  const char* hb = static_cast<const char*>(h_handles);
  for (uint32_t r = 0; r < x->world; ++r) {
    if (r == x->rank) {
      x->h_peers[r] = x->window;
      continue;
    }
    cudaIpcMemHandle_t hd;
    memcpy(&hd, hb + (size_t)r * SLO_EXCHANGE_HANDLE_BYTES, sizeof hd);
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {       // unmap what this call mapped so a retry starts clean (no leaked mappings)
      for (uint32_t q = 0; q < r; ++q)
        if (q != x->rank && x->h_peers[q]) cudaIpcCloseMemHandle(x->h_peers[q]);
      for (uint32_t q = 0; q < x->world; ++q) x->h_peers[q] = nullptr;
      return fail(x->h, SLO_E_CUDA, "exchange_open: rank %u: %s", r, cudaGetErrorString(e));
    }
    x->h_peers[r] = static_cast<char*>(p);
  }
  CUDA_TRY(x->h, cudaMemcpy(x->d_peers, x->h_peers, sizeof(char*) * slo::kXMaxRanks, cudaMemcpyHostToDevice));
  x->opened = true;
  return SLO_OK;
}

slo_status slo_aggregate_exchange(slo_sim* h, slo_exchange* x, const slo_replica_result* d_detail, uint32_t n_seeds,
                                  slo_config_agg* d_pooled, void* stream) {
  if (!h || !x || !x->opened || x->h != h || !d_detail || !d_pooled || n_seeds == 0)
    return fail(h, SLO_E_INVAL, "aggregate_exchange: bad arguments (exchange opened on this handle?)");
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned threads = 256, warps = threads / 32;
  const unsigned pblocks = (unsigned)((x->n_cfg + warps - 1) / warps);
  slo::slo_aggregate_push_kernel<<<pblocks, threads, 0, st>>>(d_detail, x->n_cfg, n_seeds, x->d_peers, x->world,
                                                              x->rank, x->st);
  CUDA_TRY(h, cudaGetLastError());
  unsigned wblocks = (unsigned)((x->n_cfg + threads - 1) / threads);
  if (wblocks > (unsigned)h->sm_count) wblocks = (unsigned)h->sm_count;
  slo::slo_exchange_wait_kernel<<<wblocks, threads, 0, st>>>(x->window, x->n_cfg, x->world, x->st, d_pooled);
  CUDA_TRY(h, cudaGetLastError());
  return SLO_OK;
}

slo_status slo_pareto_front(slo_sim* h, const slo_config_agg* d_agg, uint32_t n_cfg, uint8_t* d_on_front,
                            uint32_t* d_count, void* stream) {
  if (!h || !d_agg || !d_on_front || n_cfg == 0) return fail(h, SLO_E_INVAL, "pareto_front: bad arguments");
  if (n_cfg >= (1u << 30)) return fail(h, SLO_E_RANGE, "pareto_front: n_cfg >= 2^30");
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  size_t cub_bytes = 0;
  const size_t need = slo::pareto_scratch_bytes(n_cfg, &cub_bytes);
  slo_status s;
  if ((s = ensure(h, h->d_pareto, h->pareto_cap, need, st)) != SLO_OK) return s;
  CUDA_TRY(h, slo::pareto_launch(d_agg, n_cfg, d_on_front, d_count, h->d_pareto, cub_bytes, st));
  return SLO_OK;
}

slo_status slo_philox_peak(slo_sim* h, uint32_t iters, uint32_t* d_sink, void* stream) {
  if (!h || !d_sink || iters == 0) return fail(h, SLO_E_INVAL, "philox_peak: bad arguments");
  DeviceGuard g(h->device);
  slo::slo_philox_peak_kernel<<<(unsigned)h->sm_count * 8u, 256, 0, (cudaStream_t)stream>>>(iters, d_sink);
  CUDA_TRY(h, cudaGetLastError());
  return SLO_OK;
}

slo_status slo_selftest_transforms(slo_sim* h, uint32_t what, uint32_t arg0, uint32_t arg1, uint32_t arg2,
                                   uint64_t* d_out, uint32_t out_len, void* stream) {
  if (!h || !d_out) return fail(h, SLO_E_INVAL, "selftest: null argument");
  slo::SelftestArgs a{};
  a.what = what;
  a.arg0 = arg0;
  a.arg1 = arg1;
  a.arg2 = arg2;
  uint32_t need = 0;
  switch (what) {
    case SLO_SELFTEST_EXP:
      need = 4097;
      break;
    case SLO_SELFTEST_LENGTH: {
      if (arg0 >= h->n_wl || arg1 > 1) return fail(h, SLO_E_INVAL, "selftest: bad workload / table");
      const slo::DevWorkload& w = h->h_wl[arg0];
      a.off = arg1 ? w.o_off : w.p_off;
      a.goff = arg1 ? w.o_goff : w.p_goff;
      a.lo = arg1 ? w.o_lo : w.p_lo;
      a.nbins = (arg1 ? w.o_ncw : w.p_ncw) + 1;
      a.viol_slot = a.nbins;
      need = a.nbins + 1;
      break;
    }
    case SLO_SELFTEST_ACCEPT:
    case SLO_SELFTEST_ACCEPT2:
      if (arg0 > 65536 || arg1 < 1 || arg1 > 4 || arg2 > 16) return fail(h, SLO_E_INVAL, "selftest: bad acceptance");
      a.nbins = 17;
      a.viol_slot = 17;
      need = 18;
      break;
    case SLO_SELFTEST_NOISE:
      if (arg0 > 1960) return fail(h, SLO_E_INVAL, "selftest: noise step > 1960");
      a.nbins = 1021;
      a.viol_slot = 1021;
      need = 1022;
      break;
    default:
      return fail(h, SLO_E_INVAL, "selftest: unknown what %u", what);
  }
  if (out_len < need) return fail(h, SLO_E_INVAL, "selftest: out_len %u < %u", out_len, need);
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(h, cudaMemsetAsync(d_out, 0, (size_t)need * sizeof(uint64_t), st));
  const size_t smem = (size_t)a.nbins * sizeof(uint32_t);
  slo::slo_selftest_kernel<<<4096, 256, smem, st>>>(a, h->d_tables, d_out);
  CUDA_TRY(h, cudaGetLastError());
  return SLO_OK;
}

slo_status slo_select_rows(slo_sim* h, const uint32_t* d_rows, uint32_t n_rows, uint32_t row_len,
                           const uint32_t* d_n_measured, uint32_t* d_p99_us, uint32_t* d_p50_us, uint32_t* d_p95_us,
                           void* stream) {
  if (!h || !d_rows || !d_p99_us || n_rows == 0 || row_len == 0)
    return fail(h, SLO_E_INVAL, "select_rows: null pointer or empty rows");
  if ((uint64_t)n_rows * row_len >= (1ull << 40)) return fail(h, SLO_E_RANGE, "select_rows: rows too large");
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  slo_status s;
  if ((s = ensure(h, h->d_part, h->part_cap, (size_t)n_rows, st)) != SLO_OK) return s;
  if ((s = ensure(h, h->d_sel_gp, h->sel_gp_cap, (size_t)n_rows, st)) != SLO_OK) return s;
  select_rows_part_kernel<<<(n_rows + 255) / 256, 256, 0, st>>>(h->d_part, n_rows, row_len, d_n_measured);
  CUDA_TRY(h, cudaGetLastError());
  slo::SimParams p{};
  p.lat = const_cast<uint32_t*>(d_rows);
  p.part = h->d_part;
  p.p99 = d_p99_us;
  p.p50 = d_p50_us;
  p.p95 = d_p95_us;
  p.goodput = h->d_sel_gp;
  p.n_rep = n_rows;
  p.n_seeds = 1;
  p.n_cfg = n_rows;
  p.r_base = 0;
  p.n_chunk = n_rows;
  p.warmup = 0;
  p.seg = row_len;
  const uint32_t thr = n_rows < (uint32_t)h->sm_count ? 256u : (uint32_t)sel_threads_for(row_len);
  const uint32_t wave = (uint32_t)h->sm_count * (uint32_t)h->sel_bps[thr == 64 ? 0 : (thr == 128 ? 1 : 2)];
  slo::slo_select_kernel<<<n_rows < wave ? n_rows : wave, thr, 0, st>>>(p);
  CUDA_TRY(h, cudaGetLastError());
  return SLO_OK;
}

slo_status slo_exchange_error(slo_exchange* x, uint32_t* h_err) {
  if (!x || !h_err) return fail(nullptr, SLO_E_INVAL, "exchange_error: null");
  DeviceGuard g(x->h->device);
  slo::XState s;
  CUDA_TRY(x->h, cudaMemcpy(&s, x->st, sizeof s, cudaMemcpyDeviceToHost));
  *h_err = s.error;
  return SLO_OK;
}

slo_status slo_exchange_destroy(slo_exchange* x) {
  if (!x) return SLO_OK;
  {
    DeviceGuard g(x->h->device);
    cudaDeviceSynchronize();
    for (uint32_t r = 0; r < x->world && x->opened; ++r)
      if (r != x->rank && x->h_peers[r]) cudaIpcCloseMemHandle(x->h_peers[r]);
    if (x->window) cudaFree(x->window);
    if (x->st) cudaFree(x->st);
    if (x->d_peers) cudaFree(x->d_peers);
  }
  delete x;
  return SLO_OK;
}

}  // extern "C\"
