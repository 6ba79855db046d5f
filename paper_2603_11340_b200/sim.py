"""Python face of libslosim.so: torch supplies device memory and streams; the library does all the work.

    from paper_2603_11340_b200 import inputs, sim
    s = sim.Simulator([inputs.preset_ll()])
    out = s.run_batch(sim.knobs_tensor(cfg.knobs), sim.seeds_tensor(cfg.seeds()), 10_000)
    out["p99_us"], out["goodput"]        # per replica (config-major)

Paper map: run_batch = the simulator segment + Eq. (1) goodput + empirical p99;
aggregate / hillclimb_step = Eq. (2)-(3) + Alg. 1.  Exact definitions: DESIGN.md §2.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Iterable, List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import (AGG_DTYPE, CLIMB_DTYPE, KNOB_DTYPE, RESULT_DTYPE, STATS_DTYPE, check, lib, slo_knobs,
                   slo_score_params, slo_space)

__all__ = ["Simulator", "pack_knobs", "knobs_tensor", "seeds_tensor", "neighbors", "space_struct",
           "score_struct", "unpack"]


# ------------------------------------------------------------------------------------------------
# packing helpers
# ------------------------------------------------------------------------------------------------
def pack_knobs(knobs: Sequence[Dict]) -> np.ndarray:
    arr = np.zeros(len(knobs), KNOB_DTYPE)
    for f in ("conc", "max_num_seqs", "draft_len", "spec_on", "draft_width", "workload", "rate_scale_q8",
              "accept_q16", "max_wait_us"):
        arr[f] = np.fromiter((k[f] for k in knobs), dtype=np.int64, count=len(knobs))
    for i, k in enumerate(knobs):
        if "reserved" in k:
            arr[i]["reserved"] = k["reserved"]
    return arr


def unpack_knobs(arr) -> List[Dict]:
    a = np.asarray(arr).view(KNOB_DTYPE).reshape(-1)
    return [dict(conc=int(x["conc"]), max_num_seqs=int(x["max_num_seqs"]), draft_len=int(x["draft_len"]),
                 spec_on=int(x["spec_on"]), draft_width=int(x["draft_width"]), workload=int(x["workload"]),
                 rate_scale_q8=int(x["rate_scale_q8"]), accept_q16=int(x["accept_q16"]),
                 max_wait_us=int(x["max_wait_us"])) for x in a]


def knobs_tensor(knobs, device="cuda") -> torch.Tensor:
    """uint8 [n, 32] tensor of slo_knobs records."""
    arr = knobs if isinstance(knobs, np.ndarray) else pack_knobs(knobs)
    t = torch.from_numpy(arr.view(np.uint8).reshape(-1, 32).copy())
    return t.to(device) if device != "cpu" else t


def seeds_tensor(seeds: Iterable[int], device="cuda") -> torch.Tensor:
    """int64 tensor holding the u64 seed bits."""
    a = np.array(list(seeds), dtype=np.uint64).view(np.int64)
    t = torch.from_numpy(a.copy())
    return t.to(device) if device != "cpu" else t


def unpack(t: torch.Tensor, dtype: np.dtype) -> np.ndarray:
    """Host numpy structured view of a byte tensor holding PODs."""
    return t.detach().cpu().contiguous().view(torch.uint8).numpy().view(dtype).reshape(-1)


def space_struct(space: Dict) -> slo_space:
    s = slo_space()
    s.stencil = space["stencil"]
    for d in range(5):
        s.lo[d], s.hi[d], s.step[d] = space["lo"][d], space["hi"][d], space["step"][d]
    return s


def score_struct(sp: Dict) -> slo_score_params:
    s = slo_score_params()
    defaults = dict(w_W_micro=0, w_k_micro=0, viol_mult=1, k_max=16, ema_beta_q16=0, reserved=0)
    for f, _ in slo_score_params._fields_:
        setattr(s, f, sp.get(f, defaults.get(f)))
    return s


def neighbors(space: Dict, K: Dict) -> List[Dict]:
    """Host-side neighbour list (same generator the climb kernel runs)."""
    k = pack_knobs([K])
    out = np.zeros(32, KNOB_DTYPE)
    n = C.c_uint32(0)
    check(lib().slo_neighbors(C.byref(space_struct(space)), k.ctypes.data, out.ctypes.data, 32, C.byref(n)))
    return unpack_knobs(out[: n.value])


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


# ------------------------------------------------------------------------------------------------
class Simulator:
    """One libslosim handle on one CUDA device."""

    def __init__(self, workloads: Sequence[Dict], device: Optional[int] = None, crn: int = 1,
                 warps_per_block: int = 0, blocks_per_sm: int = 0, scratch_mb: int = 0, group_policy: int = 0,
                 gen_policy: int = 0):
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        self.options = dict(crn=crn, warps_per_block=warps_per_block, blocks_per_sm=blocks_per_sm,
                            scratch_mb=scratch_mb, group_policy=group_policy, gen_policy=gen_policy)
        self.workloads = list(workloads)
        n = len(self.workloads)
        arr = (_lib.slo_workload * n)()
        self._keep = []
        for w, d in zip(arr, self.workloads):
            ar = d["arrivals"]
            w.arr.kind, w.arr.start_state = ar["kind"], ar["start_state"]
            for s in range(2):
                w.arr.mean_gap_q16[s] = ar["mean_gap_q16"][s]
                w.arr.mean_sojourn_us[s] = ar["mean_sojourn_us"][s]
            for name in ("prompt", "output"):
                cw = list(d[name]["cw"])
                buf = (C.c_uint32 * max(1, len(cw)))(*cw)
                self._keep.append(buf)
                setattr(w, name + "_cw", C.cast(buf, C.POINTER(C.c_uint32)))
                setattr(w, name + "_lo", d[name]["lo"])
                setattr(w, name + "_ncw", len(cw))
            for f, v in d["timing"].items():
                setattr(w.timing, f, v)
            w.stream_id = d["stream_id"]
            w.batching = d.get("batching", 0)
        opts = _lib.slo_sim_opts()
        opts.crn, opts.warps_per_block, opts.blocks_per_sm = crn, warps_per_block, blocks_per_sm
        opts.scratch_mb = scratch_mb
        opts.group_policy = group_policy
        opts.gen_policy = gen_policy
        h = C.c_void_p()
        check(lib().slo_sim_create(self.device, arr, n, C.byref(opts), C.byref(h)))
        self.h = h

    def twin(self) -> "Simulator":
        """A new handle on the same device with the same workloads and options (its own scratch)."""
        return Simulator(self.workloads, device=self.device, **self.options)

    def close(self):
        if getattr(self, "h", None):
            lib().slo_sim_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> Dict:
        i = _lib.slo_sim_info()
        check(lib().slo_sim_get_info(self.h, C.byref(i)), self.h)
        return {f: getattr(i, f) for f, _ in _lib.slo_sim_info._fields_ if f != "reserved"}

    # -------------------------------------------------------------------------------------------
    def alloc_outputs(self, n_rep: int, detail=True, latencies_n: int = 0, stats=False,
                      percentiles=False) -> Dict:
        dev = torch.device("cuda", self.device)
        out = dict(p99_us=torch.empty(n_rep, dtype=torch.int32, device=dev),
                   goodput=torch.empty(n_rep, dtype=torch.float64, device=dev))
        if percentiles:
            out["p50_us"] = torch.empty(n_rep, dtype=torch.int32, device=dev)
            out["p95_us"] = torch.empty(n_rep, dtype=torch.int32, device=dev)
        if detail:
            out["detail"] = torch.empty((n_rep, 32), dtype=torch.uint8, device=dev)
        if latencies_n:
            out["latencies"] = torch.empty(n_rep * latencies_n, dtype=torch.int32, device=dev)
        if stats:
            out["stats"] = torch.empty(64, dtype=torch.uint8, device=dev)
        return out

    def run_batch(self, configs: torch.Tensor, seeds: torch.Tensor, segment_len: int, warmup_len: int = 0,
                  slo_us: int = 1_200_000, detail: bool = True, latencies: bool = False, stats: bool = False,
                  percentiles: bool = False, out: Optional[Dict] = None, stream=None, stop_n_min: int = 0,
                  stop_t_min_us: int = 0, live_configs_ptr: int = 0) -> Dict:
        """K0/K1/K1b over n_configs x n_seeds replicas (config-major).  Asynchronous on `stream`."""
        n_cfg = configs.shape[0]
        n_seeds = seeds.shape[0]
        if out is None:
            out = self.alloc_outputs(n_cfg * n_seeds, detail, (segment_len + warmup_len) if latencies else 0, stats,
                                     percentiles)
        a = _lib.slo_run_args()
        a.d_configs, a.n_configs, a.d_seeds, a.n_seeds = configs.data_ptr(), n_cfg, seeds.data_ptr(), n_seeds
        a.segment_len, a.warmup_len, a.slo_us = segment_len, warmup_len, slo_us
        a.d_p99_us, a.d_goodput = out["p99_us"].data_ptr(), out["goodput"].data_ptr()
        a.d_detail, a.d_latencies, a.d_stats = _ptr(out.get("detail")), _ptr(out.get("latencies")), _ptr(out.get("stats"))
        a.d_p50_us, a.d_p95_us = _ptr(out.get("p50_us")), _ptr(out.get("p95_us"))
        a.stop_min_completions, a.stop_min_time_us = stop_n_min, stop_t_min_us
        a.d_live_configs = live_configs_ptr or None     # device u32: only configs [0, value) simulated
        check(lib().slo_sim_run(self.h, C.byref(a), _stream_ptr(stream)), self.h)
        return out

    def run_batch_host(self, h_configs: np.ndarray, h_seeds: np.ndarray, segment_len: int, warmup_len: int = 0,
                       slo_us: int = 1_200_000, out: Optional[Dict] = None, detail: bool = False,
                       stats: bool = False, stream=None) -> Dict:
        """The end-to-end call on host buffers (pinned torch CPU tensors recommended); synchronous."""
        n_cfg = h_configs.shape[0]
        n_seeds = h_seeds.shape[0]
        R = n_cfg * n_seeds
        if out is None:
            pin = torch.cuda.is_available()
            out = dict(p99_us=torch.empty(R, dtype=torch.int32, pin_memory=pin),
                       goodput=torch.empty(R, dtype=torch.float64, pin_memory=pin))
            if detail:
                out["detail"] = torch.empty((R, 32), dtype=torch.uint8, pin_memory=pin)
            if stats:
                out["stats"] = torch.empty(64, dtype=torch.uint8, pin_memory=pin)
        check(lib().slo_sim_run_batch_host(self.h, h_configs.data_ptr(), n_cfg, h_seeds.data_ptr(), n_seeds,
                                           segment_len, warmup_len, slo_us, out["p99_us"].data_ptr(),
                                           out["goodput"].data_ptr(), _ptr(out.get("detail")),
                                           _ptr(out.get("stats")), _stream_ptr(stream)), self.h)
        return out

    def aggregate(self, detail: torch.Tensor, n_configs: int, n_seeds: int, out: Optional[torch.Tensor] = None,
                  stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty((n_configs, 32), dtype=torch.uint8, device=detail.device)
        check(lib().slo_aggregate(self.h, detail.data_ptr(), n_configs, n_seeds, out.data_ptr(),
                                  _stream_ptr(stream)), self.h)
        return out

    def aggregate_reduce(self, parts: torch.Tensor, n_parts: int, n_configs: int,
                         out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty((n_configs, 32), dtype=torch.uint8, device=parts.device)
        check(lib().slo_aggregate_reduce(self.h, parts.data_ptr(), n_parts, n_configs, out.data_ptr(),
                                         _stream_ptr(stream)), self.h)
        return out

    # ---- NEXT-4 peer exchange (include/slo_sim.h: slo_exchange_*) -------------------------------
    def exchange_create(self, world: int, rank: int, n_cfg: int):
        """This rank's exchange window; returns (opaque handle, 64-byte CUDA IPC handle as bytes)."""
        x = C.c_void_p()
        hbuf = (C.c_uint8 * _lib.EXCHANGE_HANDLE_BYTES)()
        check(lib().slo_exchange_create(self.h, world, rank, n_cfg, C.byref(x), hbuf), self.h)
        return x, bytes(hbuf)

    def exchange_open(self, x, handles: bytes) -> None:
        buf = (C.c_uint8 * len(handles)).from_buffer_copy(handles)
        check(lib().slo_exchange_open(x, buf), self.h)

    def aggregate_exchange(self, x, detail: torch.Tensor, n_seeds: int, out: torch.Tensor, stream=None) -> torch.Tensor:
        """K2x + K2w: per-config aggregates pooled over all ranks, pushed through the peers' windows."""
        check(lib().slo_aggregate_exchange(self.h, x, detail.data_ptr(), n_seeds, out.data_ptr(),
                                           _stream_ptr(stream)), self.h)
        return out

    def pareto_front(self, agg: torch.Tensor, count: bool = False, stream=None):
        """K5: uint8 [n_cfg] on-front flags of the per-config aggregates (min mean p99, max goodput)."""
        n = agg.shape[0]
        front = torch.empty(n, dtype=torch.uint8, device=agg.device)
        cnt = torch.zeros(1, dtype=torch.int32, device=agg.device) if count else None
        check(lib().slo_pareto_front(self.h, agg.data_ptr(), n, front.data_ptr(), _ptr(cnt), _stream_ptr(stream)),
              self.h)
        return (front, cnt) if count else front

    def profile(self, enable: bool = True) -> None:
        """Record per-kernel CUDA events around every later run (slo_sim_profile)."""
        check(lib().slo_sim_profile(self.h, 1 if enable else 0), self.h)

    def profile_read(self) -> Dict:
        """Summed ms of the recorded runs: K0, K1g, the chain kernels, K1b and the simulation wall time (K1g and
        the chains overlap when pipelined), and the chunk count; clears them."""
        ms = (C.c_double * 5)()
        n = C.c_uint32(0)
        check(lib().slo_sim_profile_read(self.h, ms, C.byref(n)), self.h)
        return {"k0_ms": ms[0], "gen_ms": ms[1], "sim_ms": ms[2], "k1b_ms": ms[3], "wall_ms": ms[4], "chunks": n.value}

    def selftest(self, what: str, arg0: int = 0, arg1: int = 0, arg2: int = 0, stream=None) -> np.ndarray:
        """K6: exhaustive 2^32-input hashes / histograms of a transform (slo_selftest_transforms), as uint64."""
        from ._lib import SELFTEST
        out = torch.empty(8192, dtype=torch.int64, device=torch.device("cuda", self.device))
        check(lib().slo_selftest_transforms(self.h, SELFTEST[what], arg0, arg1, arg2, out.data_ptr(), out.numel(),
                                            _stream_ptr(stream)), self.h)
        torch.cuda.synchronize(self.device)
        return out.cpu().numpy().view(np.uint64)

    def select_rows(self, rows: torch.Tensor, n_measured: Optional[torch.Tensor] = None, percentiles: bool = False,
                    stream=None) -> Dict:
        """K1b on caller rows (slo_select_rows): nearest-rank p99 (and p50/p95) of each row of a contiguous
        [n_rows, row_len] int32/uint32 device tensor.  Asynchronous on `stream`."""
        assert rows.dim() == 2 and rows.is_contiguous() and rows.element_size() == 4
        n_rows, row_len = rows.shape
        dev = rows.device
        out = {"p99_us": torch.empty(n_rows, dtype=torch.int32, device=dev)}
        if percentiles:
            out["p50_us"] = torch.empty(n_rows, dtype=torch.int32, device=dev)
            out["p95_us"] = torch.empty(n_rows, dtype=torch.int32, device=dev)
        check(lib().slo_select_rows(self.h, rows.data_ptr(), n_rows, row_len, _ptr(n_measured),
                                    out["p99_us"].data_ptr(), _ptr(out.get("p50_us")), _ptr(out.get("p95_us")),
                                    _stream_ptr(stream)), self.h)
        return out

    def philox_peak(self, iters: int = 2048, repeats: int = 3) -> float:
        """K4: measured Philox4x32-10 blocks/s at full occupancy (the RNG roofline)."""
        sm = self.info()["sm_count"]
        sink = torch.empty(sm * 2048, dtype=torch.int32, device=torch.device("cuda", self.device))
        st = torch.cuda.current_stream()
        check(lib().slo_philox_peak(self.h, iters, sink.data_ptr(), _stream_ptr(st)), self.h)   # warm-up
        best = 0.0
        for _ in range(repeats):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            check(lib().slo_philox_peak(self.h, iters, sink.data_ptr(), _stream_ptr(st)), self.h)
            e1.record(st)
            e1.synchronize()
            best = max(best, sm * 2048 * iters / (e0.elapsed_time(e1) / 1000.0))
        return best

    def exchange_error(self, x) -> int:
        e = C.c_uint32(0)
        check(lib().slo_exchange_error(x, C.byref(e)), self.h)
        return e.value

    def exchange_destroy(self, x) -> None:
        lib().slo_exchange_destroy(x)

    def climb_state(self, K0: Dict) -> torch.Tensor:
        st = np.zeros(1, CLIMB_DTYPE)
        k = pack_knobs([K0])[0]
        st[0]["K"] = k
        st[0]["K_best"] = k
        st[0]["S_best_micro"] = -(1 << 63)
        return torch.from_numpy(st.view(np.uint8).copy()).to(torch.device("cuda", self.device))

    def candidates(self, space: Dict, K: Dict, n_cand: int) -> torch.Tensor:
        """[K, neighbours(K), padding] as a device uint8 [n_cand, 32] tensor (the climb's first step)."""
        from .inputs import PAD_KNOBS
        nb = neighbors(space, K)[: n_cand - 1]
        cands = [K] + nb + [PAD_KNOBS] * (n_cand - 1 - len(nb))
        return knobs_tensor(cands, device=torch.device("cuda", self.device))

    def lookahead_prepare(self, space: Dict, state: torch.Tensor, table: torch.Tensor, sim_list: torch.Tensor,
                          stream=None) -> None:
        """Lookahead climb round, part 1 (slo_lookahead_prepare): U(K) minus the cache -> sim_list."""
        check(lib().slo_lookahead_prepare(self.h, C.byref(space_struct(space)), state.data_ptr(), table.data_ptr(),
                                          sim_list.data_ptr(), _stream_ptr(stream)), self.h)

    def lookahead_step(self, space: Dict, sp: Dict, table: torch.Tensor, aggs: torch.Tensor, n_parts: int,
                       n_cand: int, state: torch.Tensor, traj: torch.Tensor, stream=None) -> None:
        """Lookahead climb round, part 2 (slo_lookahead_step): two Alg. 1 steps from U's aggregates."""
        check(lib().slo_lookahead_step(self.h, C.byref(space_struct(space)), C.byref(score_struct(sp)),
                                       table.data_ptr(), aggs.data_ptr(), n_parts, n_cand, state.data_ptr(),
                                       traj.data_ptr(), _stream_ptr(stream)), self.h)

    def hillclimb_step(self, space: Dict, sp: Dict, cands: torch.Tensor, aggs: torch.Tensor, n_parts: int,
                       state: torch.Tensor, scores: Optional[torch.Tensor] = None, stream=None) -> None:
        """K3: Alg. 1 step on the device; rewrites `cands` in place with the next candidate list."""
        n_cand = cands.shape[0]
        check(lib().slo_hillclimb_step(self.h, C.byref(space_struct(space)), C.byref(score_struct(sp)),
                                       cands.data_ptr(), n_cand, aggs.data_ptr(), n_parts, state.data_ptr(),
                                       _ptr(scores), _stream_ptr(stream)), self.h)
