"""ctypes binding of libslosim.so (include/slo_sim.h) — argument marshalling only.

Every step of the simulation, aggregation and climb runs in the library's CUDA kernels; this module only
mirrors the C structs and loads the library.  There is no CPU fallback: if libslosim.so is missing or
cannot be loaded, `lib()` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SLO_SIM_LIB") or os.path.join(HERE, "libslosim.so")   # env: experiment builds (in-tree)

SLO_OK = 0
STATUS = {0: "ok", -1: "SLO_E_INVAL", -2: "SLO_E_NOMEM", -3: "SLO_E_CUDA", -4: "SLO_E_RANGE",
          -5: "SLO_E_DEVICE", -6: "SLO_E_UNSUPPORTED"}

# symbols include/slo_sim.h declares (checked by tests/test_abi_cpu.py)
EXPORTS = ("slo_sim_create", "slo_sim_destroy", "slo_sim_get_info", "slo_sim_run", "slo_sim_run_batch",
           "slo_sim_run_batch_host", "slo_aggregate", "slo_aggregate_reduce", "slo_neighbors",
           "slo_hillclimb_step", "slo_exchange_create", "slo_exchange_open", "slo_aggregate_exchange",
           "slo_exchange_error", "slo_exchange_destroy", "slo_philox_peak", "slo_pareto_front", "slo_status_string",
           "slo_last_error", "slo_selftest_transforms", "slo_sim_profile", "slo_sim_profile_read", "slo_select_rows",
           "slo_lookahead_prepare", "slo_lookahead_step")
SELFTEST = {"exp": 0, "length": 1, "accept": 2, "noise": 3, "accept2": 4}   # SLO_SELFTEST_* (include/slo_sim.h)
EXCHANGE_HANDLE_BYTES = 64


class SloError(RuntimeError):
    def __init__(self, status, detail=""):
        super().__init__(f"{STATUS.get(status, status)}: {detail}")
        self.status = status


class slo_timing(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("pre_base_us", "pre_tok_us", "dec_base_us", "dec_seq_us",
                                          "dr_base_us", "dr_seq_us", "ver_base_us", "ver_seq_us",
                                          "ver_tok_us", "noise_step_ppm")]


class slo_arrivals(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("start_state", C.c_uint32), ("mean_gap_q16", C.c_uint64 * 2),
                ("mean_sojourn_us", C.c_uint64 * 2)]


class slo_workload(C.Structure):
    _fields_ = [("arr", slo_arrivals),
                ("prompt_cw", C.POINTER(C.c_uint32)), ("prompt_lo", C.c_uint32), ("prompt_ncw", C.c_uint32),
                ("output_cw", C.POINTER(C.c_uint32)), ("output_lo", C.c_uint32), ("output_ncw", C.c_uint32),
                ("timing", slo_timing), ("stream_id", C.c_uint32), ("batching", C.c_uint32)]


class slo_sim_opts(C.Structure):
    _fields_ = [("crn", C.c_uint32), ("warps_per_block", C.c_uint32), ("blocks_per_sm", C.c_uint32),
                ("scratch_mb", C.c_uint32), ("group_policy", C.c_uint32), ("gen_policy", C.c_uint32),
                ("reserved", C.c_uint32 * 2)]


class slo_sim_info(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("device", "sm_count", "warps_per_block", "blocks_per_sm",
                                         "regs_per_thread", "smem_per_warp_bytes")] + [("reserved", C.c_int32 * 2)]


class slo_knobs(C.Structure):
    _fields_ = [("conc", C.c_uint8), ("max_num_seqs", C.c_uint8), ("draft_len", C.c_uint8),
                ("spec_on", C.c_uint8), ("draft_width", C.c_uint8), ("workload", C.c_uint8),
                ("rate_scale_q8", C.c_uint16), ("accept_q16", C.c_uint32), ("max_wait_us", C.c_uint32),
                ("reserved", C.c_uint32 * 4)]


class slo_run_args(C.Structure):
    _fields_ = [("d_configs", C.c_void_p), ("n_configs", C.c_uint32), ("d_seeds", C.c_void_p),
                ("n_seeds", C.c_uint32), ("segment_len", C.c_uint32), ("warmup_len", C.c_uint32),
                ("slo_us", C.c_uint32), ("d_p99_us", C.c_void_p), ("d_goodput", C.c_void_p),
                ("d_detail", C.c_void_p), ("d_latencies", C.c_void_p), ("d_stats", C.c_void_p),
                ("d_p50_us", C.c_void_p), ("d_p95_us", C.c_void_p), ("stop_min_completions", C.c_uint32),
                ("stop_min_time_us", C.c_uint32), ("d_live_configs", C.c_void_p)]


class slo_space(C.Structure):
    _fields_ = [("stencil", C.c_uint32), ("lo", C.c_int32 * 5), ("hi", C.c_int32 * 5), ("step", C.c_int32 * 5)]


class slo_score_params(C.Structure):
    _fields_ = [("lambda_milli", C.c_int64), ("w_conc_micro", C.c_int64), ("w_max_micro", C.c_int64),
                ("w_spec_micro", C.c_int64), ("delta_micro", C.c_int64), ("slo_us", C.c_uint32),
                ("strict_alg1", C.c_uint32), ("w_W_micro", C.c_int64), ("w_k_micro", C.c_int64),
                ("viol_mult", C.c_uint32), ("k_max", C.c_uint32), ("ema_beta_q16", C.c_uint32),
                ("reserved", C.c_uint32)]


# numpy views of the 32-byte PODs (little-endian)
KNOB_DTYPE = np.dtype([("conc", "u1"), ("max_num_seqs", "u1"), ("draft_len", "u1"), ("spec_on", "u1"),
                       ("draft_width", "u1"), ("workload", "u1"), ("rate_scale_q8", "<u2"),
                       ("accept_q16", "<u4"), ("max_wait_us", "<u4"), ("reserved", "<u4", (4,))])
RESULT_DTYPE = np.dtype([("p99_us", "<u4"), ("slo_met", "<u4"), ("n_measured", "<u4"), ("flags", "<u4"),
                         ("window_us", "<u8"), ("sum_latency_us", "<u8")])
AGG_DTYPE = np.dtype([("sum_p99_us", "<u8"), ("sum_slo_met", "<u8"), ("sum_window_us", "<u8"),
                      ("n_seeds", "<u4"), ("flags", "<u4")])
STATS_DTYPE = np.dtype([("requests", "<u8"), ("batches", "<u8"), ("decode_steps", "<u8"),
                        ("member_steps", "<u8"), ("philox_blocks", "<u8"), ("replicas", "<u8"),
                        ("reserved", "<u8", (2,))])
CLIMB_DTYPE = np.dtype([("K", KNOB_DTYPE), ("K_best", KNOB_DTYPE), ("S_best_micro", "<i8"), ("step", "<u4"),
                        ("has_best", "<u4"), ("moved", "<i4"), ("argmax", "<u4"), ("n_next", "<u4"),
                        ("has_ema", "<u4"), ("ema_p99_us", "<u8")])
assert KNOB_DTYPE.itemsize == 32 and RESULT_DTYPE.itemsize == 32 and AGG_DTYPE.itemsize == 32
assert STATS_DTYPE.itemsize == 64 and CLIMB_DTYPE.itemsize == 104

_lib = None
vp = C.c_void_p


def lib():
    """Load libslosim.so (built in-tree by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.slo_sim_create.argtypes = [C.c_int, C.POINTER(slo_workload), C.c_uint32, C.POINTER(slo_sim_opts),
                                     C.POINTER(vp)]
        L.slo_sim_destroy.argtypes = [vp]
        L.slo_sim_get_info.argtypes = [vp, C.POINTER(slo_sim_info)]
        L.slo_sim_run.argtypes = [vp, C.POINTER(slo_run_args), vp]
        L.slo_sim_run_batch.argtypes = [vp, vp, C.c_uint32, vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                        vp, vp, vp, vp, vp, vp]
        L.slo_sim_run_batch_host.argtypes = [vp, vp, C.c_uint32, vp, C.c_uint32, C.c_uint32, C.c_uint32,
                                             C.c_uint32, vp, vp, vp, vp, vp]
        L.slo_aggregate.argtypes = [vp, vp, C.c_uint32, C.c_uint32, vp, vp]
        L.slo_aggregate_reduce.argtypes = [vp, vp, C.c_uint32, C.c_uint32, vp, vp]
        L.slo_neighbors.argtypes = [C.POINTER(slo_space), vp, vp, C.c_uint32, C.POINTER(C.c_uint32)]
        L.slo_hillclimb_step.argtypes = [vp, C.POINTER(slo_space), C.POINTER(slo_score_params), vp, C.c_uint32,
                                         vp, C.c_uint32, vp, vp, vp]
        L.slo_exchange_create.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(vp), vp]
        L.slo_exchange_open.argtypes = [vp, vp]
        L.slo_aggregate_exchange.argtypes = [vp, vp, vp, C.c_uint32, vp, vp]
        L.slo_exchange_error.argtypes = [vp, C.POINTER(C.c_uint32)]
        L.slo_exchange_destroy.argtypes = [vp]
        L.slo_philox_peak.argtypes = [vp, C.c_uint32, vp, vp]
        L.slo_pareto_front.argtypes = [vp, vp, C.c_uint32, vp, vp, vp]
        L.slo_sim_profile.argtypes = [vp, C.c_uint32]
        L.slo_sim_profile_read.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_uint32)]
        L.slo_selftest_transforms.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, vp, C.c_uint32, vp]
        L.slo_select_rows.argtypes = [vp, vp, C.c_uint32, C.c_uint32, vp, vp, vp, vp, vp]
        L.slo_lookahead_prepare.argtypes = [vp, C.POINTER(slo_space), vp, vp, vp, vp]
        L.slo_lookahead_step.argtypes = [vp, C.POINTER(slo_space), C.POINTER(slo_score_params), vp, vp, C.c_uint32,
                                         C.c_uint32, vp, vp, vp]
        L.slo_status_string.argtypes = [C.c_int32]
        L.slo_status_string.restype = C.c_char_p
        L.slo_last_error.argtypes = [vp]
        L.slo_last_error.restype = C.c_char_p
        for name in EXPORTS:
            if name not in ("slo_status_string", "slo_last_error"):
                getattr(L, name).restype = C.c_int32
        _lib = L
    return _lib


def check(status, handle=None):
    if status != SLO_OK:
        detail = lib().slo_last_error(handle)
        raise SloError(status, detail.decode() if detail else "")
