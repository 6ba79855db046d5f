"""oracle — TEST INFRASTRUCTURE ONLY.

The plain CPU oracle of the SLO-Tuner serving simulator (arXiv 2603.11340 §2.2) and of
its scoring / hill-climb (Eq. 1-3, Alg. 1), written from DESIGN.md §2.  It shares no
code with the CUDA path (paper_2603_11340_b200/csrc); only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import it.

Pins (tests/test_oracle_*.py):
  * Philox4x32-10 — Random123 known-answer vectors (tests/golden/philox_kat.txt);
  * E_q — bound vs libm -ln over a dense sample, mean = 1, exact at powers of two;
  * lengths / thresholds / noise — exact counting identities and Leviathan's closed form;
  * event loop — hand traces T1-T5 (tests/golden/traces.json), an independent per-microsecond brute-force
    simulator on small random traces, the Lindley recursion at B = 1 (textbook special case),
    Pollaczek-Khinchine M/D/1 mean wait (statistical), conservation / gate / FCFS invariants;
  * p99 / goodput — SPEC nearest-rank examples and S:135-136;
  * score / neighbours / move — S:73-75, S:201-202, S:210, S:278-280 (oracle/climb.py);
  * Pareto front — the O(n^2) definition (oracle/pareto.py): hand example, floors, front properties.
Parity unpinned: absolute paper simulator values (calibration unpublished).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libslo_oracle.so")


def build(force: bool = False) -> str:
    """Compile the C oracle (plain gcc, -O2, no fast-math)."""
    src = os.path.join(_HERE, "slo_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "slo_oracle.h"))):
        import subprocess
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-fPIC", "-shared",
                               "-o", _LIB_PATH, src])
    return _LIB_PATH


class Arrivals(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("start_state", C.c_uint32),
                ("mean_gap_q16", C.c_uint64 * 2), ("mean_sojourn_us", C.c_uint64 * 2)]


class Timing(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("pre_base_us", "pre_tok_us", "dec_base_us", "dec_seq_us",
                                          "dr_base_us", "dr_seq_us", "ver_base_us", "ver_seq_us",
                                          "ver_tok_us", "noise_step_ppm")]


class Workload(C.Structure):
    _fields_ = [("arr", Arrivals),
                ("prompt_cw", C.POINTER(C.c_uint32)), ("prompt_lo", C.c_uint32), ("prompt_ncw", C.c_uint32),
                ("output_cw", C.POINTER(C.c_uint32)), ("output_lo", C.c_uint32), ("output_ncw", C.c_uint32),
                ("timing", Timing), ("stream_id", C.c_uint32), ("batching", C.c_uint32)]


class Knobs(C.Structure):
    _fields_ = [("conc", C.c_uint8), ("max_num_seqs", C.c_uint8), ("draft_len", C.c_uint8),
                ("spec_on", C.c_uint8), ("draft_width", C.c_uint8), ("workload", C.c_uint8),
                ("rate_scale_q8", C.c_uint16), ("accept_q16", C.c_uint32), ("max_wait_us", C.c_uint32),
                ("reserved", C.c_uint32 * 4)]


class Result(C.Structure):
    _fields_ = [("p99_us", C.c_uint32), ("slo_met", C.c_uint32), ("n_measured", C.c_uint32),
                ("flags", C.c_uint32), ("window_us", C.c_uint64), ("sum_latency_us", C.c_uint64),
                ("goodput", C.c_double), ("p50_us", C.c_uint32), ("p95_us", C.c_uint32)]


class Counters(C.Structure):
    _fields_ = [("philox_blocks", C.c_uint64), ("batches", C.c_uint64), ("decode_steps", C.c_uint64),
                ("member_steps", C.c_uint64)]


class Req(C.Structure):
    _fields_ = [("a", C.c_uint64), ("s", C.c_uint64), ("form", C.c_uint64), ("c", C.c_uint64),
                ("batch", C.c_uint32), ("steps", C.c_uint32), ("P", C.c_uint32), ("O", C.c_uint32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = build()
        L = C.CDLL(path)
        L.orc_philox4x32_10.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.orc_exp_q32.argtypes = [C.c_uint32]
        L.orc_exp_q32.restype = C.c_uint64
        L.orc_length.argtypes = [C.POINTER(C.c_uint32), C.c_uint32, C.c_uint32, C.c_uint32]
        L.orc_length.restype = C.c_uint32
        L.orc_thresholds.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64)]
        L.orc_thresholds.restype = C.c_uint32
        L.orc_noise_factor.argtypes = [C.c_uint32, C.c_uint32]
        L.orc_noise_factor.restype = C.c_uint32
        L.orc_phases.argtypes = [C.POINTER(Workload), C.POINTER(Knobs), C.c_uint64, C.c_uint32, C.c_uint32,
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_uint32)]
        L.orc_fnv1a_knobs.argtypes = [C.POINTER(Knobs)]
        L.orc_fnv1a_knobs.restype = C.c_uint32
        L.orc_knobs_valid.argtypes = [C.POINTER(Knobs), C.c_uint32]
        L.orc_request_draws.argtypes = [C.POINTER(Workload), C.POINTER(Knobs), C.c_uint64, C.c_uint32,
                                        C.c_uint32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32),
                                        C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.orc_run.argtypes = [C.POINTER(Workload), C.c_uint32, C.POINTER(Knobs), C.c_uint64, C.c_uint32,
                              C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(Result),
                              C.POINTER(C.c_uint32), C.POINTER(Req), C.POINTER(Counters)]
        L.orc_run_stop.argtypes = [C.POINTER(Workload), C.c_uint32, C.POINTER(Knobs), C.c_uint64, C.c_uint32,
                                   C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(Result),
                                   C.POINTER(C.c_uint32), C.POINTER(Req), C.POINTER(Counters)]
        L.orc_run_trace_stop.argtypes = [C.POINTER(Timing), C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                         C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.c_uint32, C.c_uint32,
                                         C.c_uint32, C.c_uint32, C.POINTER(Result), C.POINTER(C.c_uint32),
                                         C.POINTER(Req), C.POINTER(Counters)]
        L.orc_run_trace.argtypes = [C.POINTER(Timing), C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32),
                                    C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                    C.POINTER(C.c_uint32), C.c_uint32, C.c_uint32, C.POINTER(Result),
                                    C.POINTER(C.c_uint32), C.POINTER(Req), C.POINTER(Counters)]
        _lib = L
    return _lib


# ------------------------------------------------------------------------------------------------
# marshalling of the plain-dict inputs (paper_2603_11340_b200.inputs)
# ------------------------------------------------------------------------------------------------
class _WorkloadSet:
    """Keeps the ctypes arrays alive for the duration of the calls."""

    def __init__(self, workloads: Sequence[Dict]):
        self.n = len(workloads)
        self.arr = (Workload * self.n)()
        self._keep = []
        for w, d in zip(self.arr, workloads):
            ar = d["arrivals"]
            w.arr.kind = ar["kind"]
            w.arr.start_state = ar["start_state"]
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
            for k, v in d["timing"].items():
                setattr(w.timing, k, v)
            w.stream_id = d["stream_id"]
            w.batching = d.get("batching", 0)


def make_knobs(d: Dict) -> Knobs:
    k = Knobs()
    for name in ("conc", "max_num_seqs", "draft_len", "spec_on", "draft_width", "workload",
                 "rate_scale_q8", "accept_q16", "max_wait_us"):
        setattr(k, name, d[name])
    for i, v in enumerate(d.get("reserved", [0, 0, 0, 0])):
        k.reserved[i] = v
    return k


def philox(ctr: Sequence[int], key: Sequence[int]) -> List[int]:
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return list(o)


def exp_q32(u: int) -> int:
    return lib().orc_exp_q32(u)


def length(table: Dict, u: int) -> int:
    cw = list(table["cw"])
    buf = (C.c_uint32 * max(1, len(cw)))(*cw)
    return lib().orc_length(buf, len(cw), table["lo"], u)


def thresholds(accept_q16: int, width: int, gamma: int):
    T = (C.c_uint64 * 16)()
    ae = lib().orc_thresholds(accept_q16, width, gamma, T)
    return ae, list(T)[:gamma]


def noise_factor(w: int, step_ppm: int) -> int:
    return lib().orc_noise_factor(w, step_ppm)


def phases(workloads: Sequence[Dict], knobs: Dict, seed: int, n: int, crn: int = 1):
    """The first n bursty phases of a replica: (start, D, U, state) arrays."""
    ws = _WorkloadSet(workloads)
    k = make_knobs(knobs)
    st = np.zeros(n, np.uint64)
    D = np.zeros(n, np.uint64)
    U = np.zeros(n, np.uint64)
    s = np.zeros(n, np.uint32)
    rc = lib().orc_phases(ws.arr, C.byref(k), seed, crn, n, st.ctypes.data_as(C.POINTER(C.c_uint64)),
                          D.ctypes.data_as(C.POINTER(C.c_uint64)), U.ctypes.data_as(C.POINTER(C.c_uint64)),
                          s.ctypes.data_as(C.POINTER(C.c_uint32)))
    if rc != 0:
        raise ValueError("orc_phases: not a bursty arrival kind")
    return st, D, U, s


def fnv1a_knobs(d: Dict) -> int:
    k = make_knobs(d)
    return lib().orc_fnv1a_knobs(C.byref(k))


def knobs_valid(d: Dict, n_wl: int = 1) -> bool:
    k = make_knobs(d)
    return bool(lib().orc_knobs_valid(C.byref(k), n_wl))


def request_draws(workloads: Sequence[Dict], knobs: Dict, seed: int, n: int, crn: int = 1):
    ws = _WorkloadSet(workloads)
    k = make_knobs(knobs)
    a = np.zeros(n, np.uint64)
    P = np.zeros(n, np.uint32)
    O = np.zeros(n, np.uint32)
    w3 = np.zeros(n, np.uint32)
    lib().orc_request_draws(ws.arr, C.byref(k), seed, crn, n,
                            a.ctypes.data_as(C.POINTER(C.c_uint64)), P.ctypes.data_as(C.POINTER(C.c_uint32)),
                            O.ctypes.data_as(C.POINTER(C.c_uint32)), w3.ctypes.data_as(C.POINTER(C.c_uint32)))
    return a, P, O, w3


def _pack(res: Result, cnt: Counters, lat, trace) -> Dict:
    out = dict(p99_us=res.p99_us, slo_met=res.slo_met, n_measured=res.n_measured, flags=res.flags,
               window_us=res.window_us, sum_latency_us=res.sum_latency_us, goodput=res.goodput,
               p50_us=res.p50_us, p95_us=res.p95_us,
               counters=dict(philox_blocks=cnt.philox_blocks, batches=cnt.batches,
                             decode_steps=cnt.decode_steps, member_steps=cnt.member_steps))
    if lat is not None:
        out["latencies"] = lat
    if trace is not None:
        out["trace"] = {f: np.array([getattr(r, f) for r in trace]) for f, _ in Req._fields_}
    return out


def run(workloads: Sequence[Dict], knobs: Dict, seed: int, segment_len: int, warmup_len: int = 0,
        slo_us: int = 1_200_000, crn: int = 1, latencies: bool = False, trace: bool = False,
        stop_n_min: int = 0, stop_t_min_us: int = 0) -> Dict:
    """One replica in Philox mode (with a segment stop rule, §2.14)."""
    ws = _WorkloadSet(workloads)
    k = make_knobs(knobs)
    N = segment_len + warmup_len
    res, cnt = Result(), Counters()
    lat = np.zeros(N, np.uint32) if latencies else None
    tr = (Req * N)() if trace else None
    rc = lib().orc_run_stop(ws.arr, ws.n, C.byref(k), seed, crn, segment_len, warmup_len, slo_us, stop_n_min,
                            stop_t_min_us, C.byref(res),
                            lat.ctypes.data_as(C.POINTER(C.c_uint32)) if lat is not None else None,
                            tr, C.byref(cnt))
    if rc != 0:
        raise ValueError(f"orc_run failed: {rc}")
    return _pack(res, cnt, lat, tr)


def run_trace(timing: Dict, conc: int, max_num_seqs: int, gamma: int, max_wait_us: int,
              a: Sequence[int], P: Sequence[int], O: Sequence[int], f: Optional[Sequence[int]] = None,
              A: Optional[Sequence[Sequence[int]]] = None, warmup_len: int = 0, slo_us: int = 1_200_000,
              issue_origin: int = 0, continuous: int = 0, stop_n_min: int = 0, stop_t_min_us: int = 0,
              width: int = 1) -> Dict:
    """Trace mode: explicit requests (a, P, O), per-request noise factor f (ppm) and accepted-prefix draws;
    `width` = draft width W in the speculative step cost (R28)."""
    n = len(a)
    tm = Timing(**timing)
    a_ = (C.c_uint64 * n)(*a)
    P_ = (C.c_uint32 * n)(*P)
    O_ = (C.c_uint32 * n)(*O)
    f_ = (C.c_uint32 * n)(*(f if f is not None else [1_000_000] * n))
    A = A if A is not None else [[] for _ in range(n)]
    off = [0]
    vals = []
    for row in A:
        vals.extend(row)
        off.append(len(vals))
    off_ = (C.c_uint32 * (n + 1))(*off)
    val_ = (C.c_uint32 * max(1, len(vals)))(*vals)
    res, cnt = Result(), Counters()
    lat = np.zeros(n, np.uint32)
    tr = (Req * n)()
    rc = lib().orc_run_trace_stop(C.byref(tm), conc, max_num_seqs, gamma, width, max_wait_us, issue_origin, continuous, n,
                                  a_, P_, O_, f_, off_, val_, warmup_len, slo_us, stop_n_min, stop_t_min_us,
                                  C.byref(res), lat.ctypes.data_as(C.POINTER(C.c_uint32)), tr, C.byref(cnt))
    if rc != 0:
        raise ValueError(f"orc_run_trace failed: {rc}")
    return _pack(res, cnt, lat, tr)
