"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/slo_sim.h declares, and its
host-only entry points behave (no GPU compute here)."""
import ctypes as C
import itertools
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="session")
def L():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2603_11340_b200 import _lib
    return _lib


def test_header_symbols_exported(L):
    hdr = open(os.path.join(ROOT, "include", "slo_sim.h")).read()
    declared = set(re.findall(r"^\s*(?:slo_status|const char\*)\s+(slo_\w+)\s*\(", hdr, re.M))
    assert declared == set(L.EXPORTS)
    nm = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (slo_\w+)", nm))
    assert declared <= exported, declared - exported
    lib = L.lib()
    for name in declared:
        assert hasattr(lib, name)


def test_library_is_sm100a(L):
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(L):
    lib = L.lib()
    assert lib.slo_status_string(0) == b"ok"
    assert lib.slo_status_string(-1) == b"invalid argument"
    assert lib.slo_status_string(-3) == b"CUDA error"


def test_create_rejects_bad_arguments(L):
    lib = L.lib()
    h = C.c_void_p()
    assert lib.slo_sim_create(0, None, 0, None, C.byref(h)) == -1
    # invalid workload (noise step too large) is rejected before touching a device
    from paper_2603_11340_b200 import inputs, sim
    w = L.slo_workload()
    w.arr.kind = 0
    w.arr.mean_gap_q16[0] = inputs.mean_gap_q16(10.0)
    w.prompt_lo = 40
    w.output_lo = 1
    w.timing.noise_step_ppm = 5000
    assert lib.slo_sim_create(0, C.byref(w), 1, None, C.byref(h)) == -1
    assert b"noise" in lib.slo_last_error(None)
    w.timing.noise_step_ppm = 0
    w.output_lo = 0                    # lengths must be >= 1
    assert lib.slo_sim_create(0, C.byref(w), 1, None, C.byref(h)) == -1
    w.output_lo = 1
    w.arr.mean_gap_q16[0] = (1 << 64) - 1   # Poisson needs a finite gap
    assert lib.slo_sim_create(0, C.byref(w), 1, None, C.byref(h)) == -1
    w.arr.mean_gap_q16[0] = inputs.mean_gap_q16(10.0)
    w.timing.ver_tok_us = (1 << 20) - 1  # each value < 2^20, but the worst-case step (gamma 16, W 4, n 32) >= 2^31
    assert lib.slo_sim_create(0, C.byref(w), 1, None, C.byref(h)) == -1
    assert b"worst-case" in lib.slo_last_error(None)
    w.timing.ver_tok_us = 0
    w.batching = 2                     # 0 static, 1 continuous
    assert lib.slo_sim_create(0, C.byref(w), 1, None, C.byref(h)) == -1
    assert b"batching" in lib.slo_last_error(None)
    w.batching = 1
    opts = L.slo_sim_opts()
    opts.crn = 1
    opts.group_policy = 4              # 0..3
    assert lib.slo_sim_create(0, C.byref(w), 1, C.byref(opts), C.byref(h)) == -1
    opts.group_policy = 0
    opts.reserved[0] = 1
    assert lib.slo_sim_create(0, C.byref(w), 1, C.byref(opts), C.byref(h)) == -1
    # a valid workload on a machine without a GPU: no device
    import torch
    if not torch.cuda.is_available():
        assert lib.slo_sim_create(0, C.byref(w), 1, None, C.byref(h)) == -5


def test_null_handle_calls(L):
    lib = L.lib()
    x = C.c_void_p()
    hb = (C.c_uint8 * 64)()
    assert lib.slo_exchange_create(None, 2, 0, 32, C.byref(x), hb) == -1
    assert lib.slo_exchange_open(None, hb) == -1
    assert lib.slo_aggregate_exchange(None, None, None, 1, None, None) == -1
    assert lib.slo_exchange_destroy(None) == 0
    assert lib.slo_philox_peak(None, 1, None, None) == -1
    assert lib.slo_sim_run_batch(None, None, 1, None, 1, 1, 0, 1, None, None, None, None, None, None) == -1
    assert lib.slo_aggregate(None, None, 1, 1, None, None) == -1
    assert lib.slo_sim_destroy(None) == 0


def test_neighbors_match_oracle(L):
    """The library's neighbour generator (also run by the climb kernel) equals oracle/climb.py's."""
    from oracle import climb
    from paper_2603_11340_b200 import inputs, sim
    for space in (inputs.SPACE_LIVE, inputs.SPACE_SIM, inputs.SPACE_WIDE32):
        for c, b, g, on, w, mw in itertools.product((1, 2, 8, 16, 32), (1, 4, 8, 16, 32), (0, 2, 8, 16), (0, 1),
                                                    (1, 2, 4), (0, 10_000, 50_000)):
            k = inputs.knobs(conc=c, max_num_seqs=b, draft_len=g, spec_on=on, draft_width=w, max_wait_us=mw)
            assert sim.neighbors(space, k) == climb.neighbours(space, k)


def test_pod_layouts(L):
    assert C.sizeof(L.slo_knobs) == 32
    assert C.sizeof(L.slo_timing) == 40
    assert C.sizeof(L.slo_arrivals) == 40
    assert C.sizeof(L.slo_space) == 64
    assert C.sizeof(L.slo_score_params) == 80
