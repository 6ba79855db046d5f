"""The boundary used from plain C: examples/c_api_demo.c links libslosim.so with gcc (no Python, no torch).

CPU: it compiles and links against the in-tree library.  GPU: its results equal the oracle's on the same
integer workload, replica by replica (p99, goodput bits, SLO count, window)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    import __graft_entry__
    __graft_entry__.build()
    exe = str(tmp_path / "c_api_demo")
    pkg = os.path.join(ROOT, "paper_2603_11340_b200")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "c_api_demo.c"), "-L", pkg, "-lslosim",
                           f"-Wl,-rpath,{pkg}", "-o", exe])
    return exe


def test_c_demo_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


def _workload():
    from paper_2603_11340_b200 import inputs
    w = inputs.workload(kind=0, rate=10.0, prompt=inputs.point_mass(40),
                        output={"lo": 1, "cw": [(l << 32) // 64 for l in range(1, 64)]}, timing=inputs.LL_TIMING)
    w["arrivals"]["mean_gap_q16"] = [100000 << 16, 100000 << 16]
    return w


@pytest.mark.gpu
def test_c_demo_matches_oracle(tmp_path, orc):
    import struct
    from paper_2603_11340_b200 import inputs
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    rows = [l.split() for l in out.stdout.splitlines() if l and l[0].isdigit()]
    assert len(rows) == 8
    ks = [inputs.knobs(conc=8, max_num_seqs=16),
          inputs.knobs(conc=8, max_num_seqs=8, draft_len=8, spec_on=1, accept_q16=32768)]
    seeds = [1, 2, 3, 0x5EED0000]
    wls = [_workload()]
    for ci, k in enumerate(ks):
        for si, sd in enumerate(seeds):
            r = ci * 4 + si
            ref = orc.run(wls, k, sd, 2000)
            rid, p99, gp, met, win = rows[r]
            assert int(rid) == r and int(p99) == ref["p99_us"] and int(met) == ref["slo_met"]
            assert int(win) == ref["window_us"]
            assert struct.pack("<d", float(gp)) == struct.pack("<d", ref["goodput"])
