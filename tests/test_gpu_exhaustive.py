"""Exhaustive device-vs-oracle / device-vs-closed-form checks of the integer transforms over all 2^32 inputs
(SURVEY §8(c) pins table), through K6 `slo_selftest_transforms`, which runs the same device functions K1/K1c
call:

* E_q: the device's per-2^20-block hashes equal the oracle's (tests/golden/exp_q32_block_hash.txt,
  written by tools/gen_golden_exp_hash.py from oracle/ only) — bit equality on every u — and the count of
  adjacent increases equals the oracle's (R27);
* lengths (§2.4): for each table, #{u : length(u) = lo + i} = cw[i] − cw[i−1] exactly (cw[−1] = 0,
  cw[ncw] = 2^32) and length is non-decreasing in u, which together fix the function at every u;
* acceptance (§2.5): #{u : A(u) ≥ a} = T_a exactly (T_a from the oracle's thresholds, pinned by
  test_oracle_transforms) and A is non-increasing in u — again fixing A at every u;
* noise (§2.4): the histogram of f over every word is the 4-fold byte convolution on the lattice.
"""
import os

import numpy as np
import pytest

from paper_2603_11340_b200 import inputs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def S():
    import torch
    from paper_2603_11340_b200 import sim
    assert torch.cuda.is_available()
    wls = [inputs.preset_ll(), inputs.preset_sim(), inputs.preset_stress(kind=1)]
    s = sim.Simulator(wls, device=0)
    yield s, wls
    s.close()


def test_exp_q32_all_inputs_bit_equal_to_oracle(S):
    s, _ = S
    out = s.selftest("exp")
    gold, nonmono = {}, None
    with open(os.path.join(GOLD, "exp_q32_block_hash.txt")) as fh:
        for line in fh:
            if line.startswith("# nonmono"):
                nonmono = int(line.split()[2])
            elif not line.startswith("#"):
                b, v = line.split()
                gold[int(b)] = int(v, 16)
    dev = [int(x) for x in out[:4096]]
    bad = [b for b in range(4096) if dev[b] != gold[b]]
    assert not bad, f"{len(bad)} blocks differ, first {bad[:5]}"
    assert int(out[4096]) == nonmono


@pytest.mark.parametrize("wl,table", [(0, 1), (1, 0), (1, 1), (2, 1), (0, 0)])
def test_length_tables_all_inputs(S, wl, table):
    s, wls = S
    t = wls[wl]["output" if table else "prompt"]
    cw = [int(x) for x in t["cw"]]
    out = s.selftest("length", wl, table)
    n = len(cw)
    bounds = [0] + cw + [2 ** 32]
    expect = [bounds[i + 1] - bounds[i] for i in range(n + 1)]
    assert [int(x) for x in out[:n + 1]] == expect
    assert int(out[n + 1]) == 0                      # monotone and in range: the function is fixed at every u


@pytest.mark.parametrize("accept,width,gamma", [(32768, 1, 16), (inputs.q16(0.3), 2, 8), (inputs.q16(0.9), 4, 16),
                                                (0, 1, 4), (65536, 3, 16), (12345, 1, 1), (60000, 2, 12),
                                                (inputs.q16(0.3), 1, 16), (65500, 1, 16), (inputs.q16(0.7), 2, 16)])
@pytest.mark.parametrize("guide", ["accept", "accept2"], ids=["byte-guide", "two-level-guide"])
def test_acceptance_all_inputs(S, orc, accept, width, gamma, guide):
    """Both acceptance guides (K1 / K1c's byte guide, K1g's two-level guide) fix A at every u."""
    s, _ = S
    out = s.selftest(guide, accept, width, gamma)
    _, T = orc.thresholds(accept, width, gamma)
    hist = [int(x) for x in out[:17]]
    assert sum(hist) == 2 ** 32
    for a in range(1, gamma + 1):
        assert sum(hist[a:]) == T[a - 1], (a, sum(hist[a:]), T[a - 1])
    assert sum(hist[gamma + 1:]) == 0
    assert int(out[17]) == 0                          # non-increasing in u


@pytest.mark.parametrize("step", [0, 1, 338, 1960])
def test_noise_all_inputs(S, step):
    s, _ = S
    out = s.selftest("noise", step)
    if step == 0:
        assert int(out[510]) == 2 ** 32
    else:
        one = np.ones(256, dtype=object)
        law = one
        for _ in range(3):
            law = np.convolve(law, one)
        assert [int(x) for x in out[:1021]] == [int(x) for x in law]
    assert int(out[1021]) == 0
