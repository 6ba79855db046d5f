"""Pins for the oracle's random-number layer against things other than itself."""
import math
import os
import random

import numpy as np
import pytest

from paper_2603_11340_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _kats():
    rows = []
    with open(os.path.join(GOLD, "philox_kat.txt")) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(x, 16) for x in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answers(orc):
    """Random123 KATs (Salmon et al. SC'11) — tests/golden/philox_kat.txt."""
    kats = _kats()
    assert len(kats) == 3
    for ctr, key, out in kats:
        assert orc.philox(ctr, key) == out


def test_exp_exact_at_powers_of_two(orc):
    """x = u+1 = 2^e gives t = 0, so E_q = floor((32-e)*2^31*round(ln2*2^32)/2^31) exactly."""
    ln2q = 2977044472
    for e in range(0, 32):
        u = (1 << e) - 1
        assert orc.exp_q32(u) == (32 - e) * ln2q
    assert orc.exp_q32(0xFFFFFFFF) == 0


def test_exp_accuracy_vs_libm(orc):
    """|E_q/2^32 - (-ln((u+1)/2^32))| <= 2^-26 on a dense stratified sample."""
    rng = random.Random(1)
    us = [rng.getrandbits(32) for _ in range(20000)]
    us += [(1 << e) + d for e in range(32) for d in (-1, 0, 1) if 0 <= (1 << e) + d < (1 << 32)]
    us += list(range(0, 200)) + [0xFFFFFFFF - i for i in range(200)]
    worst = 0.0
    for u in us:
        ref = -math.log((u + 1) / 2.0 ** 32)
        got = orc.exp_q32(u) / 2.0 ** 32
        worst = max(worst, abs(got - ref))
    assert worst <= 2.0 ** -26, worst


def test_exp_mean_is_one(orc):
    """E[Exp(1)] = 1: the mean over a stratified grid of u (midpoints) matches within 1e-6."""
    n = 1 << 16
    step = (1 << 32) // n
    m = sum(orc.exp_q32(i * step + step // 2) for i in range(n)) / n / 2.0 ** 32
    assert abs(m - 1.0) < 2e-4  # stratified quadrature of -ln; the tail bin dominates the error


def test_lengths_count_cut_points(orc):
    """length(u) = lo + #{cw <= u} — equals numpy.searchsorted(side='right') and the
    probability of each value is exactly (cw[l] - cw[l-1]) / 2^32 (boundary checks)."""
    tab = inputs.lognormal_table(math.log(80.0), 0.4, 1, 64)
    cw = tab["cw"]
    assert all(cw[i] <= cw[i + 1] for i in range(len(cw) - 1))
    rng = random.Random(2)
    arr = np.array(cw, dtype=np.uint64)
    for _ in range(3000):
        u = rng.getrandbits(32)
        assert orc.length(tab, u) == tab["lo"] + int(np.searchsorted(arr, u, side="right"))
    for l, c in enumerate(cw):
        if c > 0 and (l == 0 or cw[l - 1] < c):
            assert orc.length(tab, c - 1) == tab["lo"] + l
        assert orc.length(tab, c) >= tab["lo"] + l + 1
    # point mass
    assert orc.length(inputs.point_mass(40), 12345) == 40
    # 64-token cap: a large share at the cap ("caps responses at 64 tokens")
    cap_share = (2 ** 32 - cw[-1]) / 2 ** 32
    assert 0.6 < cap_share < 0.8


def test_thresholds_and_leviathan(orc):
    """#{u : A(u) >= a} = T_a exactly (boundary), E[tokens/step] = sum_a T_a/2^32 which equals
    Leviathan et al.'s (1 - alpha^(gamma+1)) / (1 - alpha) up to Q16 quantisation."""
    for alpha in (0.3, 0.5, 0.7, 0.9):
        aq = inputs.q16(alpha)
        for gamma in (1, 2, 4, 8, 16):
            ae, T = orc.thresholds(aq, 1, gamma)
            assert ae == aq  # W = 1 => alpha_eff = alpha
            assert all(T[i] >= T[i + 1] for i in range(len(T) - 1))
            exp_tokens = 1.0 + sum(T) / 2.0 ** 32
            lev = (1 - (aq / 65536.0) ** (gamma + 1)) / (1 - aq / 65536.0)
            assert abs(exp_tokens - lev) < 1e-6 * gamma + 1e-7
    # widths: alpha_eff = 1 - (1 - alpha)^W
    for W in (1, 2, 3, 4):
        ae, _ = orc.thresholds(inputs.q16(0.5), W, 1)
        assert abs(ae / 65536.0 - (1 - 0.5 ** W)) < 1e-4
    # extremes
    assert orc.thresholds(0, 2, 4)[1] == [0, 0, 0, 0]
    assert orc.thresholds(65536, 1, 3)[1] == [1 << 32] * 3


def test_fnv_and_validity(orc):
    """FNV-1a-32 (Fowler/Noll/Vo) of the 32 knob bytes: check against a direct byte-level FNV."""
    k = inputs.knobs(conc=8, max_num_seqs=16, draft_len=4, spec_on=1, draft_width=2, workload=0,
                     rate_scale_q8=300, accept_q16=40000, max_wait_us=1234)
    b = bytes([8, 16, 4, 1, 2, 0]) + (300).to_bytes(2, "little") + (40000).to_bytes(4, "little") + \
        (1234).to_bytes(4, "little") + bytes(16)
    h = 2166136261
    for x in b:
        h = ((h ^ x) * 16777619) & 0xFFFFFFFF
    assert orc.fnv1a_knobs(k) == h
    assert orc.knobs_valid(k)
    for bad in (dict(conc=0), dict(conc=33), dict(max_num_seqs=0), dict(draft_len=17), dict(spec_on=2),
                dict(draft_width=0), dict(draft_width=5), dict(workload=1), dict(rate_scale_q8=0),
                dict(accept_q16=65537), dict(max_wait_us=50001)):
        assert not orc.knobs_valid(dict(k, **bad)), bad
