"""Pins for the oracle's bursty arrival processes ("bursty on/off", P:208, P:232;
BASELINE C5 "bursty MMPP arrivals").  Each check is fixed by the process's definition, not by the oracle's
code, and each catches a distinct plausible mistake:

* on/off (kind 2) with no arrivals in the low state: every arrival lies in an on phase, which for fixed
  sojourns is the closed form a mod (D_on + D_off) < D_on (start in the high state) or ≥ D_off (start low) —
  catches a swapped state, a wrong start state or a phase off by one;
* on/off with λ_H = λ_L is a plain Poisson process of that rate (mean gap within 4 s.e., CV ≈ 1) — catches a
  wrong per-state gap;
* MMPP-2 (kind 1): phases alternate from start_state and tile the time axis; the mean sojourn of each state
  is its configured mean (exponential, within 4 s.e.); arrivals per unit time within each state's phases are
  that state's rate; the long-run rate is the sojourn-weighted mean (λ_H m_H + λ_L m_L)/(m_H + m_L), with
  asymmetric sojourns so a swapped state would give a different number;
* the operational capacity U_p (reading R26) is within its derived error bound of the exact D_p·2^48/ḡ_s.
"""
from fractions import Fraction

import numpy as np
import pytest

from paper_2603_11340_b200 import inputs

U64 = 2 ** 64 - 1


def _draws(orc, wl, n, seed=7, knobs=None):
    k = knobs or inputs.knobs()
    a, _, _, _ = orc.request_draws([wl], k, seed, n)
    return a.astype(np.int64) if a.max() < 2 ** 62 else a


@pytest.mark.parametrize("start_state", [0, 1])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_on_off_no_arrival_in_off_phase(orc, start_state, seed):
    D_on, D_off = 700_000, 1_300_000
    wl = inputs.workload(kind=2, rate_hi=25.0, rate_lo=None, sojourn_us=(D_on, D_off), start_state=start_state)
    a = _draws(orc, wl, 20_000, seed=seed)
    assert np.all(np.diff(a) >= 0)
    period = D_on + D_off
    ph = a % period
    if start_state == 0:          # phases: on [0, D_on), off [D_on, period), ...
        assert np.all(ph < D_on)
    else:                         # phases: off [0, D_off), on [D_off, period), ...
        assert np.all(ph >= D_off)
    # and the on phases are all used: arrivals reach both ends of an on phase (25/s over 0.7 s ~ 17.5 each)
    lo_end = D_off if start_state else 0
    assert ph.min() - lo_end < 50_000 and (lo_end + D_on) - ph.max() < 50_000
    # arrivals per on phase ~ Poisson(25 * 0.7 = 17.5)
    n_periods = int(a[-1] // period)
    per = np.bincount((a // period).astype(np.int64), minlength=n_periods + 1)[:n_periods]
    assert abs(per.mean() - 17.5) < 4 * np.sqrt(17.5 / len(per))


@pytest.mark.parametrize("seed", [11, 12])
def test_on_off_equal_rates_is_poisson(orc, seed):
    lam = 40.0                                      # req/s in both states
    wl = inputs.workload(kind=2, rate_hi=lam, rate_lo=lam, sojourn_us=(333_333, 777_777))
    n = 200_000
    a = _draws(orc, wl, n, seed=seed).astype(np.float64)
    gaps = np.diff(np.concatenate([[0.0], a]))
    mean = 1e6 / lam
    assert abs(gaps.mean() - mean) < 4 * mean / np.sqrt(n)
    cv = gaps.std() / gaps.mean()
    assert abs(cv - 1.0) < 0.01
    # memorylessness: P(gap > mean) = e^-1
    assert abs((gaps > mean).mean() - np.exp(-1.0)) < 4 * np.sqrt(np.exp(-1) * (1 - np.exp(-1)) / n)


def _mmpp(lam_h, lam_l, m_h, m_l, start_state=0):
    return inputs.workload(kind=1, rate_hi=lam_h, rate_lo=lam_l, sojourn_us=(m_h, m_l), start_state=start_state)


@pytest.mark.parametrize("start_state", [0, 1])
def test_mmpp_phases_alternate_tile_and_have_mean_sojourn(orc, start_state):
    m_h, m_l = 1_000_000, 3_000_000
    wl = _mmpp(18.0, 2.0, m_h, m_l, start_state)
    n = 40_000
    st, D, U, s = orc.phases([wl], inputs.knobs(), 99, n)
    st = st.astype(np.int64)
    D = D.astype(np.int64)
    assert list(s[:4]) == [start_state, 1 - start_state, start_state, 1 - start_state]
    assert np.all(s[1:] != s[:-1])                   # strict alternation
    assert st[0] == 0 and np.all(st[1:] == st[:-1] + D[:-1])   # phases tile the time axis
    for state, m in ((0, m_h), (1, m_l)):
        d = D[s == state].astype(np.float64)
        assert abs(d.mean() - m) < 4 * m / np.sqrt(len(d))        # exponential: sd = mean
        assert abs(d.std() / d.mean() - 1.0) < 0.03


def _scaled_gap(mean_gap_q16, rate_scale_q8=256):
    return mean_gap_q16 if mean_gap_q16 == U64 else (mean_gap_q16 * 256) // rate_scale_q8


@pytest.mark.parametrize("rate_scale", [256, 77, 1000])
def test_mmpp_capacity_error_bound(orc, rate_scale):
    """R26: U_p = ⌊D·⌊(2^64−1)/ḡ⌋/2^16⌋ (capped at 2^62) lies in [D·2^48/ḡ − D/2^16 − 2, D·2^48/ḡ]."""
    wl = _mmpp(18.0, 2.0, 1_000_000, 3_000_000)
    k = inputs.knobs(rate_scale_q8=rate_scale)
    st, D, U, s = orc.phases([wl], k, 5, 2000)
    g = [_scaled_gap(x, rate_scale) for x in wl["arrivals"]["mean_gap_q16"]]
    for d, u, state in zip(D.tolist(), U.tolist(), s.tolist()):
        exact = Fraction(d * 2 ** 48, g[state])
        assert u <= exact
        assert exact - u <= Fraction(d, 2 ** 16) + 2
    # a state without arrivals has capacity 0 (its phases are skipped by the time change)
    wl0 = _mmpp(18.0, None, 1_000_000, 3_000_000)
    _, D0, U0, s0 = orc.phases([wl0], k, 5, 50)
    assert np.all(U0[s0 == 1] == 0) and np.all(U0[s0 == 0] > 0)


@pytest.mark.parametrize("seed", [21, 22])
def test_mmpp_per_state_and_long_run_rates(orc, seed):
    lam_h, lam_l, m_h, m_l = 18.0, 2.0, 1_000_000, 3_000_000
    wl = _mmpp(lam_h, lam_l, m_h, m_l)
    n = 300_000
    a = _draws(orc, wl, n, seed=seed)
    n_ph = 200_000
    st, D, U, s = orc.phases([wl], inputs.knobs(), seed, n_ph)
    st = st.astype(np.int64)
    D = D.astype(np.int64)
    T = int(a[-1])
    assert st[-1] > T                                 # enough phases drawn to cover the arrivals
    p_of = np.searchsorted(st, a, side="right") - 1   # phase holding each arrival (by the phase table)
    assert np.all(a < st[p_of] + D[p_of])
    last = int(p_of[-1])                              # complete phases only
    cnt = np.bincount(p_of[p_of < last], minlength=last)[:last]
    Dh, sh = D[:last], s[:last]
    rate_h = cnt[sh == 0].sum() / (Dh[sh == 0].sum() / 1e6)
    rate_l = cnt[sh == 1].sum() / (Dh[sh == 1].sum() / 1e6)
    nh, nl = cnt[sh == 0].sum(), cnt[sh == 1].sum()
    assert abs(rate_h - lam_h) < 4 * lam_h / np.sqrt(nh)
    assert abs(rate_l - lam_l) < 4 * lam_l / np.sqrt(nl)
    # long-run rate = sojourn-weighted mean = (18·1 + 2·3)/4 = 6/s (a swapped state would give 14/s)
    lr = (lam_h * m_h + lam_l * m_l) / (m_h + m_l)
    assert abs(lr - 6.0) < 1e-12
    long_run = n / (T / 1e6)
    assert abs(long_run - lr) < 0.05 * lr


@pytest.mark.parametrize("seed", [31, 32])
def test_mmpp_positions_within_a_phase_are_uniform(orc, seed):
    """Given its count, a Poisson process's points in an interval are i.i.d. uniform: the relative position
    (a − start_p)/D_p of the arrivals is Uniform(0, 1) in both states — catches a time change that maps a
    phase's operational time with another state's gap (points squeezed to the front or piled at the end)."""
    wl = _mmpp(18.0, 2.0, 1_000_000, 3_000_000)
    n = 200_000
    a = _draws(orc, wl, n, seed=seed)
    st, D, U, s = orc.phases([wl], inputs.knobs(), seed, 200_000)
    st = st.astype(np.int64)
    D = D.astype(np.int64)
    p_of = np.searchsorted(st, a, side="right") - 1
    x = (a - st[p_of]) / D[p_of]
    for state in (0, 1):
        xs = x[s[p_of] == state]
        m = len(xs)
        assert abs(xs.mean() - 0.5) < 4 * np.sqrt(1 / 12 / m)
        for lo in (0.0, 0.5, 0.9):                   # deciles at the front, middle and end
            frac = ((xs >= lo) & (xs < lo + 0.1)).mean()
            assert abs(frac - 0.1) < 4 * np.sqrt(0.09 / m)
