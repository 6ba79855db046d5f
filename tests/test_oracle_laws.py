"""Queueing laws the oracle must obey (SURVEY §8(c) pins; BASELINE north star "Little's law", "p99 monotone
in offered load past the knee").

* Little's law as an exact integer identity: over a drained segment (warmup 0) the oracle's Σℓ equals
  ∫N(t)dt, where N(t) = arrivals(≤ t) − departures(≤ t) is built by an independent event sweep over the
  trace's arrival (or, in a closed loop, issue) and completion instants — catches a latency measured from the
  wrong origin, a dropped or double-counted request, or a Σℓ over the wrong set.
* p99 monotone in offered load past the knee (BASELINE): for B > 1 the seed-mean p99 is
  non-decreasing in `rate_scale_q8` once the offered load exceeds the service capacity — catches a load
  scaling applied the wrong way (gap × scale instead of ÷) or one that does not reach the arrivals.
"""
import numpy as np
import pytest

from paper_2603_11340_b200 import inputs


def _integral_of_N(t_in, t_out):
    """∫ N(t) dt for N(t) = #{i : t_in_i <= t < t_out_i}, by sweeping the sorted event instants."""
    ev_t = np.concatenate([t_in, t_out]).astype(object)
    ev_d = np.concatenate([np.ones(len(t_in), dtype=np.int64), -np.ones(len(t_out), dtype=np.int64)])
    order = sorted(range(len(ev_t)), key=lambda k: (int(ev_t[k]), int(ev_d[k])))
    area, n, prev = 0, 0, None
    for k in order:
        t = int(ev_t[k])
        if prev is not None:
            area += n * (t - prev)
        n += int(ev_d[k])
        prev = t
    assert n == 0
    return area


CASES = [
    ("ll", dict(conc=8, max_num_seqs=4)),
    ("ll", dict(conc=16, max_num_seqs=8, draft_len=4, spec_on=1, accept_q16=inputs.q16(0.6))),
    ("ll", dict(conc=4, max_num_seqs=16, max_wait_us=20_000, rate_scale_q8=400)),
    ("stress", dict(conc=12, max_num_seqs=6, draft_len=2, spec_on=1, draft_width=2)),
    ("sim", dict(conc=6, max_num_seqs=3, max_wait_us=5_000)),
    ("cont", dict(conc=10, max_num_seqs=5, draft_len=3, spec_on=1)),
    ("closed", dict(conc=6, max_num_seqs=4)),
    ("think", dict(conc=8, max_num_seqs=3)),
]


def _wl(name):
    return {"ll": inputs.preset_ll(), "stress": inputs.preset_stress(kind=1), "sim": inputs.preset_sim(),
            "cont": inputs.continuous(inputs.preset_ll()), "closed": inputs.preset_closed(),
            "think": inputs.preset_closed(think_us=150_000)}[name]


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("seed", [3, 4])
def test_littles_law_exact(orc, case, seed):
    name, kk = CASES[case]
    wl = _wl(name)
    k = inputs.knobs(**kk)
    n = 3000
    r = orc.run([wl], k, inputs.seeds(seed + 1)[seed], n, trace=True)
    tr = r["trace"]
    closed = wl["arrivals"]["kind"] >= 3
    t_in = tr["s"] if closed else tr["a"]           # the latency origin (R2 / DESIGN.md §2.11)
    t_out = tr["c"]
    assert np.all(t_out >= t_in)
    area = _integral_of_N(t_in, t_out)
    assert r["sum_latency_us"] == area                # Σℓ = ∫ N(t) dt, exactly
    # time-average form L = λ W over the segment [min t_in, max t_out]
    span = int(t_out.max()) - int(t_in.min())
    L = area / span
    lam = n / span
    W = r["sum_latency_us"] / n
    assert abs(L - lam * W) <= 1e-9 * max(1.0, L)


@pytest.mark.parametrize("kk", [dict(conc=16, max_num_seqs=4), dict(conc=32, max_num_seqs=8),
                                dict(conc=16, max_num_seqs=8, draft_len=4, spec_on=1, accept_q16=inputs.q16(0.5)),
                                dict(conc=24, max_num_seqs=12, max_wait_us=20_000)])
def test_p99_monotone_in_load_past_knee(orc, kk):
    wl = inputs.preset_ll()
    seeds = inputs.seeds(8)
    n = 2000

    def mean_p99(scale_q8):
        k = inputs.knobs(rate_scale_q8=scale_q8, **kk)
        return sum(orc.run([wl], k, s, n)["p99_us"] for s in seeds) / len(seeds)

    def goodput(scale_q8):
        k = inputs.knobs(rate_scale_q8=scale_q8, **kk)
        return sum(orc.run([wl], k, s, n)["goodput"] for s in seeds) / len(seeds)

    # locate the knee: the smallest load (10 req/s x scale) whose seed-mean p99 exceeds 2x the light-load p99
    light = mean_p99(64)                                  # 2.5 req/s
    scales = [64 * m for m in range(2, 33)]               # 5 .. 80 req/s
    p = [mean_p99(s) for s in scales]
    knee = next(i for i, v in enumerate(p) if v > 2 * light)
    past = p[knee:]
    assert len(past) >= 4
    assert all(b >= a for a, b in zip(past, past[1:])), (knee, past)
    assert past[-1] > 3 * light
    # and goodput never exceeds throughput (slo_met <= n): the SLO-met rate is bounded by the offered load
    assert goodput(scales[-1]) <= 80.0 + 1e-9
