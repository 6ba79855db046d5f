"""Pins for oracle/climb.py (Eq. 2-3, Alg. 1) against the worked examples SPEC.md derives from the paper."""
import itertools

import pytest

from oracle import climb
from paper_2603_11340_b200 import inputs

SP = dict(inputs.SCORE_DEFAULTS)


def test_hw_cost_examples():
    """hw_cost(8,8,8,on) = 0.32, hw_cost(2,4,0,on) = 0.06 (Eq. 2, weights P:126)."""
    assert climb.hw_cost_micro(inputs.knobs(conc=8, max_num_seqs=8, draft_len=8, spec_on=1), SP) == 320_000
    assert climb.hw_cost_micro(inputs.knobs(conc=2, max_num_seqs=4, draft_len=0, spec_on=1), SP) == 60_000
    # R20: spec off => gamma counts 0
    assert climb.hw_cost_micro(inputs.knobs(conc=8, max_num_seqs=8, draft_len=8, spec_on=0), SP) == 160_000


def _agg_for(goodput_rps, p99_s, n=1):
    """An aggregate whose pooled goodput and mean p99 are exactly the given values."""
    T = 1_000_000 * 100
    return dict(sum_p99_us=int(round(p99_s * 1e6)) * n, sum_slo_met=int(round(goodput_rps * 100)) * n,
                sum_window_us=T * n, n_seeds=n, flags=0)


def test_score_table1_baseline():
    """S:210 / S:655: goodput 8.13, p99 1.36, SLO 1.2, lambda 5, hw 0.32 -> 8.13 - 0.80 - 0.32 = 7.01
    (Table I baseline)."""
    k = inputs.knobs(conc=8, max_num_seqs=8, draft_len=8, spec_on=1)
    assert climb.score_micro(_agg_for(8.13, 1.36), k, SP) == 7_010_000
    assert climb.score_micro(_agg_for(8.13, 1.36, n=4), k, SP) == 7_010_000


def test_score_table1_tuned():
    """tuned point p99 0.70 <= SLO: no penalty, 15.0 - hw_cost(8,8,0)."""
    k = inputs.knobs(conc=8, max_num_seqs=8, draft_len=0, spec_on=1)
    assert climb.score_micro(_agg_for(15.0, 0.70), k, SP) == 15_000_000 - 160_000
    assert climb.score_micro(_agg_for(15.0, 1.2), k, SP) == 15_000_000 - 160_000   # p99 == SLO: no penalty


def test_score_invalid():
    k = inputs.knobs()
    a = _agg_for(10.0, 1.0)
    a["flags"] = 1
    assert climb.score_micro(a, k, SP) == climb.INT64_MIN


def test_neighbours_live_space():
    """K0 = (8,8,8,on) has 7 neighbours; conc 16 has 6 (clamp-to-self dropped)."""
    k0 = inputs.knobs(conc=8, max_num_seqs=8, draft_len=8, spec_on=1)
    nb = climb.neighbours(inputs.SPACE_LIVE, k0)
    got = [(n["conc"], n["max_num_seqs"], n["draft_len"], n["spec_on"]) for n in nb]
    assert got == [(6, 8, 8, 1), (10, 8, 8, 1), (8, 5, 8, 1), (8, 11, 8, 1), (8, 8, 4, 1), (8, 8, 12, 1),
                   (8, 8, 8, 0)]
    nb16 = climb.neighbours(inputs.SPACE_LIVE, dict(k0, conc=16))
    assert len(nb16) == 6
    # exhaustive properties over the live space
    for c, b, g, on in itertools.product(range(2, 17), range(4, 17), range(0, 17), (0, 1)):
        k = dict(k0, conc=c, max_num_seqs=b, draft_len=g, spec_on=on)
        nb = climb.neighbours(inputs.SPACE_LIVE, k)
        assert len(nb) <= 7 and k not in nb
        assert len({tuple(sorted(x.items())) for x in nb}) == len(nb)
        for x in nb:
            assert 2 <= x["conc"] <= 16 and 4 <= x["max_num_seqs"] <= 16 and 0 <= x["draft_len"] <= 16


def test_neighbours_sim_space():
    """at (W 1, k 2, B 12, wait 0) the lower W / k / wait steps clamp to self and are dropped."""
    k = inputs.knobs(conc=8, max_num_seqs=12, draft_len=2, spec_on=1, draft_width=1, max_wait_us=0)
    nb = climb.neighbours(inputs.SPACE_SIM, k)
    got = [(n["draft_width"], n["draft_len"], n["max_num_seqs"], n["max_wait_us"]) for n in nb]
    assert got == [(2, 2, 12, 0), (1, 4, 12, 0), (1, 2, 8, 0), (1, 2, 16, 0), (1, 2, 12, 10_000)]


def test_neighbours_wide32():
    k0 = inputs.K0
    nb = climb.neighbours(inputs.SPACE_WIDE32, k0)
    assert len(nb) == 31 - 2   # draft_width 1-1 and max_wait 0-10ms clamp to self
    assert nb[0]["conc"] == 6 and nb[0]["max_num_seqs"] == 5 and nb[0]["draft_len"] == 4


def test_decide_move_examples():
    """dS = .03 -> move; dS = .01 with p99 <= SLO -> stay; dS = .001 with p99 > SLO -> move."""
    d = SP["delta_micro"]
    assert climb.decide_move(1_000_000, False, 1_030_000, d)
    assert not climb.decide_move(1_000_000, False, 1_010_000, d)
    assert climb.decide_move(1_000_000, True, 1_001_000, d)
    assert not climb.decide_move(1_000_000, True, 1_000_000, d)


def test_climb_converges_on_concave_surface():
    """a mock surface score = -(conc-10)^2 converges to conc = 10 within the budget."""
    space = inputs.SPACE_LIVE
    st = climb.initial_state(inputs.knobs(conc=4, max_num_seqs=8, draft_len=8, spec_on=1))
    sp = dict(SP, strict_alg1=1)
    for _ in range(8):
        cands = [st["K"]] + climb.neighbours(space, st["K"])
        # encode the mock score into aggregates: goodput only, T = 1e6 us, slo_met = 100 - (conc-10)^2 ...
        aggs = []
        for c in cands:
            target = 10_000_000 - 100_000 * (c["conc"] - 10) ** 2 + climb.hw_cost_micro(c, sp)
            aggs.append(dict(sum_p99_us=0, sum_slo_met=target, sum_window_us=10 ** 12, n_seeds=1, flags=0))
        st, moved, idx, scores = climb.step(st, cands, aggs, sp)
    assert st["K"]["conc"] == 10
    assert st["K_best"]["conc"] in (8, 10)   # strict Alg. 1: best only from measured current points


# ---------------------------------------------------------------------------------------------------
# simulator-controller variant (NEXT-3: P:173-174 EMA, P:188 10-lambda violation + draft/verifier cost)
# ---------------------------------------------------------------------------------------------------
def test_sim_violation_is_ten_lambda():
    """goodput 1.29, p99 1.30, SLO 1.2, lambda 5 -> violation 10*5*0.10 = 5.0; and the sim
    penalty is exactly 10x the live one."""
    k = inputs.knobs(conc=8, max_num_seqs=8, draft_len=0, spec_on=0)
    agg = _agg_for(1.29, 1.30)
    live = climb.score_micro(agg, k, SP)
    sim = climb.score_micro(agg, k, dict(SP, viol_mult=10))
    assert live == 1_290_000 - 500_000 - 160_000
    assert sim == 1_290_000 - 5_000_000 - 160_000
    assert (1_290_000 - 160_000 - sim) == 10 * (1_290_000 - 160_000 - live)
    # no violation -> goodput - hw cost only
    assert climb.score_micro(_agg_for(1.29, 1.10), k, dict(SP, viol_mult=10)) == 1_290_000 - 160_000


def test_sim_draft_verifier_cost_monotone():
    """equal goodput and p99, larger W -> strictly lower score; sparser verification (larger k)
    costs less; the terms vanish with speculation off."""
    sp = dict(inputs.SCORE_SIM)
    agg = _agg_for(10.0, 1.0)
    base = inputs.knobs(conc=8, max_num_seqs=8, draft_len=8, spec_on=1, draft_width=1)
    s1 = climb.score_micro(agg, base, sp)
    s2 = climb.score_micro(agg, dict(base, draft_width=2), sp)
    assert s1 - s2 == sp["w_W_micro"]
    s_k4 = climb.score_micro(agg, dict(base, draft_len=4), sp)
    assert s_k4 - s1 == 4 * sp["w_spec_micro"] - 4 * sp["w_k_micro"]
    off = dict(base, spec_on=0)
    assert climb.score_micro(agg, off, sp) == climb.score_micro(agg, off, SP)


def test_ema_examples():
    """S:153-155 / S:442: EMA 1.4 then 1.0 at beta .5 -> 1.2; 1.5, beta .3, sample 1.0 -> 1.35."""
    e = climb.ema_update(None, 1_400_000, 32768)
    assert e == 1_400_000
    assert climb.ema_update(e, 1_000_000, 32768) == 1_200_000
    e3 = climb.ema_update(1_500_000, 1_000_000, int(round(0.3 * 65536)))
    assert abs(e3 - 1_350_000) <= 2          # Q16 beta (0.3 -> 19661/65536) and the floor
    # stays inside the hull of the samples
    x = None
    for v in (900_000, 1_800_000, 1_100_000, 1_300_000):
        x = climb.ema_update(x, v, 20000)
        assert 900_000 <= x <= 1_800_000


def test_sim_controller_uses_ema_for_the_move():
    """With the EMA below the SLO while the raw p99 violates it, a small improvement no longer escapes."""
    sp = dict(inputs.SCORE_SIM)
    k0 = inputs.knobs(conc=8, max_num_seqs=8, draft_len=8, spec_on=1)
    st = climb.initial_state(k0)
    st["ema"], st["has_ema"] = 800_000, 1
    cands = [k0, dict(k0, conc=10)]
    a0 = _agg_for(10.0, 1.30)           # raw p99 violates; EMA = (1.3 + 0.8)/2 = 1.05 s does not
    a1 = dict(a0)
    a1["sum_slo_met"] += 0              # identical measurements: neighbour differs only by hw cost
    st2, moved, idx, scores = climb.step(st, cands, [a0, a1], sp)
    assert st2["ema"] == 1_050_000 and not moved
