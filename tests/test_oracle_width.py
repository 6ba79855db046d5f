"""Pins for the factorised speculation cost (R28; "draft width W and verifier cadence k ... model
acceptance/verification dynamics", "wider drafts add verifier and compute cost").

The step cost with speculation is d(n) = γW(dr_base + dr_seq n) + ver_base + ver_seq n + ver_tok (Wγ + 1) n;
W also sets α_eff = 1 − (1 − α)^W (R8).  Pins:
* W = 1 is R10's model bit for bit: the hand traces T3/T4 (golden, derived before R28) and every W = 1
  brute-force case are unchanged, and T7a/T7b give the W-dependence by hand;
* W is free in the timing exactly when dr_base = dr_seq = ver_tok = 0: then, at an α whose α_eff does not depend
  on W (α = 0 or α = 1), every output is bit-identical across W;
* at such an α, B = 1 (a Lindley queue, service non-decreasing in W) makes every latency pathwise non-decreasing
  in W, and for B > 1 the seed-mean p99 is non-decreasing in W;
* the paper's trend: past W = 2 a wider draft inflates p99 and does not raise goodput under
  bursty load.
"""
import numpy as np
import pytest

from paper_2603_11340_b200 import inputs

WIDTHS = (1, 2, 3, 4)


def _run(orc, wl, k, seed, n=1500, **kw):
    return orc.run([wl], k, seed, n, latencies=True, **kw)


@pytest.mark.parametrize("accept", [0, 65536])
@pytest.mark.parametrize("cont", [0, 1])
def test_width_free_without_width_terms(orc, accept, cont):
    wl = inputs.preset_ll()
    wl["timing"].update(dr_base_us=0, dr_seq_us=0, ver_tok_us=0)
    if cont:
        wl = inputs.continuous(wl)
    for seed in inputs.seeds(3):
        outs = []
        for W in WIDTHS:
            k = inputs.knobs(conc=12, max_num_seqs=6, draft_len=6, spec_on=1, draft_width=W, accept_q16=accept,
                             max_wait_us=0 if cont else 10_000)
            r = _run(orc, wl, k, seed)
            outs.append((r["latencies"].tolist(), r["p99_us"], r["slo_met"], r["window_us"], r["counters"]))
        assert all(o == outs[0] for o in outs[1:])


@pytest.mark.parametrize("accept", [0, 65536])
@pytest.mark.parametrize("preset", ["ll", "sim"])
def test_batch_one_pathwise_monotone_in_width(orc, accept, preset):
    wl = inputs.preset_ll() if preset == "ll" else inputs.preset_sim()
    for seed in inputs.seeds(3):
        prev = None
        for W in WIDTHS:
            k = inputs.knobs(conc=4, max_num_seqs=1, draft_len=4, spec_on=1, draft_width=W, accept_q16=accept)
            lat = _run(orc, wl, k, seed, n=800)["latencies"].astype(np.int64)
            if prev is not None:
                assert np.all(lat >= prev)
                assert np.any(lat > prev)          # the width terms are non-zero in both presets
            prev = lat


@pytest.mark.parametrize("kk", [dict(conc=16, max_num_seqs=4, draft_len=4), dict(conc=16, max_num_seqs=8, draft_len=2)])
def test_seed_mean_p99_monotone_in_width_at_fixed_alpha_eff(orc, kk):
    wl = inputs.preset_ll()
    seeds = inputs.seeds(8)
    p = []
    for W in WIDTHS:
        k = inputs.knobs(spec_on=1, draft_width=W, accept_q16=0, **kk)     # alpha_eff = 0 for every W
        p.append(sum(orc.run([wl], k, s, 2000)["p99_us"] for s in seeds) / len(seeds))
    assert all(b >= a for a, b in zip(p, p[1:])), p
    assert p[-1] > p[0]


@pytest.mark.parametrize("preset", ["stress", "ll"])
def test_wide_drafts_inflate_p99_past_width_two(orc, preset):
    """P:232 "wider drafts ... push p99 close to the SLO boundary or beyond it while delivering only marginal
    goodput gains"; P:222 the climb converges to small W: at α = 0.7, γ = 4, C = B = 8, W = 4 has a higher
    seed-mean p99 than W = 2 and no more goodput."""
    wl = inputs.preset_stress(kind=1) if preset == "stress" else inputs.preset_ll()
    seeds = inputs.seeds(8)
    res = {}
    for W in (2, 4):
        k = inputs.knobs(conc=8, max_num_seqs=8, draft_len=4, spec_on=1, accept_q16=inputs.q16(0.7), draft_width=W)
        rs = [orc.run([wl], k, s, 2000) for s in seeds]
        res[W] = (sum(r["p99_us"] for r in rs) / 8, sum(r["goodput"] for r in rs) / 8)
    assert res[4][0] > 1.2 * res[2][0]
    assert res[4][1] <= res[2][1]


def test_width_cost_hand_values(orc):
    """R28 at n = 1..3 through a one-member batch per n (γ = 1, every draft rejected: one token per step)."""
    tm = dict(pre_base_us=0, pre_tok_us=0, dec_base_us=0, dec_seq_us=0, dr_base_us=7, dr_seq_us=2, ver_base_us=50,
              ver_seq_us=3, ver_tok_us=1, noise_step_ppm=0)
    for W in WIDTHS:
        for n in (1, 2, 3):
            # n identical members (O = 1) form one batch of n at t = 0: c = d(n)
            r = orc.run_trace(tm, n, n, 1, 0, [0] * n, [1] * n, [1] * n, A=[[0]] * n, width=W)
            d = 1 * W * (7 + 2 * n) + 50 + 3 * n + 1 * (W * 1 + 1) * n
            assert list(r["trace"]["c"]) == [d] * n
