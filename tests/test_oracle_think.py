"""Pins for the oracle's closed loop with exponential think time (arrival kind 4):
the zero-think special case, a single-user hand derivation, an independent per-microsecond brute force
and the interactive response-time law."""
import math
import random

import numpy as np
import pytest

from paper_2603_11340_b200 import inputs


def _think_draws(orc, seed, n, g):
    """Z_k = floor(E_q(w0) * g / 2^48), w0 = word 0 of the THINK block (k, 4, 0, 0)."""
    k0, k1 = seed & 0xFFFFFFFF, seed >> 32          # crn = 1, stream_id = 0: the key is the seed
    return [(orc.exp_q32(orc.philox([k, 4, 0, 0], [k0, k1])[0]) * g) >> 48 for k in range(n)]


def _tiny(rng, think_us, noise):
    tm = dict(pre_base_us=rng.randrange(0, 5), pre_tok_us=rng.randrange(0, 3), dec_base_us=rng.randrange(1, 9),
              dec_seq_us=rng.randrange(0, 4), dr_base_us=0, dr_seq_us=0, ver_base_us=0, ver_seq_us=0,
              ver_tok_us=0, noise_step_ppm=noise)
    w = inputs.preset_closed(think_us=think_us)
    w["prompt"] = inputs.lognormal_table(math.log(3.0), 0.5, 1, 6)
    w["output"] = inputs.lognormal_table(math.log(3.0), 0.6, 1, 7)
    w["timing"] = tm
    return w


def brute_force_think(tm, C, B, mw, N, P, O, f, Z):
    """Per-microsecond time stepping of the kind-4 closed loop (static batching, gamma = 0), written
    separately from the oracle's event loop: completion k (numbered by batch, then step count, then request
    index) makes user chain k + C ready Z_k later; ready chains issue in chain order."""
    s, c = [None] * N, [None] * N
    ready = {q: 0 for q in range(min(C, N))}
    ordinal, in_service = {}, {}
    t = issued = batched = done = nord = 0
    while done < N:
        again = True
        while again:
            again = False
            for m in sorted((m for m, cm in in_service.items() if cm == t), key=lambda m: ordinal[m]):
                del in_service[m]
                done += 1
                if ordinal[m] + C < N:
                    ready[ordinal[m] + C] = t + Z[ordinal[m]]
            for q in sorted(q for q, r in ready.items() if r == t):
                del ready[q]
                s[issued] = t
                issued += 1
            if not in_service and batched < issued:
                q = issued - batched
                if mw == 0 or q >= B or t >= s[batched] + mw:
                    mem = list(range(batched, batched + min(B, q)))
                    Dp = f[mem[0]] * (tm["pre_base_us"] + tm["pre_tok_us"] * max(P[m] for m in mem)) // 10 ** 6
                    rem = {m: O[m] for m in mem}
                    cum = 0
                    while rem:
                        cum += tm["dec_base_us"] + tm["dec_seq_us"] * len(rem)
                        for m in sorted(rem):
                            rem[m] -= 1
                            if rem[m] == 0:
                                del rem[m]
                                c[m] = t + Dp + f[mem[0]] * cum // 10 ** 6
                                in_service[m] = c[m]
                    for m in sorted(mem, key=lambda m: (O[m], m)):
                        ordinal[m] = nord
                        nord += 1
                    batched += len(mem)
                    if any(cm == t for cm in in_service.values()):
                        again = True
        t += 1
    return s, c


@pytest.mark.parametrize("C,B", [(1, 1), (4, 2), (6, 8), (16, 4), (32, 32)])
def test_zero_think_is_the_zero_think_closed_loop(orc, C, B):
    """Mean think time 0: every Z_k = 0, so chain k + C is ready at the k-th completion — kind 3's gate
    s_j = kappa_{j-C} (§2.11) — and every output equals kind 3's; the THINK blocks are still drawn."""
    k = inputs.knobs(conc=C, max_num_seqs=B, draft_len=4, spec_on=1)
    for N, warm in ((300, 0), (517, 40), (3, 1)):
        r3 = orc.run([inputs.preset_closed()], k, 11, N - warm, warmup_len=warm, latencies=True, trace=True)
        r4 = orc.run([inputs.preset_closed(think_us=0)], k, 11, N - warm, warmup_len=warm, latencies=True,
                     trace=True)
        assert np.array_equal(r3["latencies"], r4["latencies"])
        assert np.array_equal(r3["trace"]["s"], r4["trace"]["s"])
        for key in ("p99_us", "slo_met", "window_us", "sum_latency_us", "p50_us", "p95_us", "flags"):
            assert r3[key] == r4[key]
        assert r4["counters"]["philox_blocks"] == r3["counters"]["philox_blocks"] + max(0, N - C)


def test_single_user_hand_derivation(orc):
    """One user, B = 1, no noise, point-mass lengths: request k is served alone for
    D = pre_base + pre_tok P + O (dec_base + dec_seq), and the user issues request k + 1 Z_k after request
    k completes: s_0 = 0, c_k = s_k + D, s_{k+1} = c_k + Z_k; latency D; window c_{N-1} - s_0."""
    w = inputs.preset_closed(think_us=250_000)
    w["prompt"], w["output"] = inputs.point_mass(40), inputs.point_mass(20)
    w["timing"] = dict(inputs.LL_TIMING, noise_step_ppm=0)
    tm = w["timing"]
    D = tm["pre_base_us"] + tm["pre_tok_us"] * 40 + 20 * (tm["dec_base_us"] + tm["dec_seq_us"])
    seed, N = 0x1234_5678_9ABC, 64
    r = orc.run([w], inputs.knobs(conc=1, max_num_seqs=1), seed, N, latencies=True, trace=True)
    Z = _think_draws(orc, seed, N, 250_000 * 65536)
    s = [0]
    for k in range(N - 1):
        s.append(s[-1] + D + Z[k])
    assert list(r["trace"]["s"]) == s
    assert list(r["trace"]["c"]) == [x + D for x in s]
    assert np.all(r["latencies"] == D)
    assert r["window_us"] == s[-1] + D
    assert r["counters"]["philox_blocks"] == N + (N - 1)
    assert len(set(Z)) > N // 2 and min(Z) >= 0     # the think times do vary


@pytest.mark.parametrize("case", range(80))
def test_think_matches_brute_force(orc, case):
    rng = random.Random(4000 + case)
    think = rng.choice([0, 1, 3, 8])
    w = _tiny(rng, think, rng.choice([0, 0, 1_500]))
    C, B, mw = rng.randrange(1, 7), rng.randrange(1, 7), rng.choice([0, 0, 2, 5])
    N = rng.randrange(1, 14)
    seed = rng.getrandbits(64)
    k = inputs.knobs(conc=C, max_num_seqs=B, max_wait_us=mw)
    r = orc.run([w], k, seed, N, latencies=True, trace=True)
    _, P, O, w3 = orc.request_draws([w], k, seed, N)
    noise = w["timing"]["noise_step_ppm"]
    f = [1_000_000 + (sum((int(x) >> (8 * i)) & 0xFF for i in range(4)) - 510) * noise for x in w3]
    Z = _think_draws(orc, seed, N, think * 65536)
    s, c = brute_force_think(w["timing"], C, B, mw, N, [int(x) for x in P], [int(x) for x in O], f, Z)
    assert list(r["trace"]["s"]) == s
    assert list(r["trace"]["c"]) == c
    assert list(r["latencies"]) == [ci - si for ci, si in zip(c, s)]


@pytest.mark.parametrize("C,B,think_s", [(8, 4, 2.0), (16, 8, 0.5), (4, 16, 5.0)])
def test_interactive_response_time_law(orc, C, B, think_s):
    """Interactive response-time law (closed system with think time): C = X (R + Z) over a long run, with
    X the completion rate, R the mean latency from issue and Z the mean think time; the finite segment
    (initial transient, the users idle after the source runs out) costs a few per cent."""
    N = 20_000
    r = orc.run([inputs.preset_closed(think_us=think_s * 1e6)], inputs.knobs(conc=C, max_num_seqs=B), 3, N,
                trace=True)
    tr = r["trace"]
    X = N / ((int(tr["c"].max()) - int(tr["s"].min())) * 1e-6)
    R = float(np.mean(tr["c"] - tr["s"])) * 1e-6
    assert X * (R + think_s) == pytest.approx(C, rel=0.04)


def brute_force_continuous_think(tm, C, B, N, P, O, Z):
    """Per-microsecond time stepping of the kind-4 closed loop under continuous batching (DESIGN.md §2.11,
    §2.12; gamma = 0, no noise), written separately from the oracle: completions at one iteration end are
    numbered in request-index order; completion k makes chain k + C ready Z_k later."""
    s, c = [None] * N, [None] * N
    rem = list(O)
    ready = {q: 0 for q in range(min(C, N))}
    t = issued = admitted = done = 0
    running, joining, finishing = [], [], []
    end = None
    while done < N:
        again = True
        while again:
            again = False
            if end == t:
                for m in sorted(finishing):
                    c[m] = t
                    if done + C < N:
                        ready[done + C] = t + Z[done]
                    done += 1
                running = [m for m in running if m not in finishing] + joining
                finishing, joining, end = [], [], None
            for q in sorted(q for q, r in ready.items() if r == t):
                del ready[q]
                s[issued] = t
                issued += 1
            if end is None:
                if len(running) < B and admitted < issued:
                    new = list(range(admitted, admitted + min(B - len(running), issued - admitted)))
                    admitted += len(new)
                    joining, end = new, t + tm["pre_base_us"] + tm["pre_tok_us"] * max(P[m] for m in new)
                elif running:
                    for m in running:
                        rem[m] -= 1
                        if rem[m] == 0:
                            finishing.append(m)
                    end = t + tm["dec_base_us"] + tm["dec_seq_us"] * len(running)
                if end == t:
                    again = True
        t += 1
    return s, c


@pytest.mark.parametrize("case", range(60))
def test_continuous_think_matches_brute_force(orc, case):
    rng = random.Random(7000 + case)
    think = rng.choice([0, 1, 4, 9])
    w = inputs.continuous(_tiny(rng, think, 0))
    C, B, N = rng.randrange(1, 7), rng.randrange(1, 7), rng.randrange(1, 14)
    seed = rng.getrandbits(64)
    k = inputs.knobs(conc=C, max_num_seqs=B)
    r = orc.run([w], k, seed, N, latencies=True, trace=True)
    _, P, O, _ = orc.request_draws([w], k, seed, N)
    Z = _think_draws(orc, seed, N, think * 65536)
    s, c = brute_force_continuous_think(w["timing"], C, B, N, [int(x) for x in P], [int(x) for x in O], Z)
    assert list(r["trace"]["s"]) == s
    assert list(r["trace"]["c"]) == c
    assert list(r["latencies"]) == [ci - si for ci, si in zip(c, s)]


@pytest.mark.parametrize("C,B", [(1, 1), (6, 8), (16, 4)])
def test_continuous_zero_think_is_kind_3(orc, C, B):
    k = inputs.knobs(conc=C, max_num_seqs=B, draft_len=4, spec_on=1)
    for N, warm in ((300, 0), (517, 40)):
        r3 = orc.run([inputs.continuous(inputs.preset_closed())], k, 11, N - warm, warmup_len=warm, latencies=True)
        r4 = orc.run([inputs.continuous(inputs.preset_closed(think_us=0))], k, 11, N - warm, warmup_len=warm,
                     latencies=True)
        assert np.array_equal(r3["latencies"], r4["latencies"])
        for key in ("p99_us", "slo_met", "window_us", "sum_latency_us", "flags"):
            assert r3[key] == r4[key]
        assert r4["counters"]["philox_blocks"] == r3["counters"]["philox_blocks"] + max(0, N - C)


def test_think_requires_a_finite_mean(orc):
    w = inputs.preset_closed(think_us=1000)
    w["arrivals"]["mean_gap_q16"][0] = inputs.NO_ARRIVALS
    with pytest.raises(ValueError):
        orc.run([w], inputs.knobs(), 1, 10)
