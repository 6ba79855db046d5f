"""Pins for the oracle's event simulator against hand traces, an independent
brute-force simulator, textbook queueing results and exact invariants."""
import json
import math
import os
import random

import numpy as np
import pytest

from paper_2603_11340_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------------------------------------
# hand-enumerated traces
# ------------------------------------------------------------------------------------------------
def _traces():
    with open(os.path.join(GOLD, "traces.json")) as fh:
        return json.load(fh)["traces"]


@pytest.mark.parametrize("tr", _traces(), ids=lambda t: t["name"].split()[0])
def test_hand_traces(orc, tr):
    r = orc.run_trace(tr["timing"], tr["conc"], tr["B"], tr["gamma"], tr["max_wait_us"], tr["a"], tr["P"],
                      tr["O"], f=tr.get("f"), A=tr.get("A"), slo_us=tr["slo_us"], continuous=tr.get("continuous", 0),
                      width=tr.get("W", 1))
    ex = tr["expect"]
    assert list(r["trace"]["c"]) == ex["c"]
    if "s" in ex:
        assert list(r["trace"]["s"]) == ex["s"]
    if "latencies" in ex:
        assert list(r["latencies"]) == ex["latencies"]
    for key in ("p99_us", "slo_met", "window_us"):
        if key in ex:
            assert r[key] == ex[key]
    if "window_us" in ex:
        assert r["goodput"] == ex["slo_met"] * 1e6 / ex["window_us"]


# ------------------------------------------------------------------------------------------------
# an independent brute-force simulator: advances time one microsecond at a time
# ------------------------------------------------------------------------------------------------
def brute_force(tm, C, B, gamma, mw, a, P, O, f, A, W=1):
    """Per-microsecond time stepping of DESIGN.md §2.6 (written separately from the oracle's event loop)."""
    N = len(a)
    s = [None] * N
    c = [None] * N
    t = 0
    arrived = issued = batched = done = 0
    in_service = {}          # member -> completion time
    while done < N:
        again = True
        while again:          # several passes at the same instant only if a zero-length batch completes
            again = False
            for m, cm in list(in_service.items()):
                if cm == t:
                    del in_service[m]
                    done += 1
            while arrived < N and a[arrived] <= t:
                arrived += 1
            while issued < arrived and issued - done < C:
                s[issued] = t
                issued += 1
            if not in_service and batched < issued:
                q = issued - batched
                if mw == 0 or q >= B or t >= s[batched] + mw:
                    b = min(B, q)
                    mem = list(range(batched, batched + b))
                    fh = f[mem[0]]
                    Dp = fh * (tm["pre_base_us"] + tm["pre_tok_us"] * max(P[m] for m in mem)) // 10 ** 6
                    rem = {m: O[m] for m in mem}
                    cum, j = 0, 0
                    while rem:
                        n = len(rem)
                        if gamma == 0:
                            d = tm["dec_base_us"] + tm["dec_seq_us"] * n
                        else:
                            d = (gamma * W * (tm["dr_base_us"] + tm["dr_seq_us"] * n) + tm["ver_base_us"]
                                 + tm["ver_seq_us"] * n + tm["ver_tok_us"] * (W * gamma + 1) * n)
                        cum += d
                        for m in sorted(rem):
                            e = 1 if gamma == 0 else min(A[m][j] + 1, rem[m])
                            rem[m] -= e
                            if rem[m] == 0:
                                del rem[m]
                                c[m] = t + Dp + fh * cum // 10 ** 6
                                in_service[m] = c[m]
                        j += 1
                    batched += b
                    if any(cm == t for cm in in_service.values()):
                        again = True
        t += 1
    return s, c


def _random_trace(rng, n, gamma):
    a = sorted(rng.randrange(0, 400) for _ in range(n))
    P = [rng.randrange(1, 6) for _ in range(n)]
    O = [rng.randrange(1, 7) for _ in range(n)]
    f = [rng.choice([1_000_000, rng.randrange(900_000, 1_100_000)]) for _ in range(n)]
    A = [[rng.randrange(0, gamma + 1) for _ in range(8)] for _ in range(n)]
    return a, P, O, f, A


@pytest.mark.parametrize("case", range(300))
def test_brute_force_agreement(orc, case):
    rng = random.Random(1000 + case)
    gamma = rng.choice([0, 0, 1, 2, 3])
    tm = dict(pre_base_us=rng.randrange(0, 5), pre_tok_us=rng.randrange(0, 4), dec_base_us=rng.randrange(0, 12),
              dec_seq_us=rng.randrange(0, 4), dr_base_us=rng.randrange(0, 4), dr_seq_us=rng.randrange(0, 2),
              ver_base_us=rng.randrange(0, 8), ver_seq_us=rng.randrange(0, 3), ver_tok_us=rng.randrange(0, 2),
              noise_step_ppm=0)
    n = rng.randrange(1, 13)
    a, P, O, f, A = _random_trace(rng, n, gamma)
    C = rng.randrange(1, 6)
    B = rng.randrange(1, 6)
    mw = rng.choice([0, 0, rng.randrange(1, 60)])
    W = rng.choice([1, 1, 2, 3, 4])               # draft width in the speculative step cost (R28)
    s_bf, c_bf = brute_force(tm, C, B, gamma, mw, a, P, O, f, A, W=W)
    r = orc.run_trace(tm, C, B, gamma, mw, a, P, O, f=f, A=A if gamma else None, width=W)
    assert list(r["trace"]["c"]) == c_bf
    assert list(r["trace"]["s"]) == s_bf


# ------------------------------------------------------------------------------------------------
# textbook special case: B = 1, gamma = 0 reduces to the Lindley recursion
# ------------------------------------------------------------------------------------------------
def _noise(w3, step):
    b = (w3 & 0xFF) + ((w3 >> 8) & 0xFF) + ((w3 >> 16) & 0xFF) + (w3 >> 24)
    return 10 ** 6 + (b - 510) * step


@pytest.mark.parametrize("conc,mw", [(1, 0), (3, 0), (8, 2000), (32, 50000)])
def test_lindley_at_batch_one(orc, conc, mw):
    """At B = 1 the server is a single FCFS queue: c_i = max(a_i, c_{i-1}) + S_i (Lindley 1952) with
    S_i = D_p(P_i) + floor(f_i * O_i * (dec_base + dec_seq) / 1e6); the gate and max_wait drop out."""
    wl = inputs.preset_sim(rate=4.0)
    k = inputs.knobs(conc=conc, max_num_seqs=1, max_wait_us=mw)
    seed = inputs.seeds(1, 7)[0]
    N = 3000
    r = orc.run([wl], k, seed, N, latencies=True, trace=True)
    a, P, O, w3 = orc.request_draws([wl], k, seed, N)
    tm = wl["timing"]
    c_prev = 0
    for i in range(N):
        f = _noise(int(w3[i]), tm["noise_step_ppm"])
        S = (f * (tm["pre_base_us"] + tm["pre_tok_us"] * int(P[i])) // 10 ** 6
             + f * int(O[i]) * (tm["dec_base_us"] + tm["dec_seq_us"]) // 10 ** 6)
        c = max(int(a[i]), c_prev) + S
        assert int(r["trace"]["c"][i]) == c, i
        c_prev = c


def test_no_queue_limit(orc):
    """Gaps >> service: every request is served alone on arrival, l_i = D_p(P_i) + decode(O_i)."""
    wl = inputs.preset_ll(rate=1e-5)
    k = inputs.knobs(conc=8, max_num_seqs=16)
    seed = inputs.seeds(1, 3)[0]
    r = orc.run([wl], k, seed, 500, latencies=True)
    a, P, O, w3 = orc.request_draws([wl], k, seed, 500)
    tm = wl["timing"]
    gaps = np.diff(a.astype(np.int64))
    assert gaps.min() > 600_000  # longer than any single service (<= 64 * 7.2 ms * 1.18 + prefill)
    for i in range(500):
        f = _noise(int(w3[i]), tm["noise_step_ppm"])
        l = (f * (tm["pre_base_us"] + tm["pre_tok_us"] * int(P[i])) // 10 ** 6
             + f * int(O[i]) * (tm["dec_base_us"] + tm["dec_seq_us"]) // 10 ** 6)
        assert int(r["latencies"][i]) == l


# ------------------------------------------------------------------------------------------------
# Pollaczek-Khinchine (M/D/1) mean waiting time — statistical
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("rho", [0.5, 0.7])
def test_pollaczek_khinchine_md1(orc, rho):
    """B = 1, gamma = 0, no noise, P = 40, O = 64 (LL timing): S = 2000 + 60*40 + 64*(7000+200) = 465,200 us.
    Poisson arrivals at lambda = rho / S.  M/D/1: W_q = rho * S / (2 (1 - rho))."""
    S = 465_200
    tm = dict(inputs.LL_TIMING, noise_step_ppm=0)
    wl = inputs.workload(kind=0, rate=rho / (S * 1e-6), prompt=inputs.point_mass(40),
                         output=inputs.point_mass(64), timing=tm)
    k = inputs.knobs(conc=32, max_num_seqs=1)
    means = []
    N = 20000
    for seed in inputs.seeds(24, 100):
        r = orc.run([wl], k, seed, N, warmup_len=500)
        means.append(r["sum_latency_us"] / N - S)
    m = float(np.mean(means))
    se = float(np.std(means, ddof=1) / math.sqrt(len(means)))
    wq = rho * S / (2 * (1 - rho))
    assert abs(m - wq) < 4 * se + 0.002 * wq, (m, wq, se)


# ------------------------------------------------------------------------------------------------
# exact invariants on random Philox replicas
# ------------------------------------------------------------------------------------------------
def _check_invariants(r, k, N):
    tr = r["trace"]
    a, s, form, c, batch = (tr[x].astype(np.int64) for x in ("a", "s", "form", "c", "batch"))
    C, B, mw = k["conc"], k["max_num_seqs"], k["max_wait_us"]
    assert np.all(np.diff(a) >= 0)
    assert np.all(s >= a) and np.all(np.diff(s) >= 0)           # FIFO gate, issue in order
    assert np.all(form >= s) and np.all(c >= form)
    # batches: contiguous, in order, size <= B
    assert batch[0] == 0 and np.all(np.diff(batch) >= 0) and np.all(np.diff(batch) <= 1)
    sizes = np.bincount(batch)
    assert sizes.max() <= B
    # a batch starts only after the previous batch has fully completed (one server)
    starts = np.array([form[batch == b][0] for b in range(len(sizes))])
    ends = np.array([c[batch == b].max() for b in range(len(sizes))])
    assert np.all(starts[1:] >= ends[:-1])
    # work conservation with max_wait = 0: form = max(previous end, head issue)
    heads = np.searchsorted(batch, np.arange(len(sizes)))
    if mw == 0:
        prev = np.concatenate([[0], ends[:-1]])
        assert np.all(starts == np.maximum(prev, s[heads]))
    # in flight never exceeds C: sweep issues (+1) and completions (-1), completions first at ties
    ev = sorted([(int(t), 0, -1) for t in c] + [(int(t), 1, +1) for t in s])
    cur = 0
    for _, _, d in ev:
        cur += d
        assert cur <= C
    # gate tightness: each issue happens at its arrival or at a completion instant
    cset = set(int(x) for x in c)
    for i in range(N):
        assert s[i] == a[i] or int(s[i]) in cset
    # outputs
    lat = (c - a)
    n = N
    srt = np.sort(np.minimum(lat, 2 ** 32 - 1))
    assert r["p99_us"] == srt[(99 * n + 99) // 100 - 1]
    assert r["slo_met"] == int(np.sum(lat <= 1_200_000))
    assert r["window_us"] == max(1, int(c.max() - a[0]))
    assert r["slo_met"] <= n                                      # goodput <= throughput


@pytest.mark.parametrize("case", range(40))
def test_invariants_random_replicas(orc, case):
    rng = random.Random(case)
    wls = [inputs.preset_ll(rate=rng.choice([5.0, 10.0, 20.0])), inputs.preset_sim(),
           inputs.preset_stress(kind=1), inputs.preset_stress(kind=2)]
    k = inputs.random_knobs(rng, n_wl=len(wls))
    N = rng.choice([50, 300, 1000])
    r = orc.run(wls, k, inputs.seeds(1, case)[0], N, trace=True, latencies=True)
    assert r["flags"] & 1 == 0
    _check_invariants(r, k, N)


def test_spec_off_equals_zero_draft(orc):
    """spec_on = 0 is bit-identical to draft_len = 0 (DESIGN.md §2.6 gamma_eff), and under CRN every
    acceptance value gives the same replica when gamma_eff = 0."""
    wl = inputs.preset_ll()
    seed = inputs.seeds(1, 11)[0]
    base = orc.run([wl], inputs.knobs(conc=8, max_num_seqs=8), seed, 2000, latencies=True)
    for g in (4, 16):
        for a in (0.3, 0.9):
            r = orc.run([wl], inputs.knobs(conc=8, max_num_seqs=8, draft_len=g, spec_on=0,
                                           accept_q16=inputs.q16(a)), seed, 2000, latencies=True)
            assert np.array_equal(r["latencies"], base["latencies"])


def test_acceptance_extremes(orc):
    """alpha = 0: every step emits 1 token (S_m = O_m); alpha = 1: S_m = ceil(O_m / (gamma + 1))."""
    wl = inputs.preset_ll()
    seed = inputs.seeds(1, 5)[0]
    for g in (1, 3, 8):
        r0 = orc.run([wl], inputs.knobs(conc=4, max_num_seqs=4, draft_len=g, spec_on=1, accept_q16=0),
                     seed, 400, trace=True)
        assert np.array_equal(r0["trace"]["steps"], r0["trace"]["O"])
        r1 = orc.run([wl], inputs.knobs(conc=4, max_num_seqs=4, draft_len=g, spec_on=1, accept_q16=65536),
                     seed, 400, trace=True)
        assert np.array_equal(r1["trace"]["steps"], (r1["trace"]["O"] + g) // (g + 1))


def test_mean_steps_leviathan(orc):
    """With alpha = .5, gamma = 4, the mean tokens per step over all (uncapped) steps approaches
    Leviathan's (1 - alpha^5)/(1 - alpha) = 1.9375; the cap only lowers the last step."""
    wl = inputs.workload(kind=0, rate=1.0, prompt=inputs.point_mass(10), output=inputs.point_mass(4000))
    r = orc.run([wl], inputs.knobs(conc=1, max_num_seqs=1, draft_len=4, spec_on=1,
                                   accept_q16=inputs.q16(0.5)), inputs.seeds(1, 0)[0], 200, trace=True)
    tokens = r["trace"]["O"].sum()
    steps = r["trace"]["steps"].sum()
    assert abs(tokens / steps - 1.9375) < 0.02


def test_p_mono_batch_one(orc):
    """B = 1: every latency is pathwise non-decreasing in the arrival rate under CRN (per-gap floors)."""
    wl = inputs.preset_ll()
    seed = inputs.seeds(1, 21)[0]
    prev = None
    for q8 in (200, 256, 300, 400):
        r = orc.run([wl], inputs.knobs(conc=8, max_num_seqs=1, rate_scale_q8=q8), seed, 1500, latencies=True)
        if prev is not None:
            assert np.all(r["latencies"].astype(np.int64) >= prev.astype(np.int64))
        prev = r["latencies"]


def test_slo_met_monotone_in_slo(orc):
    wl = inputs.preset_ll()
    k = inputs.knobs(conc=8, max_num_seqs=8, draft_len=8, spec_on=1)
    seed = inputs.seeds(1, 2)[0]
    prev = -1
    for slo in (100_000, 600_000, 1_200_000, 3_000_000, 50_000_000):
        r = orc.run([wl], k, seed, 2000, slo_us=slo)
        assert r["slo_met"] >= prev and r["slo_met"] <= r["n_measured"]
        prev = r["slo_met"]


def test_warmup_excluded(orc):
    """warmup requests are simulated but excluded from every output (R16)."""
    wl = inputs.preset_ll()
    k = inputs.knobs(conc=8, max_num_seqs=16)
    seed = inputs.seeds(1, 9)[0]
    full = orc.run([wl], k, seed, 1500, latencies=True, trace=True)
    w = orc.run([wl], k, seed, 1000, warmup_len=500, latencies=True)
    assert np.array_equal(full["latencies"], w["latencies"])
    lat = full["latencies"][500:]
    assert w["sum_latency_us"] == int(lat.astype(np.int64).sum())
    assert w["p99_us"] == int(np.sort(lat)[(99 * 1000 + 99) // 100 - 1])
    assert w["window_us"] == int(full["trace"]["c"][500:].max() - full["trace"]["a"][500])


def test_trend_batching_and_bursts(orc):
    """Paper trends (qualitative): B = 1 drives p99 far above the SLO; bursty arrivals at the same
    mean rate give a higher p99 than steady ones (seed means)."""
    wl = inputs.preset_ll()
    seeds = inputs.seeds(6, 40)
    p1 = np.mean([orc.run([wl], inputs.knobs(conc=16, max_num_seqs=1), s, 1500)["p99_us"] for s in seeds])
    p8 = np.mean([orc.run([wl], inputs.knobs(conc=16, max_num_seqs=8), s, 1500)["p99_us"] for s in seeds])
    assert p1 > 2 * 1_200_000 and p8 < p1
    st = inputs.preset_stress(kind=1)
    steady = inputs.workload(kind=0, rate=10.0, prompt=st["prompt"], output=st["output"])
    kk = inputs.knobs(conc=16, max_num_seqs=8)
    pb = np.mean([orc.run([st], kk, s, 1500)["p99_us"] for s in seeds])
    ps = np.mean([orc.run([steady], kk, s, 1500)["p99_us"] for s in seeds])
    assert pb > ps


def test_invalid_knobs(orc):
    r = orc.run([inputs.preset_ll()], inputs.knobs(conc=0), 1, 100)
    assert r["flags"] == 1 and r["p99_us"] == 2 ** 32 - 1 and r["goodput"] == -1.0 and r["slo_met"] == 0


def test_p99_nearest_rank_examples():
    """SPEC S:123-128 nearest-rank examples, applied with DESIGN.md's rank r = (99n+99) div 100 (q=.99)
    and its general form ceil(q n)."""
    def nearest_rank(xs, num, den):
        n = len(xs)
        r = (num * n + den - 1) // den
        return sorted(xs)[r - 1]
    assert nearest_rank(list(range(1, 101)), 99, 100) == 99
    assert nearest_rank([7], 99, 100) == 7
    assert nearest_rank([3, 1, 2], 1, 2) == 2
    assert nearest_rank([500] * 99 + [5000], 99, 100) == 500   # R23: S:145 contradicts S:123


# ------------------------------------------------------------------------------------------------
# NEXT-1: closed-loop clients (kind 3, zero think time, latency from issue) and p50 / p95
# ------------------------------------------------------------------------------------------------
def _closed(P=40, O=64, noise=0):
    w = inputs.preset_closed()
    w["prompt"] = inputs.point_mass(P)
    w["output"] = inputs.point_mass(O)
    w["timing"] = dict(inputs.LL_TIMING, noise_step_ppm=noise)
    return w


@pytest.mark.parametrize("C,B", [(4, 8), (8, 8), (8, 2), (12, 4), (16, 16)])
def test_closed_loop_closed_form(orc, C, B):
    """Deterministic service, C users, zero think time: batches of b = min(B, C) run back to back, each
    taking D = pre_base + pre_tok P + O (dec_base + dec_seq b).  The first C requests (all issued at 0) wait
    for floor(i/b) batches; afterwards, with C a multiple of b, every request waits C/b - 1 batches, so its
    latency from issue is (C/b) D and the throughput is b/D (Little's law for a closed system: C = X R)."""
    tm = inputs.LL_TIMING
    b = min(B, C)
    D = tm["pre_base_us"] + tm["pre_tok_us"] * 40 + 64 * (tm["dec_base_us"] + tm["dec_seq_us"] * b)
    N = 40 * C
    r = orc.run([_closed()], inputs.knobs(conc=C, max_num_seqs=B), 7, N, latencies=True, trace=True)
    lat = r["latencies"].astype(np.int64)
    assert np.all(lat[:C] == (np.arange(C) // b + 1) * D)
    assert np.all(lat[C:] == (C // b) * D)
    assert r["p50_us"] == r["p95_us"] == r["p99_us"] == (C // b) * D
    assert r["window_us"] == (N // b) * D                 # first issue at 0, last completion after N/b batches
    tr = r["trace"]
    assert np.all(tr["a"] == 0) and np.all(tr["s"][:C] == 0)


def test_closed_loop_matches_brute_force(orc):
    """Trace mode with every a_i = 0 and issue-origin latencies equals the per-microsecond brute force."""
    rng = random.Random(77)
    for case in range(60):
        gamma = rng.choice([0, 0, 2])
        tm = dict(pre_base_us=rng.randrange(0, 5), pre_tok_us=rng.randrange(0, 4), dec_base_us=rng.randrange(1, 12),
                  dec_seq_us=rng.randrange(0, 4), dr_base_us=rng.randrange(0, 4), dr_seq_us=rng.randrange(0, 2),
                  ver_base_us=rng.randrange(0, 8), ver_seq_us=rng.randrange(0, 3), ver_tok_us=rng.randrange(0, 2),
                  noise_step_ppm=0)
        n = rng.randrange(1, 12)
        _, P, O, f, A = _random_trace(rng, n, gamma)
        a = [0] * n
        C, B = rng.randrange(1, 6), rng.randrange(1, 6)
        s_bf, c_bf = brute_force(tm, C, B, gamma, 0, a, P, O, f, A)
        r = orc.run_trace(tm, C, B, gamma, 0, a, P, O, f=f, A=A if gamma else None, issue_origin=1)
        assert list(r["latencies"]) == [c - s for c, s in zip(c_bf, s_bf)]


def test_percentiles_nearest_rank(orc):
    """p50 / p95 / p99 are the ceil(q n)-th smallest measured latencies, monotone in q."""
    for k, wl in ((inputs.knobs(conc=8, max_num_seqs=4, draft_len=4, spec_on=1), inputs.preset_ll()),
                  (inputs.knobs(conc=6, max_num_seqs=3), inputs.preset_closed()),
                  (inputs.knobs(conc=12, max_num_seqs=6), inputs.preset_stress())):
        for n, w in ((1, 0), (7, 3), (100, 0), (1999, 17)):
            r = orc.run([wl], k, 5, n, warmup_len=w, latencies=True)
            srt = np.sort(r["latencies"][w:])
            for key, q in (("p50_us", 50), ("p95_us", 95), ("p99_us", 99)):
                assert r[key] == srt[(q * n + 99) // 100 - 1]
            assert r["p50_us"] <= r["p95_us"] <= r["p99_us"]


# ------------------------------------------------------------------------------------------------
# NEXT-2: continuous (iteration-level) batching
# ------------------------------------------------------------------------------------------------
def brute_force_continuous(tm, C, B, gamma, a, P, O, f, A, issue_origin=False, W=1):
    """Per-microsecond time stepping of DESIGN.md §2.12 (written separately from the oracle)."""
    N = len(a)
    s, c = [None] * N, [None] * N
    rem = list(O)
    steps = [0] * N
    t = arrived = issued = admitted = done = 0
    running, joining, finishing = [], [], []
    end = None                      # end instant of the current iteration (None: server free)
    while done < N:
        again = True
        while again:
            again = False
            if end == t:
                for m in finishing:
                    c[m] = t
                    done += 1
                running = [m for m in running if m not in finishing] + joining
                finishing, joining, end = [], [], None
            while arrived < N and a[arrived] <= t:
                arrived += 1
            while issued < arrived and issued - done < C:
                s[issued] = t
                issued += 1
            if end is None:
                if len(running) < B and admitted < issued:
                    k = min(B - len(running), issued - admitted)
                    new = list(range(admitted, admitted + k))
                    admitted += k
                    D = f[new[0]] * (tm["pre_base_us"] + tm["pre_tok_us"] * max(P[m] for m in new)) // 10 ** 6
                    joining, end = new, t + D
                elif running:
                    n = len(running)
                    if gamma == 0:
                        d = tm["dec_base_us"] + tm["dec_seq_us"] * n
                    else:
                        d = (gamma * W * (tm["dr_base_us"] + tm["dr_seq_us"] * n) + tm["ver_base_us"]
                             + tm["ver_seq_us"] * n + tm["ver_tok_us"] * (W * gamma + 1) * n)
                    for m in running:
                        e = 1 if gamma == 0 else min(A[m][steps[m]] + 1, rem[m])
                        rem[m] -= e
                        steps[m] += 1
                        if rem[m] == 0:
                            finishing.append(m)
                    end = t + d
                if end == t:
                    again = True
        t += 1
    origin = s if issue_origin else a
    return s, c, [ci - oi for ci, oi in zip(c, origin)]


@pytest.mark.parametrize("case", range(150))
def test_continuous_brute_force_agreement(orc, case):
    rng = random.Random(5000 + case)
    gamma = rng.choice([0, 0, 1, 3])
    tm = dict(pre_base_us=rng.randrange(0, 5), pre_tok_us=rng.randrange(0, 4), dec_base_us=rng.randrange(0, 12),
              dec_seq_us=rng.randrange(0, 4), dr_base_us=rng.randrange(0, 4), dr_seq_us=rng.randrange(0, 2),
              ver_base_us=rng.randrange(0, 8), ver_seq_us=rng.randrange(0, 3), ver_tok_us=rng.randrange(0, 2),
              noise_step_ppm=0)
    n = rng.randrange(1, 12)
    a, P, O, f, A = _random_trace(rng, n, gamma)
    A = [row + [rng.randrange(0, gamma + 1) for _ in range(8)] for row in A]
    closed = rng.random() < 0.3
    if closed:
        a = [0] * n
    C, B = rng.randrange(1, 6), rng.randrange(1, 6)
    W = rng.choice([1, 1, 2, 3, 4])
    s_bf, c_bf, l_bf = brute_force_continuous(tm, C, B, gamma, a, P, O, f, A, issue_origin=closed, W=W)
    r = orc.run_trace(tm, C, B, gamma, 0, a, P, O, f=f, A=A if gamma else None, continuous=1,
                      issue_origin=int(closed), width=W)
    assert list(r["trace"]["c"]) == c_bf and list(r["trace"]["s"]) == s_bf
    assert list(r["latencies"]) == l_bf


@pytest.mark.parametrize("wl", ["ll", "sim", "stress", "closed"])
def test_continuous_equals_static_at_batch_one(orc, wl):
    """With B = 1 and no noise, a prefill iteration followed by the request's decode iterations is exactly a
    static batch of one (same cumulative cost, no per-iteration floors to differ)."""
    w = {"ll": inputs.preset_ll(), "sim": inputs.preset_sim(), "stress": inputs.preset_stress(),
         "closed": inputs.preset_closed()}[wl]
    w["timing"] = dict(w["timing"], noise_step_ppm=0)
    for k in (inputs.knobs(conc=4, max_num_seqs=1), inputs.knobs(conc=9, max_num_seqs=1, draft_len=4, spec_on=1,
                                                                  accept_q16=inputs.q16(0.7))):
        st = orc.run([w], k, 13, 800, latencies=True)
        ct = orc.run([inputs.continuous(w)], k, 13, 800, latencies=True)
        assert np.array_equal(st["latencies"], ct["latencies"])
        assert st["counters"]["member_steps"] == ct["counters"]["member_steps"]


def test_continuous_invariants(orc):
    """Running set never exceeds B, in-flight never exceeds C, admission is FCFS, every request completes
    after its admission; goodput <= throughput."""
    rng = random.Random(9)
    for _ in range(20):
        wls = [inputs.continuous(inputs.preset_ll(rate=rng.choice([5.0, 10.0, 30.0]))),
               inputs.continuous(inputs.preset_stress()), inputs.continuous(inputs.preset_closed())]
        k = inputs.random_knobs(rng, n_wl=3)
        N = rng.choice([50, 400])
        r = orc.run(wls, k, rng.getrandbits(64), N, trace=True)
        tr = r["trace"]
        a, s, form, c = (tr[x].astype(np.int64) for x in ("a", "s", "form", "c"))
        assert np.all(s >= a) and np.all(np.diff(s) >= 0) and np.all(np.diff(form) >= 0)
        assert np.all(form >= s) and np.all(c > form - 1)
        ev = sorted([(int(t), 0, -1) for t in c] + [(int(t), 1, +1) for t in s])
        cur = 0
        for _, _, d in ev:
            cur += d
            assert cur <= k["conc"]
        # running set (admitted, not completed) never exceeds B
        ev = sorted([(int(t), 0, -1) for t in c] + [(int(t), 1, +1) for t in form])
        cur = 0
        for _, _, d in ev:
            cur += d
            assert cur <= k["max_num_seqs"]
        assert r["slo_met"] <= r["n_measured"]


# NEXT-3: the paper's segment stop rule ("minimum duration and minimum number of completions"),
# DESIGN.md §2.14
def _stop_trace(orc, n_min, t_min):
    tm = dict(pre_base_us=100, pre_tok_us=0, dec_base_us=10, dec_seq_us=0, dr_base_us=0, dr_seq_us=0,
              ver_base_us=0, ver_seq_us=0, ver_tok_us=0, noise_step_ppm=0)
    # C = B = 1, five one-token requests waiting at t = 0: served back to back, 110 us each
    return orc.run_trace(tm, 1, 1, 0, 0, [0] * 5, [1] * 5, [1] * 5, warmup_len=1, slo_us=250,
                         stop_n_min=n_min, stop_t_min_us=t_min)


def test_stop_rule_hand_trace(orc):
    """Completions 110, 220, 330, 440, 550 us; request 0 is warmup, t0 = a_1 = 0."""
    U = 0xFFFFFFFF
    r = _stop_trace(orc, 2, 300)          # k >= 2 and c >= 300: t* = 330 -> requests 1, 2
    assert list(r["latencies"]) == [110, 220, 330, U, U]
    assert (r["n_measured"], r["p99_us"], r["slo_met"], r["window_us"], r["flags"]) == (2, 330, 1, 330, 0)
    r = _stop_trace(orc, 3, 0)            # the third measured completion: t* = 440
    assert (r["n_measured"], r["window_us"], list(r["latencies"])[-1]) == (3, 440, U)
    r = _stop_trace(orc, 1, 500)          # the first completion at or after 500 us: t* = 550, all four
    assert (r["n_measured"], r["window_us"], r["flags"]) == (4, 550, 0)
    r = _stop_trace(orc, 5, 0)            # only four measured requests: the source runs out, flag bit 2
    assert (r["n_measured"], r["window_us"], r["flags"]) == (4, 550, 4)
    r0 = _stop_trace(orc, 0, 0)           # off: the fixed-count segment of R15
    assert (r0["n_measured"], r0["window_us"], r0["flags"]) == (4, 550, 0)


@pytest.mark.parametrize("cont", [0, 1])
def test_stop_rule_properties(orc, cont):
    """Philox mode, static and continuous batching: off and "all of the segment" reproduce the fixed-count
    outputs; the counted set is a prefix of the completion order that grows with n_min and t_min; the counted
    requests keep their latencies and the rest store the sentinel."""
    rng = random.Random(11 + cont)
    for _ in range(12):
        w = inputs.preset_ll(rate=rng.choice([5.0, 10.0, 40.0]))
        if cont:
            w = inputs.continuous(w)
        k = inputs.random_knobs(rng, max_wait=not cont)
        k["workload"] = 0
        seg, warm = rng.choice([(300, 0), (500, 40)])
        seed = rng.randrange(1 << 30)
        base = orc.run([w], k, seed, seg, warmup_len=warm, latencies=True, trace=True)
        full = orc.run([w], k, seed, seg, warmup_len=warm, latencies=True, stop_n_min=seg)
        for f in ("p99_us", "slo_met", "n_measured", "window_us", "sum_latency_us", "flags", "goodput"):
            assert full[f] == base[f], f
        c = base["trace"]["c"]
        cm = np.sort(c[warm:])
        t0 = int(base["trace"]["s" if w["arrivals"]["kind"] == 3 else "a"][warm])
        for n_min, t_min in ((1, 0), (seg // 4, 0), (seg // 2, 10**6), (1, 5 * 10**6), (seg // 3, 2 * 10**6)):
            r = orc.run([w], k, seed, seg, warmup_len=warm, latencies=True, stop_n_min=n_min, stop_t_min_us=t_min)
            ok = [i for i in range(n_min, seg + 1) if cm[i - 1] >= t0 + t_min]
            tstar = int(cm[ok[0] - 1]) if ok else int(cm[-1])
            inc = c <= tstar
            assert r["n_measured"] == int(inc[warm:].sum()) >= (n_min if ok else 0)
            assert (r["flags"] & 4) == (0 if ok else 4)
            lat = r["latencies"]
            assert np.array_equal(lat[inc], base["latencies"][inc]) and np.all(lat[~inc] == 0xFFFFFFFF)
            assert r["window_us"] == max(1, int(c[warm:][inc[warm:]].max()) - t0)
