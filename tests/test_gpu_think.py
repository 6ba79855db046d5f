"""GPU parity of the closed loop with exponential think time (arrival kind 4; K1t):
every latency, percentile, output field and work counter bit-exact against the oracle, in a launch that
mixes kind-4 replicas with every other arrival kind."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2603_11340_b200 import inputs  # noqa: E402


@pytest.fixture(scope="module")
def S():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2603_11340_b200 import sim
    assert torch.cuda.is_available()
    return sim


def _wls():
    sim_think = inputs.preset_closed(stream_id=8, think_us=40_000)
    sim_think["timing"] = dict(inputs.preset_sim()["timing"])
    return [inputs.preset_ll(), inputs.preset_stress(kind=1), inputs.preset_closed(stream_id=3),
            inputs.preset_closed(stream_id=5, think_us=300_000), inputs.preset_closed(stream_id=6, think_us=0),
            sim_think, inputs.preset_closed(stream_id=9, think_us=5_000_000)]


def _knobs(rng, wls):
    ks = [inputs.random_knobs(rng, n_wl=len(wls)) for _ in range(28)]
    ks[0] = inputs.knobs(conc=32, max_num_seqs=32, draft_len=16, spec_on=1, workload=3)       # G = 32
    ks[1] = inputs.knobs(conc=1, max_num_seqs=1, workload=3)                                  # one user
    ks[2] = inputs.knobs(conc=32, max_num_seqs=1, max_wait_us=50_000, workload=4)            # Z = 0
    ks[3] = inputs.knobs(conc=5, max_num_seqs=16, draft_len=4, spec_on=1, workload=5)        # G = 16
    ks[4] = inputs.knobs(conc=8, max_num_seqs=8, max_wait_us=30_000, workload=3)             # G = 8
    ks[5] = inputs.knobs(conc=24, max_num_seqs=6, workload=6, rate_scale_q8=64)              # long thinks
    ks[6] = inputs.knobs(conc=9, max_num_seqs=3, draft_len=2, spec_on=1, workload=2)         # kind 3 beside
    return ks


def _fetch(S, out, R, N):
    from paper_2603_11340_b200._lib import RESULT_DTYPE, STATS_DTYPE
    torch.cuda.synchronize()
    return dict(lat=out["latencies"].cpu().numpy().view(np.uint32).reshape(R, N),
                p99=out["p99_us"].cpu().numpy().view(np.uint32), p50=out["p50_us"].cpu().numpy().view(np.uint32),
                p95=out["p95_us"].cpu().numpy().view(np.uint32), gp=out["goodput"].cpu().numpy(),
                det=S.unpack(out["detail"], RESULT_DTYPE),
                stats=S.unpack(out["stats"], STATS_DTYPE)[0] if "stats" in out else None)


def _check(g, r, ref, tag):
    assert np.array_equal(g["lat"][r], ref["latencies"]), tag
    assert int(g["p99"][r]) == ref["p99_us"] and int(g["p50"][r]) == ref["p50_us"], tag
    assert int(g["p95"][r]) == ref["p95_us"] and g["gp"][r] == ref["goodput"], tag
    d = g["det"][r]
    for f in ("slo_met", "n_measured", "flags", "window_us", "sum_latency_us"):
        assert int(d[f]) == ref[f], (tag, f)


@pytest.mark.parametrize("policy", [1, 2, 3], ids=["narrow", "wide", "warp"])
@pytest.mark.parametrize("block", range(3))
def test_think_random_configs(S, orc, block, policy):
    rng = random.Random(9100 + block)
    wls = _wls()
    ks = _knobs(rng, wls)
    seeds = inputs.seeds(3, 31 * block + 5)
    N = rng.choice([37, 333, 1000, 1234])
    warm = rng.choice([0, 17, 100])
    s = S.Simulator(wls, device=0, group_policy=policy)
    out = s.run_batch(S.knobs_tensor(ks), S.seeds_tensor(seeds), N, warmup_len=warm, latencies=True, stats=True,
                      percentiles=True)
    g = _fetch(S, out, len(ks) * len(seeds), N + warm)
    s.close()
    tot = dict(batches=0, decode_steps=0, member_steps=0, philox_blocks=0)
    n_think = 0
    for ci, k in enumerate(ks):
        for si, sd in enumerate(seeds):
            ref = orc.run(wls, k, sd, N, warmup_len=warm, latencies=True)
            _check(g, ci * len(seeds) + si, ref, f"replica {ci},{si} knobs {k}")
            for f in tot:
                tot[f] += ref["counters"][f]
            n_think += wls[k["workload"]]["arrivals"]["kind"] == 4
    assert n_think >= 5 * len(seeds)
    for f in tot:
        assert int(g["stats"][f]) == tot[f], f


def test_think_stop_rule(S, orc):
    """The §2.14 stop rule on kind-4 replicas (K1t's stop-rule instantiation)."""
    rng = random.Random(9200)
    wls = _wls()
    ks = _knobs(rng, wls)[:10]
    seeds = inputs.seeds(2, 77)
    N, warm = 700, 30
    s = S.Simulator(wls, device=0)
    for n_min, t_min in ((50, 0), (1, 3_000_000), (300, 20_000_000), (10, 10**9)):
        out = s.run_batch(S.knobs_tensor(ks), S.seeds_tensor(seeds), N, warmup_len=warm, latencies=True,
                          percentiles=True, stop_n_min=n_min, stop_t_min_us=t_min)
        g = _fetch(S, out, len(ks) * len(seeds), N + warm)
        for ci, k in enumerate(ks):
            for si, sd in enumerate(seeds):
                ref = orc.run(wls, k, sd, N, warmup_len=warm, latencies=True, stop_n_min=n_min,
                              stop_t_min_us=t_min)
                _check(g, ci * len(seeds) + si, ref, f"stop {n_min},{t_min} replica {ci},{si}")
    s.close()


def test_think_full_size_sampled(S, orc):
    """A C2-sized grid of kind-4 replicas (512 configs x 64 seeds x 10k requests, 300 ms mean think) in the
    default launch; sampled replicas recomputed one by one by the oracle."""
    wls = [inputs.preset_closed(think_us=300_000)]
    ks = [inputs.knobs(conc=c, max_num_seqs=b, draft_len=g, spec_on=int(g > 0), accept_q16=32768)
          for c in range(1, 17) for b in range(2, 17, 2) for g in (0, 4, 8, 16)]
    seeds = inputs.seeds(64, 0)
    N = 10_000
    s = S.Simulator(wls, device=0)
    out = s.run_batch(S.knobs_tensor(ks), S.seeds_tensor(seeds), N, latencies=True, percentiles=True)
    g = _fetch(S, out, len(ks) * len(seeds), N)
    s.close()
    rng = random.Random(3)
    rows = sorted({0, len(ks) * len(seeds) - 1} | {rng.randrange(len(ks) * len(seeds)) for _ in range(10)})
    for r in rows:
        ref = orc.run(wls, ks[r // len(seeds)], seeds[r % len(seeds)], N, latencies=True)
        _check(g, r, ref, f"row {r}")


def _wls_cont():
    c = inputs.continuous
    return [c(inputs.preset_ll()), c(inputs.preset_closed(stream_id=3)),
            c(inputs.preset_closed(stream_id=5, think_us=300_000)), c(inputs.preset_closed(stream_id=6, think_us=0)),
            c(inputs.preset_closed(stream_id=9, think_us=5_000_000)), inputs.preset_closed(stream_id=8, think_us=40_000)]


@pytest.mark.parametrize("policy", [1, 2, 3], ids=["narrow", "wide", "warp"])
@pytest.mark.parametrize("block", range(3))
def test_think_continuous_random_configs(S, orc, block, policy):
    """Kind 4 under continuous batching (K1c's think-time instantiation, lists 9-11) beside plain continuous,
    zero-think continuous and static think-time replicas in one launch."""
    rng = random.Random(9300 + block)
    wls = _wls_cont()
    ks = [inputs.random_knobs(rng, n_wl=len(wls)) for _ in range(24)]
    ks[0] = inputs.knobs(conc=32, max_num_seqs=32, draft_len=16, spec_on=1, workload=2)
    ks[1] = inputs.knobs(conc=1, max_num_seqs=1, workload=2)
    ks[2] = inputs.knobs(conc=32, max_num_seqs=3, workload=3)
    ks[3] = inputs.knobs(conc=5, max_num_seqs=16, draft_len=4, spec_on=1, workload=4, rate_scale_q8=64)
    ks[4] = inputs.knobs(conc=12, max_num_seqs=12, workload=2)
    seeds = inputs.seeds(3, 11 * block + 1)
    N = rng.choice([37, 333, 1000])
    warm = rng.choice([0, 17, 100])
    s = S.Simulator(wls, device=0, group_policy=policy)
    out = s.run_batch(S.knobs_tensor(ks), S.seeds_tensor(seeds), N, warmup_len=warm, latencies=True, stats=True,
                      percentiles=True)
    g = _fetch(S, out, len(ks) * len(seeds), N + warm)
    s.close()
    tot = dict(batches=0, decode_steps=0, member_steps=0, philox_blocks=0)
    for ci, k in enumerate(ks):
        for si, sd in enumerate(seeds):
            ref = orc.run(wls, k, sd, N, warmup_len=warm, latencies=True)
            _check(g, ci * len(seeds) + si, ref, f"replica {ci},{si} knobs {k}")
            for f in tot:
                tot[f] += ref["counters"][f]
    for f in tot:
        assert int(g["stats"][f]) == tot[f], f


def test_think_continuous_stop_rule(S, orc):
    rng = random.Random(9400)
    wls = _wls_cont()
    ks = [inputs.random_knobs(rng, n_wl=len(wls)) for _ in range(10)]
    ks[0] = inputs.knobs(conc=12, max_num_seqs=4, workload=2)
    seeds = inputs.seeds(2, 78)
    N, warm = 700, 30
    s = S.Simulator(wls, device=0)
    for n_min, t_min in ((50, 0), (1, 3_000_000), (300, 20_000_000), (10, 10**9)):
        out = s.run_batch(S.knobs_tensor(ks), S.seeds_tensor(seeds), N, warmup_len=warm, latencies=True,
                          percentiles=True, stop_n_min=n_min, stop_t_min_us=t_min)
        g = _fetch(S, out, len(ks) * len(seeds), N + warm)
        for ci, k in enumerate(ks):
            for si, sd in enumerate(seeds):
                ref = orc.run(wls, k, sd, N, warmup_len=warm, latencies=True, stop_n_min=n_min,
                              stop_t_min_us=t_min)
                _check(g, ci * len(seeds) + si, ref, f"stop {n_min},{t_min} replica {ci},{si}")
    s.close()


def test_think_create_validation(S):
    from paper_2603_11340_b200._lib import SloError
    w = inputs.preset_closed(think_us=1000)
    w["arrivals"]["mean_gap_q16"][0] = inputs.NO_ARRIVALS
    with pytest.raises(SloError):
        S.Simulator([w], device=0)
