"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element, bit-exact.

Integer outputs (every latency, p99, slo_met, window, sum, flags, work counters) and the goodput double
must be identical (the model is integer-exact; goodput is one IEEE division on both sides).
"""
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


def _run_gpu(sim, wls, ks, seeds, N, warmup=0, slo=1_200_000, crn=1, latencies=True, sim_obj=None, **kw):
    s = sim_obj or sim.Simulator(wls, device=0, crn=crn, **kw)
    out = s.run_batch(sim.knobs_tensor(ks), sim.seeds_tensor(seeds), N, warmup_len=warmup, slo_us=slo,
                      latencies=latencies, stats=True, percentiles=True)
    torch.cuda.synchronize()
    from paper_2603_11340_b200._lib import RESULT_DTYPE, STATS_DTYPE
    res = dict(p99=out["p99_us"].cpu().numpy().view(np.uint32), gp=out["goodput"].cpu().numpy(),
               p50=out["p50_us"].cpu().numpy().view(np.uint32), p95=out["p95_us"].cpu().numpy().view(np.uint32),
               detail=sim.unpack(out["detail"], RESULT_DTYPE), stats=sim.unpack(out["stats"], STATS_DTYPE)[0])
    if latencies:
        res["lat"] = out["latencies"].cpu().numpy().view(np.uint32).reshape(len(ks) * len(seeds), N + warmup)
    if sim_obj is None:
        s.close()
    return res


def _compare_replica(orc, g, r, wls, k, seed, N, warmup, slo, crn=1, check_lat=True):
    ref = orc.run(wls, k, seed, N, warmup_len=warmup, slo_us=slo, crn=crn, latencies=check_lat)
    d = g["detail"][r]
    tag = f"replica {r} knobs {k}"
    if check_lat:
        assert np.array_equal(g["lat"][r], ref["latencies"]), tag
    assert int(g["p99"][r]) == ref["p99_us"], tag
    assert int(g["p50"][r]) == ref["p50_us"] and int(g["p95"][r]) == ref["p95_us"], tag
    assert g["gp"][r] == ref["goodput"], tag
    assert int(d["p99_us"]) == ref["p99_us"] and int(d["slo_met"]) == ref["slo_met"], tag
    assert int(d["n_measured"]) == ref["n_measured"] and int(d["flags"]) == ref["flags"], tag
    assert int(d["window_us"]) == ref["window_us"] and int(d["sum_latency_us"]) == ref["sum_latency_us"], tag
    return ref


def test_c1_full_bit_exact(S, orc):
    """BASELINE config 1 in full: 1 replica x 2,000 requests, every latency."""
    cfg = inputs.config_c1()
    g = _run_gpu(S, cfg.workloads, cfg.knobs, cfg.seeds(), cfg.segment_len)
    ref = _compare_replica(orc, g, 0, cfg.workloads, cfg.knobs[0], cfg.seeds()[0], cfg.segment_len, 0, cfg.slo_us)
    st = g["stats"]
    c = ref["counters"]
    assert int(st["requests"]) == 2000 and int(st["batches"]) == c["batches"]
    assert int(st["decode_steps"]) == c["decode_steps"] and int(st["member_steps"]) == c["member_steps"]
    assert int(st["philox_blocks"]) == c["philox_blocks"]


WLS = None


def _wls():
    return [inputs.preset_ll(), inputs.preset_sim(), inputs.preset_stress(kind=1), inputs.preset_stress(kind=2),
            inputs.preset_ll(rate=40.0, stream_id=7), inputs.preset_closed(stream_id=3)]


@pytest.mark.parametrize("gen", [1, 2], ids=["inline", "split"])
@pytest.mark.parametrize("policy", [1, 2, 3], ids=["narrow", "wide", "warp"])
@pytest.mark.parametrize("block", range(6))
def test_random_small_configs(S, orc, block, policy, gen):
    """Random valid knob records over every workload kind, lengths spanning several 32-request windows
    and a ragged tail, warmup on/off — every latency and output bit-exact, plus the work counters; in both
    lane-group policies (narrow G >= min(C, B), the throughput default; wide G >= max(C, B))."""
    rng = random.Random(500 + block)
    wls = _wls()
    ks = [inputs.random_knobs(rng, n_wl=len(wls)) for _ in range(24)]
    ks[0] = inputs.knobs(conc=32, max_num_seqs=32, draft_len=16, spec_on=1, accept_q16=65536, workload=1)
    ks[1] = inputs.knobs(conc=1, max_num_seqs=1, draft_len=16, spec_on=1, accept_q16=0)
    ks[2] = inputs.knobs(conc=32, max_num_seqs=1, max_wait_us=50_000, workload=2)
    ks[3] = inputs.knobs(conc=1, max_num_seqs=32, max_wait_us=50_000, workload=3)
    ks[4] = inputs.knobs(conc=24, max_num_seqs=6, draft_len=4, spec_on=1, workload=5)       # closed loop, G = 32
    ks[5] = inputs.knobs(conc=8, max_num_seqs=8, workload=5, max_wait_us=30_000)           # closed loop, G = 8
    seeds = inputs.seeds(3, 77 * block)
    ks[6] = inputs.knobs(conc=32, max_num_seqs=8, draft_len=3, spec_on=1, workload=4)     # C + B = 40 > 4G
    ks[7] = inputs.knobs(conc=30, max_num_seqs=2, max_wait_us=20_000, workload=4)
    N = rng.choice([37, 333, 1000, 1234])
    warmup = rng.choice([0, 0, 17, 100])
    g = _run_gpu(S, wls, ks, seeds, N, warmup=warmup, group_policy=policy, gen_policy=gen)
    tot = dict(batches=0, decode_steps=0, member_steps=0, philox_blocks=0)
    for ci, k in enumerate(ks):
        for si, sd in enumerate(seeds):
            ref = _compare_replica(orc, g, ci * len(seeds) + si, wls, k, sd, N, warmup, 1_200_000)
            for f in tot:
                tot[f] += ref["counters"][f]
    for f in tot:
        assert int(g["stats"][f]) == tot[f], f


@pytest.mark.parametrize("gen", [1, 2], ids=["inline", "split"])
@pytest.mark.parametrize("policy", [1, 2], ids=["narrow", "wide"])
def test_edge_cases(S, orc, policy, gen):
    """Degenerate sizes and values: one request, N < 32, invalid records, saturating SLO, zero noise."""
    wls = [inputs.preset_ll(), inputs.workload(kind=0, rate=1000.0, timing=dict(inputs.LL_TIMING, noise_step_ppm=0))]
    ks = [inputs.knobs(conc=8, max_num_seqs=16), inputs.knobs(conc=0), inputs.knobs(max_num_seqs=33),
          inputs.knobs(draft_len=17, spec_on=1), inputs.knobs(workload=2), dict(inputs.knobs(), reserved=[0, 1, 0, 0]),
          inputs.knobs(conc=32, max_num_seqs=32, workload=1), inputs.knobs(conc=3, max_num_seqs=2, workload=1,
                                                                          draft_len=3, spec_on=1)]
    seeds = inputs.seeds(2, 900)
    for N, warm in ((1, 0), (1, 5), (31, 0), (32, 1), (33, 0), (65, 64)):
        g = _run_gpu(S, wls, ks, seeds, N, warmup=warm, group_policy=policy, gen_policy=gen)
        for ci, k in enumerate(ks):
            for si, sd in enumerate(seeds):
                r = ci * len(seeds) + si
                valid = orc.knobs_valid(k, len(wls))
                if not valid:
                    assert int(g["p99"][r]) == 0xFFFFFFFF and g["gp"][r] == -1.0 and g["detail"][r]["flags"] == 1
                    continue
                _compare_replica(orc, g, r, wls, k, sd, N, warm, 1_200_000)


def test_independent_key_mode(S, orc):
    wls = [inputs.preset_ll()]
    ks = [inputs.knobs(conc=c, max_num_seqs=b) for c, b in ((4, 4), (8, 2), (16, 16))]
    seeds = inputs.seeds(2, 5)
    g = _run_gpu(S, wls, ks, seeds, 700, crn=0)
    for ci, k in enumerate(ks):
        for si, sd in enumerate(seeds):
            _compare_replica(orc, g, ci * 2 + si, wls, k, sd, 700, 0, 1_200_000, crn=0)


def test_slo_boundaries(S, orc):
    """ell <= SLO is inclusive (R7): SLO 0 and a huge SLO."""
    wls = [inputs.preset_ll()]
    ks = [inputs.knobs(conc=8, max_num_seqs=8, draft_len=4, spec_on=1)]
    sd = inputs.seeds(1, 3)
    for slo in (0, 1, 700_000, 0xFFFFFFFE):
        g = _run_gpu(S, wls, ks, sd, 400, slo=slo)
        _compare_replica(orc, g, 0, wls, ks[0], sd[0], 400, 0, slo)


def _sample_rows(n, k, rng, must=()):
    rows = set(must)
    while len(rows) < min(k, n):
        rows.add(rng.randrange(n))
    return sorted(rows)


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_full_size_sampled(S, orc, name):
    """BASELINE configs 2 and 3 at full size in the bench's launch configuration; sampled replicas
    (every speculation setting, the knob boundaries, random picks) recomputed one by one by the oracle."""
    cfg = inputs.config_c2() if name == "C2" else inputs.config_c3()
    g = _run_gpu(S, cfg.workloads, cfg.knobs, cfg.seeds(), cfg.segment_len, latencies=False)
    n_seeds = cfg.n_seeds
    rng = random.Random(11)
    cfg_rows = _sample_rows(len(cfg.knobs), 16, rng, must=(0, len(cfg.knobs) - 1, len(cfg.knobs) // 2))
    for ci in cfg_rows:
        for si in (0, rng.randrange(n_seeds), n_seeds - 1):
            r = ci * n_seeds + si
            _compare_replica(orc, g, r, cfg.workloads, cfg.knobs[ci], cfg.seeds()[si], cfg.segment_len, 0,
                             cfg.slo_us, check_lat=False)
    # properties that hold at any size
    d = g["detail"]
    assert np.all(d["slo_met"] <= d["n_measured"]) and np.all(d["flags"] & 1 == 0)
    assert np.all(g["gp"] <= d["n_measured"] * 1e6 / d["window_us"] + 1e-9)
    assert int(g["stats"]["requests"]) == cfg.requests


def test_c5_sampled(S, orc):
    """Stress grid (MMPP-2, BASELINE config 5): every 245th of its 10^6 configs (all C, B, gamma, alpha and
    rate levels), sampled replicas bit-exact."""
    cfg = inputs.config_c5(stride=245)                              # 4,082 configs spanning the grid
    g = _run_gpu(S, cfg.workloads, cfg.knobs, cfg.seeds(), cfg.segment_len, latencies=False)
    rng = random.Random(5)
    for ci in _sample_rows(len(cfg.knobs), 24, rng, must=(0, len(cfg.knobs) - 1)):
        si = rng.randrange(cfg.n_seeds)
        _compare_replica(orc, g, ci * cfg.n_seeds + si, cfg.workloads, cfg.knobs[ci], cfg.seeds()[si],
                         cfg.segment_len, 0, cfg.slo_us, check_lat=False)


def test_host_entry_matches_device_entry(S):
    cfg = inputs.config_c3(n_seeds=8, segment_len=600)
    s = S.Simulator(cfg.workloads, device=0)
    dev = s.run_batch(S.knobs_tensor(cfg.knobs), S.seeds_tensor(cfg.seeds()), 600, stats=True)
    torch.cuda.synchronize()
    hk = S.knobs_tensor(cfg.knobs, device="cpu").pin_memory()
    hs = S.seeds_tensor(cfg.seeds(), device="cpu").pin_memory()
    host = s.run_batch_host(hk, hs, 600, detail=True, stats=True)
    assert torch.equal(host["p99_us"], dev["p99_us"].cpu())
    assert torch.equal(host["goodput"], dev["goodput"].cpu())
    assert torch.equal(host["detail"], dev["detail"].cpu())
    assert torch.equal(host["stats"], dev["stats"].cpu())
    s.close()


def test_aggregate_kernels(S, orc):
    from oracle import climb
    from paper_2603_11340_b200._lib import AGG_DTYPE
    cfg = inputs.config_c3(n_seeds=5, segment_len=300)
    s = S.Simulator(cfg.workloads, device=0)
    out = s.run_batch(S.knobs_tensor(cfg.knobs), S.seeds_tensor(cfg.seeds()), 300)
    agg = s.aggregate(out["detail"], len(cfg.knobs), cfg.n_seeds)
    parts = torch.cat([agg, agg, agg])
    red = s.aggregate_reduce(parts, 3, len(cfg.knobs))
    torch.cuda.synchronize()
    a = S.unpack(agg, AGG_DTYPE)
    r3 = S.unpack(red, AGG_DTYPE)
    for ci in range(0, len(cfg.knobs), 7):
        refs = [orc.run(cfg.workloads, cfg.knobs[ci], sd, 300) for sd in cfg.seeds()]
        ra = climb.aggregate(refs)
        for f in ("sum_p99_us", "sum_slo_met", "sum_window_us", "n_seeds", "flags"):
            assert int(a[ci][f]) == ra[f]
            if f != "flags":
                assert int(r3[ci][f]) == 3 * ra[f]
    s.close()


@pytest.mark.parametrize("variant", ["live-wide32", "sim-controller", "sim-space"])
def test_device_climb_matches_oracle(S, orc, variant):
    """K3 (score, argmax, move, best-so-far, EMA, next stencil) over several Alg. 1 steps, against
    oracle/climb.py fed with oracle replicas: identical scores, moves and trajectories (C4-shaped, reduced
    sizes); also the paper's simulator controller (10 lambda, draft/verifier cost, EMA p99: P:173-174)."""
    from oracle import climb
    from paper_2603_11340_b200._lib import CLIMB_DTYPE
    wls = [inputs.preset_ll()]
    space, sp = {"live-wide32": (inputs.SPACE_WIDE32, dict(inputs.SCORE_DEFAULTS)),
                 "sim-controller": (inputs.SPACE_WIDE32, dict(inputs.SCORE_SIM)),
                 "sim-space": (inputs.SPACE_SIM, dict(inputs.SCORE_SIM, strict_alg1=0))}[variant]
    n_seeds, N, n_cand = 4, 400, 32
    seeds = inputs.seeds(n_seeds, 31)
    s = S.Simulator(wls, device=0)
    K = dict(inputs.K0)
    cands_t = s.candidates(space, K, n_cand)
    state_t = s.climb_state(K)
    seeds_t = S.seeds_tensor(seeds)
    ost = climb.initial_state(K)
    ocands = [K] + climb.neighbours(space, K)
    ocands += [inputs.PAD_KNOBS] * (n_cand - len(ocands))
    for step in range(4):
        out = s.run_batch(cands_t, seeds_t, N)
        aggs = s.aggregate(out["detail"], n_cand, n_seeds)
        scores = torch.empty(n_cand, dtype=torch.int64, device="cuda")
        s.hillclimb_step(space, sp, cands_t, aggs, 1, state_t, scores)
        torch.cuda.synchronize()
        oaggs = [climb.aggregate([orc.run(wls, c, sd, N) for sd in seeds]) for c in ocands]
        ost, moved, idx, oscores = climb.step(ost, ocands, oaggs, sp)
        assert scores.cpu().tolist() == oscores, step
        st = S.unpack(state_t, CLIMB_DTYPE)[0]
        assert int(st["moved"]) == int(moved) and int(st["argmax"]) == idx
        assert S.unpack_knobs(st["K"])[0] == ost["K"]
        assert int(st["S_best_micro"]) == ost["S_best"]
        assert S.unpack_knobs(st["K_best"])[0] == ost["K_best"]
        assert int(st["has_ema"]) == int(ost["has_ema"]) and int(st["ema_p99_us"]) == int(ost["ema"])
        ocands = [ost["K"]] + climb.neighbours(space, ost["K"])
        ocands += [inputs.PAD_KNOBS] * (n_cand - len(ocands))
        assert S.unpack_knobs(cands_t.cpu().numpy())[: int(st["n_next"])] == ocands[: int(st["n_next"])]
    s.close()


def test_launch_shapes_agree(S, orc):
    """The result does not depend on the launch shape (warps per block, blocks per SM)."""
    wls = [inputs.preset_ll()]
    cfg = inputs.config_c3(n_seeds=4, segment_len=500)
    base = _run_gpu(S, wls, cfg.knobs, cfg.seeds(), 500, latencies=True)
    for wpb, bps in ((1, 1), (8, 0), (2, 3)):
        g = _run_gpu(S, wls, cfg.knobs, cfg.seeds(), 500, latencies=True, warps_per_block=wpb, blocks_per_sm=bps)
        assert np.array_equal(g["lat"], base["lat"]) and np.array_equal(g["gp"], base["gp"])
    for pol in (1, 2):                                              # narrow / wide lane groups
        g = _run_gpu(S, wls, cfg.knobs, cfg.seeds(), 500, latencies=True, group_policy=pol)
        assert np.array_equal(g["lat"], base["lat"]) and g["detail"].tobytes() == base["detail"].tobytes()
    # latency-row scratch split into many launch chunks (1 MiB -> 524 replicas per chunk of 63 x 4 = 252... )
    base_nl = _run_gpu(S, wls, cfg.knobs, cfg.seeds(), 500, latencies=False)
    g = _run_gpu(S, wls, cfg.knobs, cfg.seeds(), 500, latencies=False, scratch_mb=1)
    assert np.array_equal(g["p99"], base_nl["p99"]) and np.array_equal(g["gp"], base_nl["gp"])
    assert g["detail"].tobytes() == base_nl["detail"].tobytes()
    cfg2 = inputs.config_c3(n_seeds=40, segment_len=3000)            # 2520 replicas x 12 KB rows > 1 MiB
    a = _run_gpu(S, wls, cfg2.knobs, cfg2.seeds(), 3000, latencies=False)
    b = _run_gpu(S, wls, cfg2.knobs, cfg2.seeds(), 3000, latencies=False, scratch_mb=1)
    assert np.array_equal(a["p99"], b["p99"]) and a["detail"].tobytes() == b["detail"].tobytes()
    assert a["stats"].tobytes() == b["stats"].tobytes()


def test_device_climb_seed_sharded_parts(S):
    """The N>1 layout: per-rank aggregates over seed slices, stacked in rank order and summed by K3,
    give exactly the single-part climb step (integer sums)."""
    from paper_2603_11340_b200._lib import CLIMB_DTYPE
    from paper_2603_11340_b200.dist import seed_block
    cfg = inputs.config_c4(n_seeds=10, segment_len=300)
    space, sp = cfg.extra["space"], cfg.extra["score"]
    s = S.Simulator(cfg.workloads, device=0)
    seeds = cfg.seeds()
    states, cands_out = [], []
    for world in (1, 3):
        cands = s.candidates(space, cfg.knobs[0], 32)
        state = s.climb_state(cfg.knobs[0])
        for _ in range(3):
            parts = []
            for rank in range(world):
                lo, hi = seed_block(len(seeds), rank, world)
                out = s.run_batch(cands, S.seeds_tensor(seeds[lo:hi]), cfg.segment_len)
                parts.append(s.aggregate(out["detail"], 32, hi - lo))
            s.hillclimb_step(space, sp, cands, torch.cat(parts), world, state)
        torch.cuda.synchronize()
        states.append(S.unpack(state, CLIMB_DTYPE)[0].tobytes())
        cands_out.append(cands.cpu().numpy().tobytes())
    assert states[0] == states[1] and cands_out[0] == cands_out[1]
    s.close()


def test_climb_cuda_graph_matches_eager(S):
    """NEXT-4: the climb step captured in a CUDA graph and replayed gives the same trajectory (state and
    candidate lists, bit for bit) as the eager host loop."""
    from paper_2603_11340_b200.dist import ClimbGraph, hillclimb
    cfg = inputs.config_c4(n_seeds=6, segment_len=400)
    s = S.Simulator(cfg.workloads, device=0)
    st_e, c_e = hillclimb(s, cfg, 5, cfg.seeds())
    g = ClimbGraph(s, cfg, cfg.seeds()).capture()
    st_g, c_g = g.run(5)
    torch.cuda.synchronize()
    assert torch.equal(st_e, st_g) and torch.equal(c_e, c_g)
    s.close()


def test_sweep_graph_matches_eager(S):
    """dist.SweepGraph (bench.py's replay for latency-bound sweeps): the captured run + aggregation replayed gives
    the same per-replica outputs and per-config aggregates, bit for bit, as the eager calls."""
    from paper_2603_11340_b200.dist import SweepGraph
    rng = random.Random(44)
    wls = _wls()
    ks = [inputs.random_knobs(rng, n_wl=len(wls)) for _ in range(12)] + [inputs.knobs(conc=8, max_num_seqs=16)]
    seeds = inputs.seeds(3, 9)
    s = S.Simulator(wls, device=0)
    kt, st = S.knobs_tensor(ks), S.seeds_tensor(seeds)
    out = s.run_batch(kt, st, 700, warmup_len=20, slo_us=900_000)
    agg = s.aggregate(out["detail"], len(ks), len(seeds))
    g = SweepGraph(s, kt, st, 700, 20, 900_000).capture()
    for _ in range(3):
        g.graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out["p99_us"], g.out["p99_us"]) and torch.equal(out["goodput"], g.out["goodput"])
    assert torch.equal(out["detail"], g.out["detail"]) and torch.equal(agg, g.agg)
    g.close()
    s.close()


def test_short_segment_window_ends_at_last_measured_completion(S, orc):
    """Segments shorter than a batch with warmup: the goodput window T ends at the last MEASURED completion
    (DESIGN.md §2.8), which can precede a warmup member's completion in the same final batch."""
    wls = [inputs.preset_ll(rate=100.0), inputs.workload(kind=0, rate=400.0)]
    ks = [inputs.knobs(conc=16, max_num_seqs=16), inputs.knobs(conc=32, max_num_seqs=32, workload=1),
          inputs.knobs(conc=8, max_num_seqs=8, draft_len=4, spec_on=1)]
    seeds = inputs.seeds(40, 4321)
    for N, warm in ((1, 3), (2, 5), (3, 4), (5, 10)):
        g = _run_gpu(S, wls, ks, seeds, N, warmup=warm)
        for ci, k in enumerate(ks):
            for si, sd in enumerate(seeds):
                _compare_replica(orc, g, ci * len(seeds) + si, wls, k, sd, N, warm, 1_200_000)


def _wls_cont():
    """Continuous-batching workloads next to a static one in the same handle, so one launch
    runs K1 and K1c side by side."""
    c = inputs.continuous
    return [c(inputs.preset_ll()), c(inputs.preset_sim()), c(inputs.preset_stress(kind=1)),
            c(inputs.preset_stress(kind=2)), c(inputs.preset_ll(rate=40.0, stream_id=7)),
            c(inputs.preset_closed(stream_id=3)), inputs.preset_ll(rate=20.0, stream_id=9),
            c(inputs.workload(kind=0, rate=200.0, timing=dict(inputs.LL_TIMING, noise_step_ppm=0), stream_id=5))]


@pytest.mark.parametrize("gen", [1, 2], ids=["inline", "split"])
@pytest.mark.parametrize("policy", [1, 2], ids=["narrow", "wide"])
@pytest.mark.parametrize("block", range(6))
def test_continuous_random_configs(S, orc, block, policy, gen):
    """Continuous batching: random knob records over every arrival kind (incl. the closed loop), noise on
    and off, speculation, several 32-request windows, ragged tails and warmup — every latency, p50/p95/p99,
    goodput and the work counters bit-exact against the oracle's iteration-level event loop."""
    rng = random.Random(900 + block)
    wls = _wls_cont()
    ks = [inputs.random_knobs(rng, n_wl=len(wls)) for _ in range(24)]
    ks[0] = inputs.knobs(conc=32, max_num_seqs=32, draft_len=16, spec_on=1, accept_q16=65536, workload=1)
    ks[1] = inputs.knobs(conc=1, max_num_seqs=1, draft_len=16, spec_on=1, accept_q16=0)
    ks[2] = inputs.knobs(conc=32, max_num_seqs=1, workload=2)
    ks[3] = inputs.knobs(conc=1, max_num_seqs=32, workload=3)
    ks[4] = inputs.knobs(conc=24, max_num_seqs=6, draft_len=4, spec_on=1, workload=5)       # closed loop
    ks[5] = inputs.knobs(conc=32, max_num_seqs=32, workload=7, draft_len=5, spec_on=1)      # no noise, overload
    ks[6] = inputs.knobs(conc=8, max_num_seqs=8, workload=6)                                # static, same launch
    ks[7] = inputs.knobs(conc=3, max_num_seqs=32, workload=4, draft_len=6, spec_on=1)      # G >= min(C, B) = 3
    ks[8] = inputs.knobs(conc=32, max_num_seqs=5, workload=5)                              # C + B > 4G
    seeds = inputs.seeds(3, 31 * block)
    N = rng.choice([37, 333, 1000, 1234])
    warmup = rng.choice([0, 0, 17, 100])
    g = _run_gpu(S, wls, ks, seeds, N, warmup=warmup, group_policy=policy, gen_policy=gen)
    tot = dict(batches=0, decode_steps=0, member_steps=0, philox_blocks=0)
    for ci, k in enumerate(ks):
        for si, sd in enumerate(seeds):
            ref = _compare_replica(orc, g, ci * len(seeds) + si, wls, k, sd, N, warmup, 1_200_000)
            for f in tot:
                tot[f] += ref["counters"][f]
    for f in tot:
        assert int(g["stats"][f]) == tot[f], f


def test_continuous_edge_cases(S, orc):
    """Continuous batching at degenerate sizes: one request, N < 32, exactly 32/33/65, short segments with a
    long warmup, B = 1 (pinned equal to static batching), invalid records mixed in."""
    wls = _wls_cont()
    ks = [inputs.knobs(conc=8, max_num_seqs=16), inputs.knobs(conc=0), inputs.knobs(max_num_seqs=1, conc=4),
          inputs.knobs(conc=32, max_num_seqs=32, workload=7), inputs.knobs(conc=3, max_num_seqs=2, workload=7,
                                                                            draft_len=3, spec_on=1),
          inputs.knobs(conc=16, max_num_seqs=4, workload=5, draft_len=8, spec_on=1, draft_width=3)]
    seeds = inputs.seeds(3, 1900)
    for N, warm in ((1, 0), (1, 5), (2, 5), (31, 0), (32, 1), (33, 0), (65, 64)):
        g = _run_gpu(S, wls, ks, seeds, N, warmup=warm)
        for ci, k in enumerate(ks):
            for si, sd in enumerate(seeds):
                r = ci * len(seeds) + si
                if not orc.knobs_valid(k, len(wls)):
                    assert int(g["p99"][r]) == 0xFFFFFFFF and g["gp"][r] == -1.0 and g["detail"][r]["flags"] == 1
                    continue
                _compare_replica(orc, g, r, wls, k, sd, N, warm, 1_200_000)


def test_continuous_full_size_sampled(S, orc):
    """The C2 knob grid served with continuous batching at full size (32,768 replicas x 10k requests) in the
    bench's launch configuration; sampled replicas bit-exact, properties on all."""
    cfg = inputs.config_c2_cont()
    g = _run_gpu(S, cfg.workloads, cfg.knobs, cfg.seeds(), cfg.segment_len, latencies=False)
    rng = random.Random(12)
    for ci in _sample_rows(len(cfg.knobs), 12, rng, must=(0, len(cfg.knobs) - 1)):
        si = rng.randrange(cfg.n_seeds)
        _compare_replica(orc, g, ci * cfg.n_seeds + si, cfg.workloads, cfg.knobs[ci], cfg.seeds()[si],
                         cfg.segment_len, 0, cfg.slo_us, check_lat=False)
    d = g["detail"]
    assert np.all(d["slo_met"] <= d["n_measured"]) and np.all(d["flags"] & 1 == 0)
    assert int(g["stats"]["requests"]) == cfg.requests


def test_climb_run_host_trajectory(S):
    """The end-to-end climb call (ClimbGraph.run_host, used by bench.py's c4 e2e): starting point copied in
    from pinned host memory, every step's climb state read back — equal, step by step, to the eager loop."""
    from paper_2603_11340_b200.dist import ClimbGraph, hillclimb
    cfg = inputs.config_c4(n_seeds=4, segment_len=300)
    s = S.Simulator(cfg.workloads, device=0)
    g = ClimbGraph(s, cfg, cfg.seeds()).capture()
    steps = 4
    h_c = g.init_cands.cpu().pin_memory()
    h_s = g.init_state.cpu().pin_memory()
    traj = torch.empty((steps, h_s.numel()), dtype=torch.uint8).pin_memory()
    g.run_host(steps, h_c, h_s, traj)
    for i in range(steps):
        st_e, _ = hillclimb(s, cfg, i + 1, cfg.seeds())
        torch.cuda.synchronize()
        assert torch.equal(traj[i], st_e.cpu().view(-1)), f"step {i}"
    s.close()


def test_continuous_launch_shapes_and_chunks_agree(S):
    """Continuous batching: the result does not depend on warps per block, blocks per SM, the lane-group
    policy or on splitting the launch into latency-row chunks."""
    cfg = inputs.config_c2_cont(n_seeds=6, segment_len=700)
    ks = cfg.knobs[::7]
    base = _run_gpu(S, cfg.workloads, ks, cfg.seeds(), 700, latencies=True)
    for kw in (dict(warps_per_block=1, blocks_per_sm=1), dict(warps_per_block=8), dict(group_policy=1),
               dict(group_policy=2)):
        g = _run_gpu(S, cfg.workloads, ks, cfg.seeds(), 700, latencies=True, **kw)
        assert np.array_equal(g["lat"], base["lat"]) and g["detail"].tobytes() == base["detail"].tobytes(), kw
        assert g["stats"].tobytes() == base["stats"].tobytes(), kw
    a = _run_gpu(S, cfg.workloads, ks, cfg.seeds(), 700, latencies=False)
    b = _run_gpu(S, cfg.workloads, ks, cfg.seeds(), 700, latencies=False, scratch_mb=1)   # 1.19 MiB of rows: 2 chunks
    assert np.array_equal(a["p99"], b["p99"]) and a["detail"].tobytes() == b["detail"].tobytes()
    assert a["stats"].tobytes() == b["stats"].tobytes()


def test_philox_peak_kernel_is_deterministic(S):
    """K4 (measurement only): positive throughput, and the XOR-folded blocks are the same on every run (every
    block is computed, nothing is elided)."""
    s = S.Simulator([inputs.preset_ll()], device=0)
    from paper_2603_11340_b200._lib import lib
    sm = s.info()["sm_count"]
    a = torch.zeros(sm * 2048, dtype=torch.int32, device="cuda")
    b = torch.ones(sm * 2048, dtype=torch.int32, device="cuda")
    assert lib().slo_philox_peak(s.h, 16, a.data_ptr(), None) == 0
    assert lib().slo_philox_peak(s.h, 16, b.data_ptr(), None) == 0
    torch.cuda.synchronize()
    assert torch.equal(a, b) and int((a != 0).sum()) > sm * 2000
    assert s.philox_peak(iters=256, repeats=1) > 1e10
    s.close()


def test_maximum_segment_and_saturated_latencies(S, orc):
    """The largest replica the ABI allows (warmup + segment = SLO_MAX_REQUESTS = 2^22 requests), static and
    continuous, one of them overloaded so far past the knee that latencies pass 2^32 - 1 us (stored
    saturated, flags bit 1): p99, SLO count, window, latency sum, flags and goodput bit-exact."""
    N = 1 << 22
    wls = [inputs.preset_ll(rate=10.0), inputs.continuous(inputs.preset_ll(rate=10.0)),
           inputs.preset_ll(rate=2000.0)]
    ks = [inputs.knobs(conc=8, max_num_seqs=16), inputs.knobs(conc=6, max_num_seqs=4, workload=1, draft_len=4,
                                                               spec_on=1),
          inputs.knobs(conc=32, max_num_seqs=2, workload=2)]                        # ~20x overload
    seeds = inputs.seeds(1, 4242)
    g = _run_gpu(S, wls, ks, seeds, N - 100, warmup=100, latencies=False)
    for ci, k in enumerate(ks):
        ref = _compare_replica(orc, g, ci, wls, k, seeds[0], N - 100, 100, 1_200_000, check_lat=False)
        if ci == 2:
            assert ref["flags"] & 2 and int(g["detail"][2]["flags"]) & 2
    # the ABI refuses one request more
    from paper_2603_11340_b200._lib import SloError
    with pytest.raises(SloError):
        _run_gpu(S, wls, ks[:1], seeds, N - 99, warmup=100, latencies=False)


def test_pareto_front_matches_oracle(S):
    """K5: the device's O(n log n) front equals the oracle's
    O(n^2) definition on random aggregates with many ties, invalid records and saturated goodput, and on the
    aggregates of a real C2-grid sweep."""
    from oracle import pareto
    from paper_2603_11340_b200._lib import AGG_DTYPE
    s = S.Simulator([inputs.preset_ll()], device=0)
    rng = np.random.default_rng(8)
    for n in (1, 2, 37, 1000, 3000):
        a = np.zeros(n, AGG_DTYPE)
        a["n_seeds"] = rng.integers(0, 5, n)
        a["sum_p99_us"] = rng.integers(0, 6, n) * 100_000 * a["n_seeds"]
        a["sum_window_us"] = rng.integers(1, 4, n) * 10**6
        a["sum_slo_met"] = rng.integers(0, 8, n)
        a["flags"] = (rng.random(n) < 0.05).astype(np.uint32)
        a[0]["sum_slo_met"], a[0]["sum_window_us"] = 2**63, 1                  # goodput saturates u64
        dev = torch.from_numpy(a.view(np.uint8).reshape(n, 32).copy()).cuda()
        f, cnt = s.pareto_front(dev, count=True)
        torch.cuda.synchronize()
        rows = [dict(zip(AGG_DTYPE.names, (int(v) for v in r))) for r in a]
        ref = pareto.pareto_front(rows)
        assert f.cpu().numpy().astype(bool).tolist() == ref and int(cnt.item()) == sum(ref), n
    cfg = inputs.config_c2(n_seeds=4, segment_len=500)
    out = s.run_batch(S.knobs_tensor(cfg.knobs), S.seeds_tensor(cfg.seeds()), 500)
    agg = s.aggregate(out["detail"], len(cfg.knobs), 4)
    f = s.pareto_front(agg)
    torch.cuda.synchronize()
    rows = [dict(zip(AGG_DTYPE.names, (int(v) for v in r))) for r in S.unpack(agg, AGG_DTYPE)]
    assert f.cpu().numpy().astype(bool).tolist() == pareto.pareto_front(rows)
    s.close()


def test_climb_trajectory_jsonl(S, orc, tmp_path):
    """ClimbGraph.trajectory (SPEC S:257/S:300 TuningTrajectory as JSON lines): every step's evaluated
    candidates and scores equal oracle/climb.py's Eq. (3) on oracle replicas, and its move, argmax and next K
    equal the oracle's Alg. 1 step."""
    import json
    from oracle import climb
    from paper_2603_11340_b200.dist import ClimbGraph
    cfg = inputs.config_c4(n_seeds=3, segment_len=300)
    s = S.Simulator(cfg.workloads, device=0)
    g = ClimbGraph(s, cfg, cfg.seeds()).capture()
    recs = g.trajectory(3, path=tmp_path / "traj.jsonl")
    lines = [json.loads(l) for l in open(tmp_path / "traj.jsonl")]
    assert lines == json.loads(json.dumps(recs)) and len(lines) == 3
    state = climb.initial_state(cfg.knobs[0])
    for r in lines:
        cands = r["candidates"]
        aggs = [climb.aggregate([orc.run(cfg.workloads, k, sd, 300) for sd in cfg.seeds()]) for k in cands]
        state, moved, am, scores = climb.step(state, cands, aggs, cfg.extra["score"])
        assert r["scores_micro"] == scores and r["moved"] == moved and r["argmax"] == am
        assert r["next"] == state["K"] and r["best"] == state["K_best"]
    s.close()


def test_pareto_front_properties_at_scale(S):
    """K5 on a 62,500-config sweep (the C5s grid, 2 seeds): properties that hold at any size — the front
    sorted by mean p99 has strictly increasing goodput, and every valid config off the front is dominated
    by a config on it (vectorised check of the definition against the front)."""
    from oracle import pareto
    from paper_2603_11340_b200._lib import AGG_DTYPE
    cfg = inputs.config_c5(stride=16, n_seeds=2, segment_len=400)
    s = S.Simulator(cfg.workloads, device=0)
    out = s.run_batch(S.knobs_tensor(cfg.knobs), S.seeds_tensor(cfg.seeds()), 400)
    agg = s.aggregate(out["detail"], len(cfg.knobs), 2)
    f = s.pareto_front(agg).cpu().numpy().astype(bool)
    a = S.unpack(agg, AGG_DTYPE)
    n = a["n_seeds"].astype(object)
    valid = (a["n_seeds"] > 0) & ((a["flags"] & 1) == 0) & (a["sum_window_us"] > 0)
    p = np.array([int(x) // int(k) if k else 0 for x, k in zip(a["sum_p99_us"], n)], dtype=np.int64)
    g = np.array([int(m) * 10**12 // int(w) if w else 0 for m, w in zip(a["sum_slo_met"], a["sum_window_us"])],
                 dtype=np.float64)                 # < 2^53 here (goodput < 10^3 rps)
    assert f.sum() > 0 and not (f & ~valid).any()
    fp, fg = p[f], g[f]
    order = np.lexsort((-fg, fp))
    up, ug = fp[order], fg[order]
    keep = np.r_[True, (up[1:] != up[:-1]) | (ug[1:] != ug[:-1])]
    assert np.all(np.diff(up[keep]) > 0) and np.all(np.diff(ug[keep]) > 0)
    off = np.where(valid & ~f)[0]
    for chunk in np.array_split(off, max(1, len(off) // 4096)):
        dom = ((fp[None, :] <= p[chunk, None]) & (fg[None, :] >= g[chunk, None]) &
               ((fp[None, :] < p[chunk, None]) | (fg[None, :] > g[chunk, None]))).any(axis=1)
        assert dom.all()
    # and the first 600 configs against the definition itself
    rows = [dict(zip(AGG_DTYPE.names, (int(v) for v in r))) for r in a[:600]]
    sub = s.pareto_front(agg[:600].contiguous()).cpu().numpy().astype(bool).tolist()
    assert sub == pareto.pareto_front(rows)
    s.close()


@pytest.mark.parametrize("gen", [1, 2], ids=["inline", "split"])
@pytest.mark.parametrize("cont", [0, 1], ids=["static", "continuous"])
def test_stop_rule_matches_oracle(S, orc, cont, gen):
    """NEXT-3 segment stop rule: with (n_min, t_min) the device stops each
    replica at t* — the first measured completion that is at least the n_min-th and t_min after t0 — and
    counts only requests completed by then; every stored latency (sentinels included), p50/p95/p99,
    n_measured, slo_met, window, sum, flags (bit 2: rule not met) and goodput equal the oracle's."""
    rng = random.Random(70 + cont)
    wls = _wls_cont() if cont else _wls()
    ks = [inputs.random_knobs(rng, n_wl=len(wls)) for _ in range(16)]
    ks[0] = inputs.knobs(conc=8, max_num_seqs=8, draft_len=4, spec_on=1, workload=5)       # closed loop
    seeds = inputs.seeds(2, 900 + cont)
    N, warm = 700, 30
    s = S.Simulator(wls, device=0, gen_policy=gen)
    for n_min, t_min in ((50, 0), (1, 3_000_000), (300, 20_000_000), (700, 0), (10, 10**9)):
        out = s.run_batch(S.knobs_tensor(ks), S.seeds_tensor(seeds), N, warmup_len=warm, latencies=True,
                          percentiles=True, stop_n_min=n_min, stop_t_min_us=t_min)
        torch.cuda.synchronize()
        from paper_2603_11340_b200._lib import RESULT_DTYPE
        lat = out["latencies"].cpu().numpy().view(np.uint32).reshape(-1, N + warm)
        det = S.unpack(out["detail"], RESULT_DTYPE)
        p99 = out["p99_us"].cpu().numpy().view(np.uint32)
        p50 = out["p50_us"].cpu().numpy().view(np.uint32)
        p95 = out["p95_us"].cpu().numpy().view(np.uint32)
        gp = out["goodput"].cpu().numpy()
        for ci, k in enumerate(ks):
            for si, sd in enumerate(seeds):
                r = ci * len(seeds) + si
                ref = orc.run(wls, k, sd, N, warmup_len=warm, latencies=True, stop_n_min=n_min,
                              stop_t_min_us=t_min)
                tag = f"stop {(n_min, t_min)} replica {r} knobs {k}"
                assert np.array_equal(lat[r], ref["latencies"]), tag
                assert (int(p99[r]), int(p50[r]), int(p95[r])) == (ref["p99_us"], ref["p50_us"], ref["p95_us"]), tag
                for f in ("slo_met", "n_measured", "window_us", "sum_latency_us", "flags"):
                    assert int(det[r][f]) == ref[f], (tag, f)
                assert gp[r] == ref["goodput"], tag
    s.close()
